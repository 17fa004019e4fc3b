"""CUDA kernels vs golden vectors from the reference and vs the CPU oracle (GPU only).
Every call goes through the C ABI of libssn_b200.so."""

import os

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
P = oracle.DEFAULT_PRIME


@pytest.fixture(scope="module")
def ssn():
    import paper_2406_02629_b200 as pkg
    pkg._lib.load()
    return pkg


@pytest.fixture(scope="module")
def vec():
    return np.load(os.path.join(GOLD, "vectors.npz"))


def dev(a):
    return torch.as_tensor(np.asarray(a, dtype=np.uint64).astype(np.int64), device="cuda")


def host(t):
    return t.cpu().numpy().astype(np.uint64)


def call(ssn, name, *args):
    ssn._lib.call(name, *args)


def test_ewise_matches_oracle(ssn):
    rng = np.random.default_rng(1)
    for p in (P, 11, 144115188075855859, 1_000_003):     # largest 57-bit prime: S/field.py:75 cap
        a = rng.integers(0, p, size=10007, dtype=np.uint64)
        b = rng.integers(0, p, size=10007, dtype=np.uint64)
        F = ssn.PrimeField(p)
        for op in ("add", "sub", "mul"):
            got = host(getattr(F, op)(dev(a), dev(b)))
            assert np.array_equal(got, oracle.ewise(op, a, b, p)), (p, op)
        assert np.array_equal(host(F.neg(dev(a))), oracle.ewise("sub", np.zeros_like(a), a, p))
    # mulmod edge values for the default prime
    F = ssn.PrimeField()
    edge = np.array([0, 1, 2, P - 1, P - 2, (P - 1) // 2, 1 << 44, (1 << 45) - 56], dtype=np.uint64)
    aa, bb = np.meshgrid(edge, edge)
    got = host(F.mul(dev(aa.ravel()), dev(bb.ravel())))
    assert np.array_equal(got, oracle.ewise("mul", aa.ravel(), bb.ravel(), P))
    assert int(F.mul(dev([1 << 23]), dev([1 << 23]))[0]) == 110      # split_mul anchor


def test_gen_rec_reduce_vs_golden(ssn, vec):
    F = ssn.PrimeField()
    for k, n in ((2, 3), (3, 5)):
        s = ssn.SssScheme(F, k, n)
        coeffs = list(vec[f"gen_coeffs_{k}{n}"])
        shares = s.gen(dev(vec[f"gen_secret_{k}{n}"]), coeffs=[dev(c) for c in coeffs])
        assert np.array_equal(np.stack([host(st.values) for st in shares]), vec[f"gen_shares_{k}{n}"])
        m = 2 * k - 1
        pts = [ssn.ShareTensor(i + 1, 2 * k - 2, dev(v), s) for i, v in enumerate(vec[f"rec_in_{k}{n}"])]
        assert np.array_equal(host(s.rec(pts, m=m)), vec[f"rec_out_{k}{n}"])
        R = s.reducing_matrix()
        rt = [R[i][t] for t in range(n) for i in range(m)]
        stack = dev(vec[f"rec_in_{k}{n}"])
        out = torch.empty((n, stack.shape[1]), dtype=torch.int64, device="cuda")
        nel = stack.shape[1]
        call(ssn, "ssn_reduce_apply", ssn._lib.ptr(stack), 0, nel, m, ssn._lib.u64_array(rt), n,
             ssn._lib.ptr(out), 0, nel, nel, 1, P, ssn._lib.stream_ptr())
        assert np.array_equal(host(out), vec[f"reduce_out_{k}{n}"])


def test_trunc_elite_vs_golden(ssn, vec):
    F = ssn.PrimeField()
    for k, n in ((2, 3), (3, 5)):
        s = ssn.SssScheme(F, k, n)
        w = s.lagrange_weights(s.front_ids)
        for (r, d) in ((1 << 12, 1), (1 << 12, 49), (8, 4)):
            tag = f"trunc_{k}{n}_{r}_{d}"
            vb, r_, d_ = (int(v) for v in vec[tag + "_vb"])
            masked = dev(vec[tag + "_masked"])
            nel = masked.shape[1]
            t = torch.empty(nel, dtype=torch.int64, device="cuda")
            call(ssn, "ssn_trunc_elite", ssn._lib.ptr(masked), nel, k, k, ssn._lib.u64_array(w), None, vb, r_, d_,
                 None, 0, 0, 0, None, 0, ssn._lib.ptr(t), 0, None, nel, P, ssn._lib.stream_ptr())
            assert np.array_equal(host(t), vec[tag + "_t"]), tag


def test_nonlin_elite_vs_golden(ssn, vec):
    F = ssn.PrimeField()
    for k, n in ((2, 3), (3, 5)):
        s = ssn.SssScheme(F, k, n)
        m = 2 * k - 1
        w = s.lagrange_weights(s.party_ids[:m])
        for pool, kind in ((None, None), ((2, 2), "max"), ((2, 2), "sum"), ((3, 3), "max")):
            tag = f"nonlin_{k}{n}_{kind}_{pool[0] if pool else 0}"
            masked = dev(vec[tag + "_masked"].reshape(m, -1))
            kh, kw = pool or (1, 1)
            code = {None: 0, "max": 1, "sum": 2}[kind]
            c, h, wd = (3, 6, 6) if pool else (108, 1, 1)
            plain = torch.empty(vec[tag + "_plain"].size, dtype=torch.int64, device="cuda")
            call(ssn, "ssn_nonlin_elite", ssn._lib.ptr(masked), masked.shape[1], m, ssn._lib.u64_array(w), 1,
                 code, 1, c, h, wd, kh, kw, ssn._lib.ptr(plain), P, ssn._lib.stream_ptr())
            assert np.array_equal(host(plain), vec[tag + "_plain"].reshape(-1)), tag
            um = F.mul(plain, dev(vec[tag + "_binv0"].reshape(-1)))
            assert np.array_equal(host(um), vec[tag + "_unmask0"].reshape(-1))


def test_simt_gemm_vs_golden_and_oracle(ssn, vec):
    from paper_2406_02629_b200.gemm import field_conv, field_dense
    for (M, K, N) in ((7, 13, 5), (33, 200, 65), (64, 576, 49)):
        A = dev(vec[f"gemm_{M}_{K}_{N}_A"])
        B = vec[f"gemm_{M}_{K}_{N}_B"]
        got = np.stack([host(field_dense(A, dev(B[:, j]), P)) for j in range(N)], axis=1)
        assert np.array_equal(got, vec[f"gemm_{M}_{K}_{N}_C"])
        # batched over images in one launch
        out = field_dense(A, dev(B.T.copy()), P, nimg=N)
        assert np.array_equal(host(out).reshape(N, M).T, vec[f"gemm_{M}_{K}_{N}_C"])
    # conv stride 2 pad 1 vs im2col oracle
    rng = np.random.default_rng(3)
    x = rng.integers(0, P, size=(5, 9, 11), dtype=np.uint64)
    w = rng.integers(0, P, size=(6, 5, 3, 3), dtype=np.uint64)
    got = host(field_conv(dev(w), dev(x), 2, 1, P))
    want = oracle.gemm(w.reshape(6, -1), oracle.im2col(x, 3, 3, 2, 1))
    assert np.array_equal(got.reshape(6, -1), want)
    assert np.array_equal(oracle.im2col(vec["im2col_x"], 3, 3, 2, 1), vec["im2col_s2p1"])


def test_inverse_and_signed(ssn, vec):
    F = ssn.PrimeField()
    assert np.array_equal(host(F.inv(dev(vec["inv_in"]))), vec["inv_out"])
    with pytest.raises(ZeroDivisionError):
        F.inv(dev([0, 1]))
    x = np.array([-5, 0, 7, -(P - 1) // 2, (P - 1) // 2], dtype=np.int64)
    enc = F.encode_signed(torch.as_tensor(x, device="cuda"))
    assert np.array_equal(host(enc), oracle.encode_signed(x))
    assert np.array_equal(F.decode_signed(enc).cpu().numpy(), x)
    with pytest.raises(ValueError):
        F.encode_signed(torch.as_tensor([P], device="cuda"))


def test_f11_worked_examples_on_device(ssn):
    F11 = ssn.PrimeField(11)
    s = ssn.SssScheme(F11, 2, 3)
    assert [int(v.values) for v in s.gen(2, coeffs=[9])] == [0, 9, 7]
    a = s.gen(2, coeffs=[4])
    b = s.gen(3, coeffs=[1])
    prod = [ssn.share_mul(x, y) for x, y in zip(a, b)]
    assert [int(v.values) for v in prod] == [2, 6, 7]
    assert int(s.rec(prod, m=3)) == 6
    assert s.lagrange_weights((1, 2)) == (2, 10)
    assert [list(r) for r in s.reducing_matrix()] == [[6, 9, 1], [1, 5, 9], [5, 9, 2]]


def test_device_rng_masks_are_valid_sharings(ssn):
    """Speed-mode trusted source: alpha = e*step, comp = -e with e in [1, emax]; beta window
    constant with beta * beta^-1 == 1; zero shares reconstruct to 0."""
    from paper_2406_02629_b200.masks import gen_additive_mask, gen_multiplicative_mask, gen_zero_shares
    from paper_2406_02629_b200.rng import DeviceRng
    F = ssn.PrimeField()
    for k, n in ((2, 3), (3, 5)):
        s = ssn.SssScheme(F, k, n)
        rng = DeviceRng(5, k)
        al, cp, _ = gen_additive_mask((4, 8, 8), 4096, 4, s, rng, 2 ** 40)
        a = host(s.rec(al[:k]))
        c = host(s.rec(cp[n - k:]))
        e = (P - c.astype(object)) % P
        assert np.all(e >= 1) and np.all(a.astype(object) == (e * 4096 * 4) % P)
        bt, bi, _ = gen_multiplicative_mask((4, 8, 8), s, rng, pool=(2, 2), value_bound=2 ** 16)
        beta = host(s.rec(bt[1:k + 1])).reshape(4, 4, 2, 4, 2)
        assert np.all(beta == beta[:, :, :1, :, :1])
        binv = host(s.rec(bi[:k]))
        prod = oracle.ewise("mul", beta[:, :, 0, :, 0].reshape(-1), binv.reshape(-1))
        assert np.all(prod == 1)
        z = gen_zero_shares((100,), s, rng)
        assert np.all(host(s.rec(z[:k])) == 0)
        assert len({int(v) for v in host(z[0].values)}) > 90


def test_inverse_table():
    """ssn_inv_table: table[b] * b == 1 (mod p) on samples of [1, 2^20), table[0] == 0."""
    import torch
    from paper_2406_02629_b200 import _lib
    p = (1 << 45) - 55
    n = 1 << 20
    t = torch.empty(n, dtype=torch.int64, device="cuda")
    _lib.call("ssn_inv_table", _lib.ptr(t), n, p, _lib.stream_ptr())
    tab = t.cpu().numpy()
    assert tab[0] == 0
    rng = np.random.default_rng(5)
    for b in list(rng.integers(1, n, size=200)) + [1, 2, n - 1, 63, 64, 65]:
        assert int(tab[b]) * int(b) % p == 1, b
