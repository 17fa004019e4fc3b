"""tcgen05 limb GEMM (csrc/ssn_gemm_tc.cu) against the CUDA-core kernel and the CPU oracle.
Structured cases first so a layout bug shows up as a readable failure.  GPU only."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
P = oracle.DEFAULT_PRIME


@pytest.fixture(scope="module")
def g():
    import paper_2406_02629_b200 as pkg
    from paper_2406_02629_b200 import gemm
    pkg._lib.load()
    return gemm


def dev(a):
    return torch.as_tensor(np.asarray(a, dtype=np.uint64).astype(np.int64), device="cuda")


def host(t):
    return t.cpu().numpy().astype(np.uint64)


def _dense_both(g, w, x, nimg):
    tc = host(g.field_dense(dev(w), dev(x), P, nimg=nimg, force="tc"))
    simt = host(g.field_dense(dev(w), dev(x), P, nimg=nimg, force="simt"))
    return tc, simt


@pytest.mark.parametrize("case", ["limb0", "limb5", "ones", "maxval"])
def test_structured_dense(g, case):
    rows, O, K = 128, 32, 64
    if case == "limb0":
        w = np.arange(O * K, dtype=np.uint64).reshape(O, K) % 7
        x = np.arange(rows * K, dtype=np.uint64).reshape(rows, K) % 5
    elif case == "limb5":
        w = (np.arange(O * K, dtype=np.uint64).reshape(O, K) % 7) << np.uint64(40)
        x = (np.arange(rows * K, dtype=np.uint64).reshape(rows, K) % 5) << np.uint64(40)
    elif case == "ones":
        w = np.ones((O, K), dtype=np.uint64)
        x = np.ones((rows, K), dtype=np.uint64)
    else:
        w = np.full((O, K), P - 1, dtype=np.uint64)
        x = np.full((rows, K), P - 1, dtype=np.uint64)
    tc, simt = _dense_both(g, w, x, rows)
    want = oracle.gemm(x, w.T)                     # (rows, O)
    assert np.array_equal(simt.reshape(rows, O), want)
    assert np.array_equal(tc.reshape(rows, O), want), (case, tc.reshape(rows, O)[:2, :4], want[:2, :4])


@pytest.mark.parametrize("rows,O,K", [(128, 32, 64), (300, 48, 200), (1000, 64, 576), (257, 1000, 2048),
                                      (640, 96, 4608)])
def test_random_dense_shapes(g, rows, O, K):
    rng = np.random.default_rng(rows + O + K)
    w = rng.integers(0, P, size=(O, K), dtype=np.uint64)
    x = rng.integers(0, P, size=(rows, K), dtype=np.uint64)
    tc, simt = _dense_both(g, w, x, rows)
    assert np.array_equal(tc, simt)
    if rows * O * K <= 64 * 1024 * 1024:
        assert np.array_equal(tc.reshape(rows, O), oracle.gemm(x, w.T))


@pytest.mark.parametrize("C,H,W,O,k,s,pad,nimg,nparty", [
    (3, 32, 32, 64, 3, 1, 1, 2, 1),
    (64, 14, 14, 64, 1, 1, 0, 3, 2),
    (16, 15, 17, 48, 3, 2, 1, 2, 3),
    (3, 56, 56, 64, 7, 2, 3, 1, 1),
    (256, 7, 7, 128, 3, 1, 1, 4, 5),
    (1, 28, 28, 6, 5, 1, 2, 3, 3),              # LeNet-28 conv1: K = 25, O = 6
    (6, 14, 14, 16, 5, 1, 0, 2, 3),             # LeNet-28 conv2: K = 150
])
def test_conv_tc_vs_simt(g, C, H, W, O, k, s, pad, nimg, nparty):
    rng = np.random.default_rng(C * H + O)
    w = rng.integers(0, P, size=(nparty, O, C, k, k), dtype=np.uint64)
    x = rng.integers(0, P, size=(nparty, nimg, C, H, W), dtype=np.uint64)
    tc = g.field_conv(dev(w), dev(x), s, pad, P, nimg=nimg, nparty=nparty, force="tc")
    simt = g.field_conv(dev(w), dev(x), s, pad, P, nimg=nimg, nparty=nparty, force="simt")
    assert np.array_equal(host(tc), host(simt))
    # one party/image against the oracle's im2col GEMM
    want = oracle.gemm(w[0].reshape(O, -1), oracle.im2col(x[0, 0], k, k, s, pad))
    got = host(tc).reshape(nparty, nimg, O, -1)[0, 0] if (nparty > 1 or nimg > 1) else host(tc).reshape(O, -1)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("kh,C,H,W,O", [(1, 64, 56, 56, 64), (1, 128, 14, 14, 96), (3, 64, 56, 56, 64),
                                        (3, 128, 28, 28, 128), (3, 64, 14, 14, 32), (3, 64, 32, 32, 64),
                                        (3, 128, 16, 16, 128)])
def test_implicit_conv_planes_vs_im2col(kh, C, H, W, O):
    """Implicit GEMM from channel-major planes (TMA M-major A, modes 1 and 2) equals the
    explicit im2col + tcgen05 GEMM path bit for bit, including the zero padding of 3x3."""
    import torch
    from paper_2406_02629_b200 import _lib, gemm as G
    p = (1 << 45) - 55
    rng = np.random.default_rng(C + H + O + kh)
    nparty, B = 2, 4          # mode 1 needs B*H*W % 16 == 0 (TMA stride alignment)
    x = torch.as_tensor(rng.integers(0, p, size=(nparty, B, C, H, W)), device="cuda")
    w = torch.as_tensor(rng.integers(0, p, size=(nparty, O, C, kh, kh)), device="cuda")
    pad = (kh - 1) // 2
    want = G.field_conv(w, x, 1, pad, p, nimg=B, nparty=nparty, force="tc")
    mode = 1 if kh == 1 else 2
    Wp = W if mode == 1 else G.conv_row_pitch(W)
    L = G.limbs(p)
    copies = 1 if mode == 1 else 3
    planes = torch.zeros((copies, nparty, L, C, B, H, Wp), dtype=torch.uint8, device="cuda")
    _lib.call("ssn_planes_cn", _lib.ptr(x), nparty, B, C, H, W, Wp, L, _lib.ptr(planes), B * C * H * W,
              copies, _lib.stream_ptr())
    wt = w.permute(0, 1, 3, 4, 2).contiguous().reshape(nparty, O, kh * kh * C)
    bpl = G.weight_planes(wt, p, nparty)
    out = torch.empty((nparty, B, O, H, W), dtype=torch.int64, device="cuda")
    _lib.call("ssn_gemm_tc_conv", _lib.ptr(planes), mode, B, C, H, W, Wp, _lib.ptr(bpl), nparty, O, _lib.ptr(out),
              B * O * H * W, p, _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(out, want)


@pytest.mark.parametrize("rows,K,O", [(16, 2048, 1000), (40, 512, 64), (1, 256, 32), (300, 25, 6), (7, 84, 10),
                                      (129, 1, 3)])
def test_small_row_dense_on_tensor_cores(rows, K, O):
    """Partial 128-row tiles (TMA zero fill beyond the rows) stay exact: classifier-sized GEMMs."""
    from paper_2406_02629_b200 import gemm as G
    p = (1 << 45) - 55
    rng = np.random.default_rng(rows + K + O)
    w = torch.as_tensor(rng.integers(0, p, size=(2, O, K)), device="cuda")
    x = torch.as_tensor(rng.integers(0, p, size=(2, rows, K)), device="cuda")
    tc = G.field_dense(w, x, p, nimg=rows, nparty=2, force="tc")
    simt = G.field_dense(w, x, p, nimg=rows, nparty=2, force="simt")
    assert torch.equal(tc, simt)


@pytest.mark.parametrize("rows,O,K", [(256, 128, 11009), (256, 64, 16384), (384, 256, 16384)])
def test_split_k_dense_exact(g, rows, O, K):
    """K > 11,008 overflows the u32 limb-diagonal budget (L*K*255^2 < 2^32) and is split into
    exact partial GEMMs added mod p (gemm.field_matmul) -- the config-5 sweep's 16384^3 path.
    Against the CUDA-core 64x64->128 GEMM everywhere, and the CPU oracle on a row block."""
    rng = np.random.default_rng(K + O)
    w = rng.integers(0, P, size=(O, K), dtype=np.uint64)
    x = rng.integers(0, P, size=(rows, K), dtype=np.uint64)
    tc, simt = _dense_both(g, w, x, rows)
    assert np.array_equal(tc, simt)
    blk = slice(0, 16)
    assert np.array_equal(tc.reshape(rows, O)[blk], oracle.gemm(x[blk], w.T))


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
@pytest.mark.parametrize("kind,nparty", [("dense", 1), ("conv", 1), ("conv", 3)])
def test_fused_subshares_equal_gemm_then_gen(g, k, n, kind, nparty):
    """ssn_gemm_tc_subshares (GEMM epilogue writes the RESHARE_OUT sub-shares) == the share GEMM
    followed by ssn_gen over the front ids with (seed, stream + party) -- bit for bit."""
    from paper_2406_02629_b200 import _lib
    from paper_2406_02629_b200.field import PrimeField
    from paper_2406_02629_b200.sss import SssScheme
    rng = np.random.default_rng(k * 10 + nparty)
    sch = SssScheme(PrimeField(), k, n)
    if kind == "dense":
        B, O, K = 70, 100, 300
        w = dev(rng.integers(0, P, size=(nparty, O, K), dtype=np.uint64))
        x = dev(rng.integers(0, P, size=(nparty, B, K), dtype=np.uint64))
        N = B * O
        run = lambda sub=None: g.field_dense(w, x, P, nimg=B, nparty=nparty, force="tc", sub=sub)  # noqa: E731
    else:
        B, C, H, O = 2, 16, 10, 40
        w = dev(rng.integers(0, P, size=(nparty, O, C, 3, 3), dtype=np.uint64))
        x = dev(rng.integers(0, P, size=(nparty, B, C, H, H), dtype=np.uint64))
        N = B * O * 5 * 5
        run = lambda sub=None: g.field_conv(w, x, 2, 1, P, nimg=B, nparty=nparty, force="tc", sub=sub)  # noqa: E731
    acc = run().reshape(nparty, N)
    ids = _lib.u64_array(sch.front_ids)
    want = torch.empty((nparty, k, N), dtype=torch.int64, device="cuda")
    for pt in range(nparty):
        _lib.call("ssn_gen", _lib.ptr(acc[pt]), N, None, 0, 1234, 77 + pt, k - 1, ids, k, _lib.ptr(want[pt]),
                  k * N, N, N, 1, P, _lib.stream_ptr())
    got = torch.empty_like(want)
    assert run(g.SubShares(got, 1234, 77, k - 1, sch.front_ids)) is None
    assert torch.equal(got, want)
