"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures (small .json/.npz files in this directory) are committed; nothing on the
GPU box reads /root/reference.  Every value here comes out of the reference's own
functions (ssnet.*), so they pin both the CPU oracle (oracle/) and the CUDA path.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from ssnet.engine import simulate_schedule, estimate_report  # noqa: E402
from ssnet.field import PrimeField  # noqa: E402
from ssnet.layers import (_window_decode, comm_estimate, plan_schedule,  # noqa: E402
                          ScheduledOp)
from ssnet.masks import (additive_mask_bound, gen_additive_mask,  # noqa: E402
                         gen_multiplicative_mask, multiplicative_mask_bound)
from ssnet.metrics import CommMetrics  # noqa: E402
from ssnet.model import (build_reference_model, im2col, plaintext_infer, pool_blocks,  # noqa: E402
                         random_input, round_half_away, ModelGraph, Conv2D, Dense,
                         Truncation, NonLinear, QuantizedTensor)
from ssnet.sss import ShareTensor, SssScheme  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
F = PrimeField()
P = F.p


def u64(a):
    return np.asarray(np.asarray(a, dtype=object).tolist(), dtype=np.uint64)


def unit_goldens():
    F11 = PrimeField(11)
    g = {}
    s11 = SssScheme(F11, 2, 3)
    g["f11_gen_2_9"] = [int(v.values) for v in s11.gen(2, coeffs=[9])]
    g["f11_gen_2_4"] = [int(v.values) for v in s11.gen(2, coeffs=[4])]
    g["f11_gen_3_1"] = [int(v.values) for v in s11.gen(3, coeffs=[1])]
    g["f11_lagrange_12"] = list(s11.lagrange_weights((1, 2)))
    g["f11_lagrange_123"] = list(s11.lagrange_weights((1, 2, 3)))
    g["f11_R"] = [[int(v) for v in row] for row in s11.reducing_matrix()]
    g["f11_zero_4"] = [int(v.values) for v in s11.gen(0, coeffs=[4])]
    for k, n in ((2, 3), (3, 5), (4, 7)):
        s = SssScheme(F, k, n)
        g[f"R_{k}{n}"] = [[int(v) for v in row] for row in s.reducing_matrix()]
        g[f"lag_front_{k}{n}"] = list(s.lagrange_weights(s.front_ids))
        g[f"lag_part_{k}{n}"] = list(s.lagrange_weights(s.participating_ids))
    g["p"] = P
    g["split_anchor"] = int(F.split_mul(1 << 23, 1 << 23))
    g["window_decode_f11"] = [int(_window_decode(v, -3, 11)) for v in range(11)]
    vals = list(range(-12, 13))
    g["round_half_away_in"] = vals
    g["round_half_away_d4"] = [int(round_half_away(v, 4)) for v in vals]
    g["round_half_away_d3"] = [int(round_half_away(v, 3)) for v in vals]
    g["inv_samples"] = [[a, int(F.inv(a))] for a in (1, 2, 3, 12345, P - 1, 2 ** 40 + 7)]
    # mask bounds (S/masks.py)
    g["emax"] = [[st, vb, additive_mask_bound(F, st, vb)]
                 for st, vb in ((4096, 2 ** 43 - 1), (4096 * 49, 2 ** 40), (8, 1000), (1, 5))]
    g["bmax"] = [[vb, multiplicative_mask_bound(F, vb)] for vb in (32776, 32776 * 4, 2 ** 43)]
    return g


def vector_goldens():
    rng = np.random.default_rng(20261017)
    out = {}
    for k, n in ((2, 3), (3, 5)):
        s = SssScheme(F, k, n)
        secret = F.rand(rng, (257,))
        coeffs = [F.rand(rng, (257,)) for _ in range(k - 1)]
        shares = s.gen(secret, coeffs=coeffs)
        out[f"gen_secret_{k}{n}"] = u64(secret)
        out[f"gen_coeffs_{k}{n}"] = u64(np.stack(coeffs))
        out[f"gen_shares_{k}{n}"] = u64(np.stack([st.values for st in shares]))
        # degree-(2k-2) product shares -> rec over all participants
        a = s.gen(F.rand(rng, (300,)), rng)
        b = s.gen(F.rand(rng, (300,)), rng)
        m = 2 * k - 1
        prod = [ShareTensor(a[i].party_id, 2 * k - 2, a[i].values * b[i].values % P, s)
                for i in range(m)]
        out[f"rec_in_{k}{n}"] = u64(np.stack([pt.values for pt in prod]))
        out[f"rec_out_{k}{n}"] = u64(s.rec(prod, m=m))
        # reducing-matrix apply (S/protocol.py:176-178)
        R = s.reducing_matrix()
        flat = np.stack([pt.values for pt in prod])
        out[f"reduce_out_{k}{n}"] = u64((R.T @ flat) % P)
        # truncation elite composition (S/layers.py:295-308), reference functions
        for (r, d, vb) in ((1 << 12, 1, 2 ** 42), (1 << 12, 49, 2 ** 40), (8, 4, 1000)):
            x = rng.integers(-vb + 1, vb, size=(400,))
            xs = s.gen(F.encode_signed(x.astype(object)), rng)
            alpha, comp, e = gen_additive_mask((400,), r, d, s, rng, vb)
            masked = [ShareTensor(xs[i].party_id, k - 1, (xs[i].values + alpha[i].values) % P, s)
                      for i in range(k)]
            v = s.rec(masked, m=k)
            shifted = _window_decode(v, -vb + r * d, P)
            t = shifted // r
            if d > 1:
                t = round_half_away(t, d)
            tag = f"trunc_{k}{n}_{r}_{d}"
            out[tag + "_masked"] = u64(np.stack([mk.values for mk in masked]))
            out[tag + "_t"] = u64(t % P)
            out[tag + "_x"] = x.astype(np.int64)
            out[tag + "_e"] = np.asarray(e.tolist(), dtype=np.int64)
            out[tag + "_vb"] = np.array([vb, r, d], dtype=np.int64)
        # nonlinear elite composition (S/layers.py:347-364)
        for pool, kind in ((None, None), ((2, 2), "max"), ((2, 2), "sum"), ((3, 3), "max")):
            shape = (3, 6, 6)
            x = rng.integers(-(2 ** 15), 2 ** 15, size=shape)
            xs = s.gen(F.encode_signed(x.astype(object)), rng)
            beta, beta_inv, bplain = gen_multiplicative_mask(shape, s, rng, pool=pool,
                                                             value_bound=2 ** 15 + 8)
            masked = [ShareTensor(xs[i].party_id, 2 * k - 2, xs[i].values * beta[i].values % P, s)
                      for i in range(m)]
            v = s.rec(masked, m=m)
            ints = F.decode_signed(v)
            ints = np.where(ints > 0, ints, 0)
            if kind == "max":
                ints = pool_blocks(ints, *pool).max(axis=(2, 4))
            elif kind == "sum":
                ints = pool_blocks(ints, *pool).sum(axis=(2, 4))
            plain = F.encode_signed(ints)
            tag = f"nonlin_{k}{n}_{kind}_{pool[0] if pool else 0}"
            out[tag + "_masked"] = u64(np.stack([mk.values for mk in masked]))
            out[tag + "_plain"] = u64(plain)
            out[tag + "_binv0"] = u64(beta_inv[0].values)
            out[tag + "_unmask0"] = u64(plain * beta_inv[0].values % P)
    # exact object-dtype GEMM (S/layers.py:252)
    for (M, K, N) in ((7, 13, 5), (33, 200, 65), (64, 576, 49)):
        A = F.rand(rng, (M, K))
        B = F.rand(rng, (K, N))
        out[f"gemm_{M}_{K}_{N}_A"] = u64(A)
        out[f"gemm_{M}_{K}_{N}_B"] = u64(B)
        out[f"gemm_{M}_{K}_{N}_C"] = u64((A @ B) % P)
    # im2col on a field tensor (S/model.py:354-371)
    x = F.rand(rng, (3, 7, 9))
    out["im2col_x"] = u64(x)
    out["im2col_s2p1"] = u64(im2col(x, 3, 3, 2, 1))
    # inverses (S/field.py:101-116)
    a = F.rand(rng, (64,))
    a[a == 0] = 1
    out["inv_in"] = u64(a)
    out["inv_out"] = u64(F.inv(a))
    np.savez_compressed(os.path.join(OUT, "vectors.npz"), **out)


def small_models():
    """Extra chain models (beyond the reference LeNet) exercising dense-only and
    avg-pool paths, built from the reference's own layer kinds."""
    rng = np.random.default_rng(5)
    layers = [Conv2D("c1", 3, (3, 3), stride=2, padding=1), Truncation(10),
              NonLinear(relu=True, pool="avg", pool_kh=2, pool_kw=2),
              Dense("d1", 6), Truncation(10), NonLinear(relu=True),
              Dense("d2", 4), Truncation(10)]
    w = {"c1.w": QuantizedTensor(rng.integers(-3000, 3000, (3, 2, 3, 3)), 12, 16),
         "c1.b": QuantizedTensor(rng.integers(-100000, 100000, (3,)), 19, 32),
         "d1.w": QuantizedTensor(rng.integers(-3000, 3000, (6, 12)), 12, 16),
         "d1.b": QuantizedTensor(rng.integers(-100000, 100000, (6,)), 19, 32),
         "d2.w": QuantizedTensor(rng.integers(-3000, 3000, (4, 6)), 12, 16),
         "d2.b": QuantizedTensor(rng.integers(-100000, 100000, (4,)), 19, 32)}
    return {"mini-avg": ModelGraph("mini-avg", (2, 8, 8), layers, w, input_scale_bits=7)}


def engine_goldens():
    cases = []
    models = {"reference-max": build_reference_model(7, pool="max")[0],
              "reference-avg": build_reference_model(7, pool="avg")[0]}
    models.update(small_models())
    arrays = {}
    for mname, model in models.items():
        weights = {name: qt.values for name, qt in model.weights.items()}
        for name, v in weights.items():
            arrays[f"{mname}/w/{name}"] = v.astype(np.int64)
        for (k, n) in ((2, 3), (3, 5)):
            scheme = SssScheme(F, k, n)
            orders = ("ltn", "lnt") if mname == "reference-max" else ("ltn",)
            for ordering in orders:
                ops, digest = plan_schedule(model, scheme, ordering)
                for idx, seed in ((0, 7), (3, 11)):
                    x, _ = random_input(seed, model, index=idx)
                    metrics = CommMetrics()
                    res = simulate_schedule(ops, digest, scheme, seed, input_int=x,
                                            weight_values=weights, metrics=metrics,
                                            input_index=idx, timeout=600)
                    tag = f"{mname}/{k}{n}/{ordering}/{idx}"
                    arrays[tag + "/x"] = x.astype(np.int64)
                    arrays[tag + "/out"] = res.output.astype(np.int64)
                    cases.append({
                        "model": mname, "k": k, "n": n, "ordering": ordering,
                        "input_index": idx, "seed": seed, "tag": tag,
                        "schedule_digest": digest.hex(),
                        "transcript_digest": res.transcript_digest(),
                        "ops": [op.meta() for op in ops],
                        "summary": metrics.summary(),
                        "estimate": comm_estimate(ops, scheme),
                        "plaintext_equal": bool(np.all(
                            res.output == plaintext_infer(model, x, mode="merged"))),
                        "arch": model.arch_meta(),
                    })
    np.savez_compressed(os.path.join(OUT, "engine.npz"), **arrays)
    with open(os.path.join(OUT, "engine.json"), "w") as fh:
        json.dump(cases, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    with open(os.path.join(OUT, "unit.json"), "w") as fh:
        json.dump(unit_goldens(), fh, indent=1, sort_keys=True)
    vector_goldens()
    engine_goldens()
    print("golden fixtures written to", OUT)
