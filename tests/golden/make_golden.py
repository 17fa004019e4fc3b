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


def _gather_obj(x, kh, kw, stride, pad):
    """Builder op "gather" on one party's reference share values (object ndarray, c x h x w):
    window (oy, ox) tap (dy, dx) -> block position (oy*kh+dy, ox*kw+dx), share 0 outside.
    Written out with explicit loops here, independently of oracle.window_gather."""
    c, h, w = x.shape
    oh, ow = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    out = np.zeros((c, oh * kh, ow * kw), dtype=object)
    for oy in range(oh):
        for ox in range(ow):
            for dy in range(kh):
                for dx in range(kw):
                    sy, sx = oy * stride - pad + dy, ox * stride - pad + dx
                    if 0 <= sy < h and 0 <= sx < w:
                        out[:, oy * kh + dy, ox * kw + dx] = x[:, sy, sx]
    return out


def residual_goldens():
    """A residual network run through the REFERENCE's own secure ops (SURVEY.md section 7
    step 1): per rank one thread over ssnet's SimHub, each op dispatched to ssnet's
    sss_linear / sss_truncation / sss_nonlinear / share_add / output_collect, with the
    reference's dealing (lanes 1, 3), trusted source (lane 4) and party streams (lane 5).
    The DAG (residual adds, the gathered 3x3/s2 stem pool, the /16 average) comes from the
    builder's tiny ResNet; the only builder-side step is the local window gather.  Masks:
    the reference's trusted_source_prepare over the schedule with every local op ("add",
    "gather") replaced by an "output" placeholder, so op indices and draw order line up.
    Stores the decoded outputs and every rank's share of every op output."""
    import threading
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_2406_02629_b200 import resnet as R
    from ssnet.engine import deal_input_shares, deal_weight_shares, receive_bundle, seeded_rng, send_bundles
    from ssnet.layers import sss_linear, sss_nonlinear, sss_truncation
    from ssnet.protocol import PartyContext, output_collect
    from ssnet.sss import share_add
    from ssnet.transport import SimHub
    net = R.tiny_resnet(seed=3)
    dag = net.op_dicts()
    ref_fields = [fl.name for fl in ScheduledOp.__dataclass_fields__.values()]

    def ref_op(m, placeholder=False):
        kw = {k: m[k] for k in ref_fields if k in m}
        kw["in_shape"], kw["out_shape"] = tuple(m["in_shape"]), tuple(m["out_shape"])
        kw["pool"] = tuple(m["pool"]) if m["pool"] else None
        if placeholder:
            kw.update(kind="output", pool=None, pool_kind=None)
        return ScheduledOp(**kw)

    ops = [ref_op(m) if m["kind"] not in ("add", "gather") else None for m in dag]
    src_ops = [ref_op(m, placeholder=m["kind"] in ("add", "gather")) for m in dag]
    weights = net.weight_values()
    arrays, cases = {}, []
    xs = net.random_inputs(5, 2)
    for k, n in ((2, 3), (3, 5)):
        scheme = SssScheme(F, k, n)
        for index in range(2):
            seed = 7
            x = xs[index]
            hub = SimHub(range(0, n + 1))
            wsh = deal_weight_shares(weights, scheme, seed)
            xsh = deal_input_shares(x, scheme, seed, index)
            vals_by_rank, outputs, errors = {}, {}, {}

            def party(rank):
                def run():
                    try:
                        ctx = PartyContext(scheme, rank, hub.transport(rank), rng=seeded_rng(seed, 5, rank))
                        receive_bundle(ctx)
                        vals = {-1: xsh[rank - 1]}
                        for idx, m in enumerate(dag):
                            x_ = vals.get(m.get("src", idx - 1))
                            kind = m["kind"]
                            if kind == "linear":
                                y = sss_linear(ctx, ops[idx], x_, wsh[rank][m["weight"] + ".w"],
                                               wsh[rank][m["weight"] + ".b"], ctx.bundle.take(idx, "zero"))
                            elif kind == "truncation":
                                y = sss_truncation(ctx, ops[idx], x_, ctx.bundle.take(idx, "alpha"),
                                                   ctx.bundle.take(idx, "comp"))
                            elif kind == "nonlinear":
                                y = sss_nonlinear(ctx, ops[idx], x_, ctx.bundle.take(idx, "beta"),
                                                  ctx.bundle.take(idx, "beta_inv"))
                            elif kind == "add":
                                o = vals.get(m["src2"])
                                y = share_add(x_, o) if (x_ is not None and o is not None) else None
                            elif kind == "gather":
                                y = None
                                if x_ is not None:
                                    g = _gather_obj(np.asarray(x_.values).reshape(tuple(m["in_shape"])),
                                                    m["pool"][0], m["pool"][1], m["stride"], m["padding"])
                                    y = ShareTensor(x_.party_id, x_.degree, g, scheme)
                            elif kind == "output":
                                vals[idx] = x_
                                out = output_collect(ctx, x_)
                                if out is not None:
                                    outputs[rank] = out
                                break
                            vals[idx] = y
                        vals_by_rank[rank] = vals
                    except BaseException as exc:       # surface thread errors
                        errors[rank] = exc
                return run

            threads = [threading.Thread(target=lambda: send_bundles(hub.transport(0), src_ops, scheme, seed))]
            threads += [threading.Thread(target=party(r)) for r in range(1, n + 1)]
            for t in threads:
                t.start()
            for t in threads:
                t.join(600)
            if errors:
                raise errors[sorted(errors)[0]]
            tag = f"tiny-resnet/{k}{n}/{index}"
            arrays[tag + "/x"] = x.astype(np.int64)
            arrays[tag + "/out"] = np.asarray(np.asarray(outputs[1]).tolist(), dtype=np.int64)
            held = {}
            for idx, m in enumerate(dag):
                if m["kind"] == "gather":
                    continue
                ranks = [r for r in range(1, n + 1) if vals_by_rank[r].get(idx) is not None]
                held[idx] = ranks
                arrays[f"{tag}/shares/{idx}"] = np.stack([u64(vals_by_rank[r][idx].values).reshape(-1)
                                                          for r in ranks])
            cases.append({"tag": tag, "k": k, "n": n, "input_index": index, "seed": seed, "held": held,
                          "transcript_digest": hub.transcript_digest()})
    with open(os.path.join(OUT, "residual.json"), "w") as fh:
        json.dump({"model": "tiny-resnet(seed=3)", "input_seed": 5, "ops": dag, "cases": cases}, fh, indent=1,
                  sort_keys=True)
    np.savez_compressed(os.path.join(OUT, "residual.npz"), **arrays)


def acceptance_goldens():
    """T/test_acceptance.py:155-176 (criterion 03): 100 inputs x {(2,3), (3,5)} through the
    reference's simulate_schedule on the reference model -- decoded outputs, the rank-1..n
    output shares and the SimHub transcript digest of every run."""
    model, _ = build_reference_model(seed=7, pool="max")
    weights = {name: qt.values for name, qt in model.weights.items()}
    arrays, meta = {}, {}
    xs = np.stack([random_input(7, model, index=i)[0] for i in range(100)])
    arrays["x"] = xs.astype(np.int64)
    for k, n in ((2, 3), (3, 5)):
        scheme = SssScheme(F, k, n)
        ops, sdig = plan_schedule(model, scheme)
        outs, digests = [], []
        for idx in range(100):
            res = simulate_schedule(ops, sdig, scheme, 7, input_int=xs[idx], weight_values=weights,
                                    input_index=idx, timeout=600)
            assert np.all(res.output == plaintext_infer(model, xs[idx]))
            outs.append(res.output.astype(np.int64))
            digests.append(res.transcript_digest())
        arrays[f"out_{k}{n}"] = np.stack(outs)
        meta[f"{k}{n}"] = digests
    np.savez_compressed(os.path.join(OUT, "acceptance.npz"), **arrays)
    with open(os.path.join(OUT, "acceptance.json"), "w") as fh:
        json.dump({"model": "reference-max(seed=7)", "seed": 7, "transcripts": meta}, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["unit", "vectors", "engine", "residual", "acceptance"]
    if "unit" in which:
        with open(os.path.join(OUT, "unit.json"), "w") as fh:
            json.dump(unit_goldens(), fh, indent=1, sort_keys=True)
    if "vectors" in which:
        vector_goldens()
    if "engine" in which:
        engine_goldens()
    if "residual" in which:
        residual_goldens()
    if "acceptance" in which:
        acceptance_goldens()
    print("golden fixtures written to", OUT)
