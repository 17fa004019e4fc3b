"""Reference arm: the UNMODIFIED reference package (ssnet, pure Python + numpy object arrays),
installed into baseline/_ref by tools/install_reference.sh, timed through its own public API
(`ssnet.simulate_inference`, S/engine.py:196-204) on the box's host cores.

Chain models (the reference's own LeNet-style graphs, config 1) run whole: one image per step.

Residual networks cannot be expressed in the reference's ModelGraph (no residual add,
S/model.py:148-149), and one ResNet-152 image takes the reference about an hour, so they are
timed PER OP: every unique (conv/dense shape, followed-by-ReLU) of the
network becomes a reference ModelGraph  Conv2D -> Truncation [-> NonLinear(relu)]  with the
same C_in, kernel, stride and padding but few output channels and a small output map, run
through ssnet.simulate_inference at two output-channel counts; the per-output-element slope of
the two runs (its fixed per-run overhead cancels) times the layer's real output elements is
the layer's time.  The stem max-pool and the global average pool are timed the same way as
reference NonLinear layers.  The network's time is the sum over its layers (the reference runs
op after op).  Conservative for the reference: the fixed per-run cost, the residual share_adds
and im2col's per-pixel cost (constant across the two channel counts) are not charged, and the
reference has no Reed-Solomon verification step to pay for.
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The installed reference package, or (None, reason)."""
    if not os.path.isdir(os.path.join(REF_DIR, "ssnet")):
        return None, f"{REF_DIR} missing (run tools/install_reference.sh)"
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import ssnet
    except Exception as exc:            # reported, never replaced silently
        return None, f"import ssnet failed: {exc!r}"
    if not os.path.realpath(ssnet.__file__).startswith(os.path.realpath(REF_DIR)):
        return None, f"ssnet imported from {ssnet.__file__}, not {REF_DIR}"
    return ssnet, None


def to_reference_graph(ssnet, model):
    """Our mirror ModelGraph (same layer vocabulary and weights) -> the reference's class."""
    from ssnet.model import ModelGraph, QuantizedTensor, layers_from_meta
    meta = model.arch_meta()
    w = {k: QuantizedTensor(np.asarray(v.values), v.scale_bits, v.bits) for k, v in model.weights.items()}
    return ModelGraph(meta["name"], meta["input_shape"], layers_from_meta(meta["layers"]), w,
                      meta["input_scale_bits"])


def _conv_graph(ssnet, C, O, k, stride, pad, oh, relu, seed):
    from ssnet.model import Conv2D, ModelGraph, NonLinear, QuantizedTensor, Truncation
    h = (oh - 1) * stride + k - 2 * pad
    rng = np.random.default_rng(seed)
    w = QuantizedTensor(rng.integers(-2000, 2000, size=(O, C, k, k)), 12, 16)
    b = QuantizedTensor(rng.integers(-(1 << 18), 1 << 18, size=(O,)), 19, 32)
    layers = [Conv2D("c", O, (k, k), stride, pad), Truncation(12)] + ([NonLinear(True, None)] if relu else [])
    g = ModelGraph("sample", (C, h, h), layers, {"c.w": w, "c.b": b})
    return g, rng.integers(-100, 100, size=(C, h, h))


def _dense_graph(ssnet, F_in, O, relu, seed):
    from ssnet.model import Dense, ModelGraph, NonLinear, QuantizedTensor, Truncation
    rng = np.random.default_rng(seed)
    w = QuantizedTensor(rng.integers(-2000, 2000, size=(O, F_in)), 12, 16)
    b = QuantizedTensor(rng.integers(-(1 << 18), 1 << 18, size=(O,)), 19, 32)
    layers = [Dense("d", O), Truncation(12)] + ([NonLinear(True, None)] if relu else [])
    g = ModelGraph("sample", (F_in,), layers, {"d.w": w, "d.b": b})
    return g, rng.integers(-100, 100, size=(F_in,))


def _pool_graph(ssnet, C, oh, kh, kind, seed):
    from ssnet.model import ModelGraph, NonLinear, Truncation
    rng = np.random.default_rng(seed)
    if kind == "max":
        layers = [NonLinear(True, "max", kh, kh)]
    else:                       # average pool: the reference requires a divide step before it
        layers = [Truncation(1), NonLinear(True, "avg", kh, kh)]
    g = ModelGraph("sample", (C, oh * kh, oh * kh), layers, {})
    return g, rng.integers(0, 100, size=(C, oh * kh, oh * kh))


def sample_plan(model):
    """[(spec, real output elements, count)] for a ResNetGraph, unique specs merged."""
    shp = model.shapes()
    nodes = model.nodes
    plan = {}

    def add(spec, elems):
        e, c = plan.get(spec, (0, 0))
        plan[spec] = (e + elems, c + 1)

    for i, nd in enumerate(nodes):
        if nd.kind in ("conv", "dense"):
            # the ReLU that consumes this layer's truncation (directly, not via an add)
            relu = any(n2.kind == "relu" and n2.src == i + 1 and n2.pool is None for n2 in nodes)
            out = shp[i]
            if nd.kind == "conv":
                spec = ("conv", shp[nd.src][0], nd.kernel, nd.stride, nd.padding, relu)
            else:
                spec = ("dense", int(np.prod(shp[nd.src])), relu)
            add(spec, int(np.prod(out)))
        elif nd.kind == "add":
            # relu after the residual add: a separate masked nonlinearity over the sum
            if any(n2.kind == "relu" and n2.src == i and n2.pool is None for n2 in nodes):
                add(("relu",), int(np.prod(shp[i])))
        elif nd.kind == "relu" and nd.pool is not None:
            add(("pool", nd.pool_kind, nd.pool[0]), int(np.prod(shp[i])))
    return [(spec, e, c) for spec, (e, c) in plan.items()]


def _relu_graph(ssnet, C, hw, seed):
    from ssnet.model import ModelGraph, NonLinear
    rng = np.random.default_rng(seed)
    g = ModelGraph("sample", (C, hw, hw), [NonLinear(True, None)], {})
    return g, rng.integers(-100, 100, size=(C, hw, hw))


def _run(ssnet, scheme, graph, x):
    t0 = time.perf_counter()
    ssnet.simulate_inference(graph, scheme, 7, x)
    return time.perf_counter() - t0


def time_op(ssnet, scheme, spec, seed=0):
    """Seconds per output element of one sampled op (slope of two reference runs)."""
    kind = spec[0]
    if kind == "conv":
        _, C, k, stride, pad, relu = spec
        oh = 2 if k >= 3 else 4
        pts = []
        for O in (8, 24):
            g, x = _conv_graph(ssnet, C, O, k, stride, pad, oh, relu, seed)
            pts.append((O * oh * oh, _run(ssnet, scheme, g, x)))
    elif kind == "dense":
        _, F_in, relu = spec
        pts = []
        for O in (8, 32):
            g, x = _dense_graph(ssnet, F_in, O, relu, seed)
            pts.append((O, _run(ssnet, scheme, g, x)))
    elif kind == "relu":
        pts = []
        for C in (8, 32):
            g, x = _relu_graph(ssnet, C, 8, seed)
            pts.append((C * 64, _run(ssnet, scheme, g, x)))
    else:                               # ("pool", kind, window)
        _, pk, kh = spec
        pts = []
        for C in (4, 16):
            g, x = _pool_graph(ssnet, C, 2, kh, "max" if pk == "max" else "avg", seed)
            pts.append((C * 4, _run(ssnet, scheme, g, x)))
    (e1, t1), (e2, t2) = pts
    return max(t2 - t1, 0.0) / (e2 - e1), t1 + t2


def describe(spec):
    if spec[0] == "conv":
        return f"conv C={spec[1]} {spec[2]}x{spec[2]}/s{spec[3]}/p{spec[4]}{' +relu' if spec[5] else ''}"
    if spec[0] == "dense":
        return f"dense F={spec[1]}{' +relu' if spec[2] else ''}"
    if spec[0] == "relu":
        return "relu (after residual add)"
    return f"{spec[1]} pool {spec[2]}x{spec[2]}"


def reference_step(ssnet, model, k, n, seed=0):
    """One reference-arm step.  Returns (seconds per image, wall seconds spent, sample text,
    per-op table)."""
    scheme = ssnet.SssScheme(ssnet.PrimeField(), k, n)
    t0 = time.perf_counter()
    if not hasattr(model, "nodes"):                 # a reference-expressible chain model: whole run
        g = to_reference_graph(ssnet, model)
        from paper_2406_02629_b200.model import random_input
        x = random_input(1, model, 0)[0]
        _run(ssnet, scheme, g, x)
        wall = time.perf_counter() - t0
        return wall, wall, f"ssnet.simulate_inference, full {n}PC run of {model.name}, 1 image", None
    total, rows = 0.0, []
    for spec, elems, count in sample_plan(model):
        per, _ = time_op(ssnet, scheme, spec, seed)
        total += per * elems
        rows.append({"op": describe(spec), "layers": count, "elements": elems, "s": round(per * elems, 3)})
    wall = time.perf_counter() - t0
    text = (f"ssnet.simulate_inference per op: {len(rows)} unique layer shapes of {model.name}, each as a "
            f"reference ModelGraph at two sample sizes (slope per output element x real elements), summed; "
            f"{wall:.1f} s of sampling for an extrapolated {total:.0f} s per image")
    return total, wall, text, rows


def gemm_rate(ssnet, S=96, reps=2):
    """The reference's share GEMM expression `(w @ x) % p` on object arrays (S/layers.py:254),
    field ops per second (size-independent: O(S^3) bignum multiply-adds)."""
    F = ssnet.PrimeField()
    rng = np.random.default_rng(0)
    a = F.rand(rng, (S, S))
    b = F.rand(rng, (S, S))
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        (a @ b) % F.p
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return 2.0 * S ** 3 / best, S
