"""CPU-only checks of the host side: the C ABI library loads and exports every symbol
include/ssn.h declares; the planner reproduces the reference's schedules, digests and
closed-form communication estimates; the metrics contract."""

import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_declared_symbol():
    from paper_2406_02629_b200 import _lib
    _lib.build()
    L = _lib.load(require_cuda=False)
    hdr = open(os.path.join(ROOT, "include", "ssn.h")).read()
    declared = set(re.findall(r"^int (ssn_\w+)\(", hdr, flags=re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(L, name), name
    assert declared <= set(_lib.exported_symbols())
    assert L.ssn_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    from paper_2406_02629_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.SsnUnavailable):
        _lib.load()


def test_planner_matches_reference_schedules():
    import paper_2406_02629_b200 as P
    from paper_2406_02629_b200.model import build_reference_model
    cases = json.load(open(os.path.join(GOLD, "engine.json")))
    F = P.PrimeField()
    seen = 0
    for case in cases:
        if not case["model"].startswith("reference"):
            continue
        model, _ = build_reference_model(7, pool=case["model"].split("-")[1])
        scheme = P.SssScheme(F, case["k"], case["n"])
        ops, digest = P.plan_schedule(model, scheme, case["ordering"])
        assert digest.hex() == case["schedule_digest"]
        assert [op.meta() for op in ops] == case["ops"]
        assert P.comm_estimate(ops, scheme) == case["estimate"]
        seen += 1
    assert seen >= 8


def test_full_layer_formula_and_constants():
    import paper_2406_02629_b200 as P
    assert [P.full_layer_formula(k) for k in (1, 2, 3)] == [3, 16, 35]
    unit = json.load(open(os.path.join(GOLD, "unit.json")))
    for k, n in ((2, 3), (3, 5), (4, 7)):
        s = P.SssScheme(P.PrimeField(), k, n)
        assert [list(r) for r in s.reducing_matrix()] == unit[f"R_{k}{n}"]
        assert list(s.lagrange_weights(s.front_ids)) == unit[f"lag_front_{k}{n}"]
    assert P.PrimeField().split_mul(1 << 23, 1 << 23) == unit["split_anchor"]


def test_scheme_validation_errors():
    import paper_2406_02629_b200 as P
    from paper_2406_02629_b200.sss import DuplicateIds
    F = P.PrimeField()
    with pytest.raises(ValueError):
        P.SssScheme(F, 2, 2)
    with pytest.raises(DuplicateIds):
        P.SssScheme(F, 2, 3, party_ids=(1, 2, 1 + F.p))
    with pytest.raises(ValueError):
        P.PrimeField(12)


def test_metrics_epochs():
    from paper_2406_02629_b200.metrics import CommMetrics
    m = CommMetrics()
    m.set_op(1, "op", 0)
    m.on_send(1, 10, 1)
    m.on_send(1, 10, 1)
    m.on_recv(1, 10, 1)
    m.on_send(1, 10, 1)
    assert m.rounds("op", 0) == 2
    assert m.elements_sent("op") == 3


def test_gathered_stem_pool_equals_overlapping_maxpool():
    """The builder op "gather" + the reference's non-overlapping max pool (S/model.py:374-377)
    is ResNet's 3x3 / stride 2 / pad 1 max-pool after ReLU (zero fill == -inf padding there)."""
    import torch
    import torch.nn.functional as F
    from oracle import window_gather
    rng = np.random.default_rng(3)
    for (c, h, w) in ((2, 16, 16), (3, 112, 112), (1, 7, 9)):
        x = rng.integers(-2 ** 15, 2 ** 15, size=(c, h, w))
        g = window_gather(np.maximum(x, 0), 3, 3, 2, 1)
        oh, ow = g.shape[1] // 3, g.shape[2] // 3
        pooled = g.reshape(c, oh, 3, ow, 3).max(axis=(2, 4))
        want = F.max_pool2d(torch.as_tensor(np.maximum(x, 0), dtype=torch.float64)[None], 3, 2, 1)[0]
        assert np.array_equal(pooled, want.numpy().astype(np.int64))


def test_resnet_head_is_true_average():
    """Global pool = round_half_away(sum / 49) (merged-divisor rounding, S/model.py:44-50)."""
    from paper_2406_02629_b200 import resnet
    g = resnet.imagenet_resnet(50, seed=7, classes=10)
    ops = g.plan_ops()
    tr = [op for op in ops if op.name == "div.gpool"][0]
    assert (tr.r, tr.divisor) == (1, 49)
    st = [op for op in ops if op.kind == "gather"]
    assert len(st) == 1 and st[0].pool == (3, 3) and (st[0].stride, st[0].padding) == (2, 1)
    assert tuple(st[0].out_shape) == (64, 168, 168)
