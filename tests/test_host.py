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
