"""End-to-end parity of the reference-API mirror on the GPU: decoded outputs, the full
SimHub transcript digest (every message byte) and CommMetrics against fixtures produced by
the reference itself (tests/golden/engine.*), plus the reference's per-op tests."""

import json
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import sim

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ssn():
    import paper_2406_02629_b200 as pkg
    pkg._lib.load()
    return pkg


@pytest.fixture(scope="module")
def engine():
    with open(os.path.join(GOLD, "engine.json")) as fh:
        cases = json.load(fh)
    return cases, np.load(os.path.join(GOLD, "engine.npz"))


def _model(ssn, case, arr):
    from paper_2406_02629_b200.model import (Conv2D, Dense, ModelGraph, NonLinear, QuantizedTensor,
                                             Truncation)
    arch = case["arch"]
    layers = []
    for item in arch["layers"]:
        if item["kind"] == "conv":
            layers.append(Conv2D(item["name"], item["out_channels"], tuple(item["kernel"]), item["stride"],
                                 item["padding"]))
        elif item["kind"] == "dense":
            layers.append(Dense(item["name"], item["out_features"]))
        elif item["kind"] == "truncation":
            layers.append(Truncation(item["shift_bits"]))
        else:
            layers.append(NonLinear(item["relu"], item["pool"], item["pool_kh"], item["pool_kw"]))
    prefix = case["model"] + "/w/"
    weights = {}
    for key in arr.files:
        if key.startswith(prefix):
            name = key[len(prefix):]
            bits = 32 if name.endswith(".b") else 16
            weights[name] = QuantizedTensor(arr[key], 19 if bits == 32 else 12, bits)
    return ModelGraph(arch["name"], arch["input_shape"], layers, weights, arch["input_scale_bits"])


def test_reference_runs_bit_exact(ssn, engine):
    from paper_2406_02629_b200.metrics import CommMetrics
    cases, arr = engine
    F = ssn.PrimeField()
    for case in cases:
        model = _model(ssn, case, arr)
        scheme = ssn.SssScheme(F, case["k"], case["n"])
        ops, digest = ssn.plan_schedule(model, scheme, case["ordering"])
        assert digest.hex() == case["schedule_digest"]
        metrics = CommMetrics()
        res = ssn.simulate_inference(model, scheme, case["seed"], arr[case["tag"] + "/x"],
                                     ordering=case["ordering"], metrics=metrics,
                                     input_index=case["input_index"], record=True)
        assert np.array_equal(res.output, arr[case["tag"] + "/out"]), case["tag"]
        assert res.transcript_digest() == case["transcript_digest"], case["tag"]
        assert metrics.summary() == case["summary"], case["tag"]
        assert ssn.comm_estimate(ops, scheme) == case["estimate"]


def test_device_rng_mode_same_outputs(ssn, engine):
    cases, arr = engine
    F = ssn.PrimeField()
    for case in cases[::3]:
        model = _model(ssn, case, arr)
        scheme = ssn.SssScheme(F, case["k"], case["n"])
        res = ssn.simulate_inference(model, scheme, case["seed"] + 100, arr[case["tag"] + "/x"],
                                     ordering=case["ordering"], input_index=case["input_index"],
                                     rng_mode="device")
        assert np.array_equal(res.output, arr[case["tag"] + "/out"]), case["tag"]


def test_verify_mode_outputs_and_counts(ssn, engine):
    from paper_2406_02629_b200.metrics import CommMetrics
    cases, arr = engine
    F = ssn.PrimeField()
    for case in cases:
        if case["ordering"] != "ltn" or case["input_index"] != 0:
            continue
        model = _model(ssn, case, arr)
        scheme = ssn.SssScheme(F, case["k"], case["n"])
        ops, _ = ssn.plan_schedule(model, scheme, verify=True)
        metrics = CommMetrics()
        res = ssn.simulate_inference(model, scheme, case["seed"], arr[case["tag"] + "/x"], metrics=metrics,
                                     verify=True)
        assert np.array_equal(res.output, arr[case["tag"] + "/out"])
        est = {(r["name"], r["layer"]): r["elements"] for r in ssn.comm_estimate(ops, scheme, verify=True)}
        for row in metrics.summary():
            if row["op"] != "offline":
                assert row["elements_sent"] == est[(row["op"], row["layer"])], row
        # oracle agrees on the verify-mode schedule
        want = sim.simulate([op.meta() for op in ops], sim.Scheme(case["k"], case["n"]), case["seed"],
                            arr[case["tag"] + "/x"], {k_: v.values for k_, v in model.weights.items()},
                            verify=True)
        assert want["checks_failed"] == 0


def test_plaintext_infer_on_device(ssn, engine):
    cases, arr = engine
    for case in cases[:4]:
        model = _model(ssn, case, arr)
        got = ssn.plaintext_infer(model, arr[case["tag"] + "/x"])
        assert np.array_equal(got, arr[case["tag"] + "/out"])
