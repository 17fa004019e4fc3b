"""T3 parity on the TIMED path: the batched lockstep engine (fused protocol chains, the kernels
bench.py measures) in reference-stream mode must reproduce every party's share of every
materialised op output of the reference run of each image, bit for bit.

Oracle: oracle/sim.py (pinned to the reference's own runs in tests/test_oracle.py) with each
rank's numpy Generator -- S/engine.py:145-193 lanes 1 (weights), 3 (input shares, per
input_index), 4 (trusted source), 5 (party streams).  Image b of the batch is the reference's
run with input_index = b (S/engine.py:52-54; masks and party streams do not depend on it,
S/engine.py:64-74,166-171)."""

import numpy as np
import pytest
import torch

from oracle import sim

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2406_02629_b200 as pkg
    pkg._lib.load()
    return pkg


def _models(P):
    from paper_2406_02629_b200 import resnet
    ref_max, _ = P.build_reference_model(7, pool="max")
    ref_avg, _ = P.build_reference_model(7, pool="avg")
    return {"reference-max": ref_max, "reference-avg": ref_avg, "tiny-resnet": resnet.tiny_resnet(seed=3)}


def _inputs(P, model, B, seed):
    if hasattr(model, "random_inputs"):
        return model.random_inputs(seed, B)
    return np.stack([P.random_input(seed, model, index=b)[0] for b in range(B)])


def _weights(model):
    if hasattr(model, "weight_values"):
        return model.weight_values()
    return {name: qt.values for name, qt in model.weights.items()}


def _check(P, model, k, n, fuse, verify, B=3, seed=7):
    from paper_2406_02629_b200.batched import BatchedEngine
    scheme = P.SssScheme(P.PrimeField(), k, n)
    eng = BatchedEngine(model, scheme, batch=B, seed=seed, rng_mode="host", fuse=fuse, verify=verify)
    if fuse:
        assert eng.chains, "expected fused protocol chains on this model"
    x = _inputs(P, model, B, seed)
    cap = {}
    out = eng.run_device(torch.as_tensor(x), capture_shares=cap).cpu().numpy()
    ops = [op.meta() for op in eng.ops]
    wv = _weights(model)
    compared = 0
    for b in range(B):
        res = sim.simulate(ops, sim.Scheme(k, n), seed, x[b], wv, input_index=b, return_shares=True,
                           verify=verify)
        assert np.array_equal(out[b], res["output"]), (b, out[b], res["output"])
        assert res["checks_failed"] == 0
        for idx, got in cap.items():
            for r, (_, want) in res["values"][idx].items():
                g = got[r - 1][b].cpu().numpy().astype(np.uint64).reshape(-1)
                assert np.array_equal(g, np.asarray(want, dtype=np.uint64).reshape(-1)), \
                    f"op {idx} ({ops[idx]['kind']}) rank {r} image {b}"
                compared += g.size
    assert compared > 0
    return eng, cap


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
@pytest.mark.parametrize("mname", ["reference-max", "reference-avg", "tiny-resnet"])
def test_fused_chain_shares_equal_reference(P, mname, k, n):
    eng, cap = _check(P, _models(P)[mname], k, n, fuse=True, verify=False)
    # the fused chains' outputs are among the compared ops
    assert any(ch[-1] in cap for ch in eng.chains.values())


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
def test_unfused_shares_equal_reference(P, k, n):
    _check(P, _models(P)["tiny-resnet"], k, n, fuse=False, verify=False)


@pytest.mark.parametrize("fuse", [True, False])
def test_verified_run_shares_equal_reference(P, fuse):
    _check(P, _models(P)["tiny-resnet"], 3, 5, fuse=fuse, verify=True)


@pytest.mark.parametrize("verify", [False, True])
def test_fused_chain_4_7_shares_equal_reference(P, verify):
    """(4,7): the chain's factored reshare (wide R numerators, sub-shares folded before the
    B^-1 columns) and its 720-scaled TRUNC_MASKED, against the reference stream."""
    eng, cap = _check(P, _models(P)["tiny-resnet"], 4, 7, fuse=True, verify=verify, B=2)
    assert any(ch[-1] in cap for ch in eng.chains.values())


# ---------------------------------------------------------------- reference-composed fixtures
import json  # noqa: E402
import os  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _residual():
    with open(os.path.join(GOLD, "residual.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLD, "residual.npz"))


@pytest.mark.parametrize("fuse", [True, False])
def test_batched_residual_net_equals_reference_composed_fixture(P, fuse):
    """Residual DAG run through the reference's OWN sss_* ops (make_golden.residual_goldens)
    vs the batched engine (fused chains with the gathered stem pool, residual add and the /16
    average) in reference-stream mode: every rank's share of every materialised op output."""
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.batched import BatchedEngine
    meta, arr = _residual()
    net = resnet.tiny_resnet(seed=3)
    for k, n in ((2, 3), (3, 5)):
        cases = [c for c in meta["cases"] if (c["k"], c["n"]) == (k, n)]
        x = np.stack([arr[c["tag"] + "/x"] for c in cases])
        eng = BatchedEngine(net, P.SssScheme(P.PrimeField(), k, n), batch=len(cases), seed=cases[0]["seed"],
                            rng_mode="host", fuse=fuse)
        assert [op.meta() for op in eng.ops] == meta["ops"]
        cap = {}
        out = eng.run_device(torch.as_tensor(x), capture_shares=cap,
                             input_indices=[c["input_index"] for c in cases]).cpu().numpy()
        compared = 0
        for b, c in enumerate(cases):
            assert np.array_equal(out[b], arr[c["tag"] + "/out"])
            for idx, got in cap.items():
                if str(idx) not in c["held"]:          # the fixture skips the local gather op
                    continue
                ranks = c["held"][str(idx)]
                want = arr[f"{c['tag']}/shares/{idx}"]
                for row, r in enumerate(ranks):
                    assert np.array_equal(got[r - 1][b].cpu().numpy().astype(np.uint64).reshape(-1), want[row]), \
                        (k, n, b, idx, r)
                    compared += 1
        assert compared > 10


def test_per_party_api_residual_transcript_equals_reference(P):
    """The per-party API path (simulate_schedule: one thread per rank over the DeviceHub, the
    reference's seam) on the residual DAG reproduces the reference-composed run's SimHub
    transcript sha256 and outputs."""
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.engine import simulate_schedule
    from paper_2406_02629_b200.layers import plan_schedule
    meta, arr = _residual()
    net = resnet.tiny_resnet(seed=3)
    for c in meta["cases"]:
        scheme = P.SssScheme(P.PrimeField(), c["k"], c["n"])
        ops, digest = plan_schedule(net, scheme)
        res = simulate_schedule(ops, digest, scheme, c["seed"], input_int=arr[c["tag"] + "/x"],
                                weight_values=net.weight_values(), input_index=c["input_index"], rng_mode="host",
                                record=True, timeout=600)
        assert np.array_equal(res.output, arr[c["tag"] + "/out"])
        assert res.transcript_digest() == c["transcript_digest"], c["tag"]


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
def test_acceptance_100_inputs_batched(P, k, n):
    """T/test_acceptance.py:155-176 (criterion 03): 100 inputs through the timed batched
    engine in one launch sequence, both randomness modes, == the reference's 100 runs."""
    from paper_2406_02629_b200.batched import BatchedEngine
    arr = np.load(os.path.join(GOLD, "acceptance.npz"))
    model, _ = P.build_reference_model(7, pool="max")
    scheme = P.SssScheme(P.PrimeField(), k, n)
    want = arr[f"out_{k}{n}"]
    for mode in ("host", "device"):
        eng = BatchedEngine(model, scheme, batch=100, seed=7, rng_mode=mode)
        got = eng.run_device(torch.as_tensor(arr["x"])).cpu().numpy()
        assert np.array_equal(got, want), mode


def test_acceptance_transcripts_per_party_api(P):
    """Transcript sha256 of every tenth acceptance run through the per-party API."""
    with open(os.path.join(GOLD, "acceptance.json")) as fh:
        meta = json.load(fh)
    arr = np.load(os.path.join(GOLD, "acceptance.npz"))
    model, _ = P.build_reference_model(7, pool="max")
    for k, n in ((2, 3), (3, 5)):
        scheme = P.SssScheme(P.PrimeField(), k, n)
        for idx in range(0, 100, 10):
            res = P.simulate_inference(model, scheme, 7, arr["x"][idx], input_index=idx, record=True)
            assert np.array_equal(res.output, arr[f"out_{k}{n}"][idx])
            assert res.transcript_digest() == meta["transcripts"][f"{k}{n}"][idx]
