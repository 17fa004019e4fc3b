"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import json
import os

import numpy as np
import pytest

import oracle
from oracle import sim

GOLD = os.path.join(os.path.dirname(__file__), "golden")
P = oracle.DEFAULT_PRIME


@pytest.fixture(scope="module")
def unit():
    with open(os.path.join(GOLD, "unit.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def vec():
    return np.load(os.path.join(GOLD, "vectors.npz"))


@pytest.fixture(scope="module")
def engine():
    with open(os.path.join(GOLD, "engine.json")) as fh:
        cases = json.load(fh)
    return cases, np.load(os.path.join(GOLD, "engine.npz"))


def test_f11_worked_examples(unit):
    assert list(oracle.gen([2], [[9]], (1, 2, 3), 11)[:, 0]) == unit["f11_gen_2_9"] == [0, 9, 7]
    assert list(oracle.gen([2], [[4]], (1, 2, 3), 11)[:, 0]) == unit["f11_gen_2_4"]
    assert list(oracle.gen([0], [[4]], (1, 2, 3), 11)[:, 0]) == unit["f11_zero_4"]
    assert list(oracle.lagrange_weights((1, 2), 11)) == unit["f11_lagrange_12"]
    assert list(oracle.lagrange_weights((1, 2, 3), 11)) == unit["f11_lagrange_123"]
    assert oracle.reducing_matrix(2, 3, p=11) == unit["f11_R"]
    # reshare golden (2,6,7) -> (9,1,4) (T/test_protocol.py:63-72)
    r = np.array(unit["f11_R"], dtype=np.uint64)
    got = oracle.reduce_apply(np.array([[2], [6], [7]], dtype=np.uint64), r.T, 11)[:, 0]
    assert list(got) == [9, 1, 4]


def test_default_prime_constants(unit):
    assert unit["p"] == P
    for k, n in ((2, 3), (3, 5), (4, 7)):
        assert oracle.reducing_matrix(k, n) == unit[f"R_{k}{n}"]
        assert list(oracle.lagrange_weights(tuple(range(1, k + 1)))) == unit[f"lag_front_{k}{n}"]
        assert list(oracle.lagrange_weights(tuple(range(1, 2 * k)))) == unit[f"lag_part_{k}{n}"]
    for a, ia in unit["inv_samples"]:
        assert oracle.lib().ssn_o_inv(a, P) == ia
    assert oracle.mulmod(1 << 23, 1 << 23) == unit["split_anchor"] == 110


def test_round_half_away_and_bounds(unit):
    v = unit["round_half_away_in"]
    assert list(oracle.round_half_away(v, 4)) == unit["round_half_away_d4"]
    assert list(oracle.round_half_away(v, 3)) == unit["round_half_away_d3"]
    for st, vb, emax in unit["emax"]:
        assert sim.additive_mask_bound(P, st, vb) == emax
    for vb, bmax in unit["bmax"]:
        assert sim.multiplicative_mask_bound(P, vb) == bmax


def test_gen_rec_reduce_vectors(vec):
    for k, n in ((2, 3), (3, 5)):
        sh = oracle.gen(vec[f"gen_secret_{k}{n}"], list(vec[f"gen_coeffs_{k}{n}"]),
                        tuple(range(1, n + 1)))
        assert np.array_equal(sh, vec[f"gen_shares_{k}{n}"])
        m = 2 * k - 1
        w = oracle.lagrange_weights(tuple(range(1, m + 1)))
        assert np.array_equal(oracle.rec(vec[f"rec_in_{k}{n}"], w), vec[f"rec_out_{k}{n}"])
        R = np.array(oracle.reducing_matrix(k, n), dtype=np.uint64)
        assert np.array_equal(oracle.reduce_apply(vec[f"rec_in_{k}{n}"], R.T),
                              vec[f"reduce_out_{k}{n}"])


def test_trunc_and_nonlin_elite_vectors(vec):
    for k, n in ((2, 3), (3, 5)):
        wf = oracle.lagrange_weights(tuple(range(1, k + 1)))
        for (r, d) in ((1 << 12, 1), (1 << 12, 49), (8, 4)):
            tag = f"trunc_{k}{n}_{r}_{d}"
            vb, r_, d_ = (int(v) for v in vec[tag + "_vb"])
            t = oracle.trunc_elite(vec[tag + "_masked"], wf, vb, r_, d_)
            assert np.array_equal(t, vec[tag + "_t"])
        wp = oracle.lagrange_weights(tuple(range(1, 2 * k)))
        for pool, kind in ((None, None), ((2, 2), "max"), ((2, 2), "sum"), ((3, 3), "max")):
            tag = f"nonlin_{k}{n}_{kind}_{pool[0] if pool else 0}"
            plain = oracle.nonlin_elite(vec[tag + "_masked"], wp, True, kind, (3, 6, 6), pool)
            assert np.array_equal(plain.reshape(-1), vec[tag + "_plain"].reshape(-1))
            um = oracle.ewise("mul", plain, vec[tag + "_binv0"].reshape(plain.shape))
            assert np.array_equal(um.reshape(-1), vec[tag + "_unmask0"].reshape(-1))


def test_gemm_im2col_inv_vectors(vec):
    for (M, K, N) in ((7, 13, 5), (33, 200, 65), (64, 576, 49)):
        c = oracle.gemm(vec[f"gemm_{M}_{K}_{N}_A"], vec[f"gemm_{M}_{K}_{N}_B"])
        assert np.array_equal(c, vec[f"gemm_{M}_{K}_{N}_C"])
    assert np.array_equal(oracle.im2col(vec["im2col_x"], 3, 3, 2, 1), vec["im2col_s2p1"])
    got = [oracle.lib().ssn_o_inv(int(a), P) for a in vec["inv_in"]]
    assert got == [int(v) for v in vec["inv_out"]]


def test_lockstep_sim_matches_reference_runs(engine):
    """Decoded output, SimHub transcript digest and per-op element counts of the
    lockstep oracle equal the threaded reference run bit-for-bit."""
    cases, arr = engine
    for case in cases:
        mname = case["model"]
        weights = {key.split("/w/")[1]: arr[key] for key in arr.files
                   if key.startswith(mname + "/w/")}
        sch = sim.Scheme(case["k"], case["n"])
        res = sim.simulate(case["ops"], sch, case["seed"], arr[case["tag"] + "/x"], weights,
                           input_index=case["input_index"], record=True)
        assert np.array_equal(res["output"], arr[case["tag"] + "/out"]), case["tag"]
        assert res["transcript_digest"] == case["transcript_digest"], case["tag"]
        for row in case["summary"]:
            assert res["elements"][(row["op"], row["layer"])] == row["elements_sent"]
        plain, _ = sim.plaintext(case["ops"], arr[case["tag"] + "/x"], weights)
        assert np.array_equal(plain, arr[case["tag"] + "/out"])


def test_verify_mode_detects_corruption(engine):
    cases, arr = engine
    case = next(c for c in cases if c["model"] == "reference-max" and c["k"] == 3
                and c["ordering"] == "ltn")
    weights = {key.split("/w/")[1]: arr[key] for key in arr.files
               if key.startswith("reference-max/w/")}
    ops = [dict(op) for op in case["ops"]]
    for i, op in enumerate(ops[:-1]):           # verification needs passive inputs
        if op["kind"] == "linear" and ops[i + 1]["kind"] == "truncation":
            op["passive_out"] = True
    sch = sim.Scheme(3, 5)
    x = arr[case["tag"] + "/x"]
    ok = sim.simulate(ops, sch, case["seed"], x, weights, input_index=case["input_index"],
                      verify=True)
    assert ok["checks_failed"] == 0
    assert np.array_equal(ok["output"], arr[case["tag"] + "/out"])
    bad = sim.simulate(ops, sch, case["seed"], x, weights, input_index=case["input_index"],
                       verify=True, corrupt=(1, 5))
    assert bad["checks_failed"] == 1


@pytest.fixture(scope="module")
def residual():
    with open(os.path.join(GOLD, "residual.json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(GOLD, "residual.npz"))


def _tiny_resnet_weights():
    from paper_2406_02629_b200 import resnet     # host-side graph builder (no GPU needed)
    return resnet.tiny_resnet(seed=3).weight_values()


def test_oracle_sim_matches_reference_composed_residual_net(residual):
    """The reference's own sss_linear / sss_truncation / sss_nonlinear / share_add /
    output_collect composed over a residual DAG (tests/golden/make_golden.py
    residual_goldens) == the lockstep oracle: decoded outputs, every rank's share of every
    op output, and the SimHub transcript sha256."""
    meta, arr = residual
    weights = _tiny_resnet_weights()
    ops = meta["ops"]
    for case in meta["cases"]:
        tag = case["tag"]
        x = arr[tag + "/x"]
        res = sim.simulate(ops, sim.Scheme(case["k"], case["n"]), case["seed"], x, weights,
                           input_index=case["input_index"], record=True, return_shares=True)
        assert np.array_equal(res["output"], arr[tag + "/out"]), tag
        assert res["transcript_digest"] == case["transcript_digest"], tag
        for idx, ranks in case["held"].items():
            want = arr[f"{tag}/shares/{idx}"]
            vals = res["values"][int(idx)]
            assert sorted(vals) == ranks, (tag, idx)
            for row, r in enumerate(ranks):
                got = np.asarray(vals[r][1], dtype=np.uint64).reshape(-1)
                assert np.array_equal(got, want[row]), (tag, idx, r)


def test_oracle_sim_acceptance_100_inputs_two_schemes():
    """T/test_acceptance.py:155-176 (criterion 03) fixture: 100 inputs x {(2,3), (3,5)} --
    decoded outputs and transcript digests of the reference's runs."""
    with open(os.path.join(GOLD, "acceptance.json")) as fh:
        meta = json.load(fh)
    arr = np.load(os.path.join(GOLD, "acceptance.npz"))
    from paper_2406_02629_b200 import build_reference_model, layers, PrimeField, SssScheme
    model, _ = build_reference_model(7, pool="max")
    weights = {name: qt.values for name, qt in model.weights.items()}
    for k, n in ((2, 3), (3, 5)):
        ops, _ = layers.plan_schedule(model, SssScheme(PrimeField(), k, n))
        ops = [op.meta() for op in ops]
        for idx in range(100):
            rec = idx % 10 == 0                  # transcript digests on a tenth (CPU time)
            res = sim.simulate(ops, sim.Scheme(k, n), 7, arr["x"][idx], weights, input_index=idx, record=rec)
            assert np.array_equal(res["output"], arr[f"out_{k}{n}"][idx]), (k, n, idx)
            if rec:
                assert res["transcript_digest"] == meta["transcripts"][f"{k}{n}"][idx]
