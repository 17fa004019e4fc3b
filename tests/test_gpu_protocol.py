"""The reference's protocol-level known-answer tests, run through the DEVICE protocol (one thread
per rank over the DeviceHub, every step a kernel of libssn_b200.so):

  * reshare golden (2,6,7) -> (9,1,4) regardless of sub-share randomness, + rerand -> (2,9,..)
    (T/test_protocol.py:63-83,134-150; T/test_acceptance.py:112-129)
  * the truncation counterexample (0,6,1): naive 8, secure 2 (T/test_acceptance.py:132-152)
  * naive degree reduction leaks the secret and the audit scanner flags it; the honest reshare
    passes the audit (T/test_protocol.py:161-186)
  * element counts / rounds of reshare (T/test_protocol.py:86-105), distributed zero shares
    (T/test_protocol.py:189-208)
  * output collection decodes signed values (T/test_protocol.py:211-222)
"""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2406_02629_b200 as pkg
    pkg._lib.load()
    return pkg


def _run(P, scheme, fn, seed=0, audit=False, metrics=None):
    """fn(ctx) on every rank over the device hub (the reference's _run, T/test_protocol.py:28-53)."""
    import torch
    from paper_2406_02629_b200.protocol import AuditLog, PartyContext
    from paper_2406_02629_b200.transport import DeviceHub
    hub = DeviceHub(range(1, scheme.n + 1), metrics)
    results, errors, audits = {}, {}, []
    dev = torch.cuda.current_device()
    threads = []
    for rank in range(1, scheme.n + 1):
        log = AuditLog(rank) if audit else None
        if log is not None:
            audits.append(log)
        ctx = PartyContext(scheme, rank, hub.transport(rank), rng=np.random.default_rng([seed, rank]), audit=log)

        def worker(ctx=ctx):
            try:
                torch.cuda.set_device(dev)
                results[ctx.rank] = fn(ctx)
            except Exception as exc:  # noqa: BLE001 - re-raised below
                errors[ctx.rank] = exc

        threads.append(threading.Thread(target=worker))
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=60)
    if errors:
        raise errors[sorted(errors)[0]]
    return results, audits


def _product(P, s, values):
    return {r: P.ShareTensor(s.party_ids[r - 1], 2 * (s.k - 1), np.array([values[r - 1]], dtype=np.int64), s)
            for r in range(1, s.n + 1)}


def _v(st):
    return int(st.values.reshape(-1)[0].item())


def test_reshare_golden_then_rerand(P):
    from paper_2406_02629_b200.protocol import reshare_degree_reduce, rerand
    s = P.SssScheme(P.PrimeField(11), 2, 3)
    pre = _product(P, s, (2, 6, 7))
    for seed in (5, 6, 99):                       # values do not depend on the sub-share randomness
        res, _ = _run(P, s, lambda ctx: reshare_degree_reduce(ctx, pre[ctx.rank], passive_out=True), seed=seed)
        assert [_v(res[r]) for r in (1, 2, 3)] == [9, 1, 4]
        assert all(res[r].degree == 1 for r in (1, 2, 3))
        assert int(s.rec([res[1], res[2]]).reshape(-1)[0].item()) == 6
    zeros = s.gen(np.array([0]), coeffs=[np.array([4])])
    post = {r: rerand(res[r], zeros[r - 1]) for r in (1, 2, 3)}
    assert [_v(post[r]) for r in (1, 2)] == [2, 9]
    assert post[1].degree == 1
    assert int(s.rec([post[1], post[2]]).reshape(-1)[0].item()) == 6
    # without passive output rank 3 gets nothing
    res, _ = _run(P, s, lambda ctx: reshare_degree_reduce(ctx, pre[ctx.rank], passive_out=False), seed=6)
    assert (_v(res[1]), _v(res[2]), res[3]) == (9, 1, None)


def test_truncation_counterexample(P):
    """Shares (0,6,1) of 5 in F_11: share-wise halving reconstructs 8, the secure masked
    truncation gives floor(5/2) = 2 (T/test_acceptance.py:132-152)."""
    from paper_2406_02629_b200.layers import ScheduledOp, sss_truncation
    from paper_2406_02629_b200.masks import gen_additive_mask
    F11 = P.PrimeField(11)
    s = P.SssScheme(F11, 2, 3)
    shares = [P.ShareTensor(i + 1, 1, np.array([v], dtype=np.int64), s) for i, v in enumerate((0, 6, 1))]
    assert int(s.rec(shares[:2]).reshape(-1)[0].item()) == 5
    naive = [P.ShareTensor(st.party_id, 1, np.array([_v(st) // 2], dtype=np.int64), s) for st in shares]
    assert int(s.rec(naive[:2]).reshape(-1)[0].item()) == 8
    op = ScheduledOp("truncation", 0, "div", (1,), (1,), r=2, value_bound=5)
    alpha, comp, _ = gen_additive_mask((1,), 2, 1, s, np.random.default_rng(7), 5)
    res, logs = _run(P, s, lambda ctx: sss_truncation(ctx, op, shares[ctx.rank - 1], alpha[ctx.rank - 1],
                                                      comp[ctx.rank - 1]), seed=5, audit=True)
    secure = int(s.rec([res[1], res[2]]).reshape(-1)[0].item())
    assert secure == 2
    from paper_2406_02629_b200.protocol import audit_violations
    assert audit_violations(logs, s.k) == []


def test_naive_reduction_leaks_and_audit_flags_it(P):
    from paper_2406_02629_b200.protocol import audit_violations, naive_degree_reduce, reshare_degree_reduce
    s = P.SssScheme(P.PrimeField(11), 2, 3)
    rng = np.random.default_rng(9)
    xs = s.gen(np.array([2]), rng)
    ys = s.gen(np.array([3]), rng)
    prod = {r: P.share_mul(xs[r - 1], ys[r - 1]) for r in (1, 2, 3)}
    res, audits = _run(P, s, lambda ctx: naive_degree_reduce(ctx, prod[ctx.rank]), seed=4, audit=True)
    reduced_1, leak = res[1]
    assert int(s.rec([reduced_1, res[2][0]]).reshape(-1)[0].item()) == 6
    assert int(leak["secret"].reshape(-1)[0].item()) == 6
    assert len(leak["foreign_shares"]) == 2
    problems = audit_violations(audits, s.k)
    assert any("rank 1" in p and "raw shares" in p for p in problems)
    assert any("unmasked reconstruction" in p for p in problems)
    # the honest protocol on the same products passes
    _, audits = _run(P, s, lambda ctx: reshare_degree_reduce(ctx, prod[ctx.rank], passive_out=True), seed=5,
                     audit=True)
    assert audit_violations(audits, s.k) == []


@pytest.mark.parametrize("kn,passive,per_elem", [((2, 3), False, 6), ((2, 3), True, 8), ((3, 5), False, 18),
                                                 ((3, 5), True, 24)])
def test_reshare_counts_and_rounds(P, kn, passive, per_elem):
    from paper_2406_02629_b200.metrics import CommMetrics
    from paper_2406_02629_b200.protocol import reshare_degree_reduce
    F = P.PrimeField()
    k, n = kn
    s = P.SssScheme(F, k, n)
    rng = np.random.default_rng(17)
    a = s.gen(rng.integers(0, F.p, size=5, dtype=np.int64), rng)
    b = s.gen(rng.integers(0, F.p, size=5, dtype=np.int64), rng)
    prod = {r: P.share_mul(a[r - 1], b[r - 1]) for r in range(1, n + 1)}
    metrics = CommMetrics()

    def fn(ctx):
        metrics.set_op(ctx.rank, "red", 0)
        return reshare_degree_reduce(ctx, prod[ctx.rank], passive_out=passive)

    res, _ = _run(P, s, fn, seed=k, metrics=metrics)
    assert metrics.elements_sent("red", 0) == per_elem * 5
    assert metrics.rounds("red", 0) == 2
    got = s.rec([res[r] for r in range(1, k + 1)]).cpu().numpy().astype(object)
    pa = s.rec(a[:k]).cpu().numpy().astype(object)
    pb = s.rec(b[:k]).cpu().numpy().astype(object)
    assert np.array_equal(got, (pa * pb) % F.p)


def test_distributed_zero_shares_on_device(P):
    from paper_2406_02629_b200.metrics import CommMetrics
    from paper_2406_02629_b200.protocol import distributed_zero_shares
    s = P.SssScheme(P.PrimeField(), 2, 3)
    metrics = CommMetrics()
    res, _ = _run(P, s, lambda ctx: distributed_zero_shares(ctx, (4,), metrics=metrics), seed=13, metrics=metrics)
    assert all(st.degree == 1 for st in res.values())
    assert np.all(s.rec([res[1], res[2]]).cpu().numpy() == 0)
    assert metrics.elements_sent("zero_dist") == 3 * 2 * 4
    assert [r["elements_sent"] for r in metrics.records() if r["op"] == "zero_dist"] == [8, 8, 8]


def test_output_collect_decodes_signed(P):
    from paper_2406_02629_b200.protocol import output_collect
    F = P.PrimeField()
    s = P.SssScheme(F, 2, 3)
    rng = np.random.default_rng(31)
    secret = np.array([-5, 0, 7], dtype=np.int64)
    shares = s.gen(F.encode_signed(secret), rng)
    res, _ = _run(P, s, lambda ctx: output_collect(ctx, shares[ctx.rank - 1]), seed=1)
    assert list(np.asarray(res[1]).reshape(-1)) == [-5, 0, 7]
    assert res[2] is None and res[3] is None
