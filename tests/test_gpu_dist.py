"""Party-per-process secure inference (dist.run_party_dist): n party processes + the trusted
source, one torch.distributed rank each, on the box's GPU (gloo backend, host-staged, since a
single GPU cannot host several NCCL ranks).  Shares, masks and every message are bit-identical
to the reference run: decoded outputs equal the lockstep oracle and the canonical transcript
digest (S/transport.py:68-80) of all ranks' frames equals the oracle's."""

import datetime
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _party(rank, world, port, k, n, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=90))
    try:
        import paper_2406_02629_b200 as P
        from paper_2406_02629_b200.dist import run_party_dist
        model, _ = P.build_reference_model(7, pool="max")
        scheme = P.SssScheme(P.PrimeField(), k, n)
        x, _ = P.random_input(7, model, index=0)
        out, metrics, frames = run_party_dist(model, scheme, 7, x, "cuda:0", record=True)
        t = metrics._tally(rank)
        q.put((rank, out, frames, t.elements_sent))
    except BaseException as exc:             # surface worker failures instead of hanging
        q.put((rank, "error", repr(exc), 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
def test_party_per_process_matches_reference(k, n):
    from oracle import sim
    import paper_2406_02629_b200 as P
    from paper_2406_02629_b200.dist import transcript_digest
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = n + 1
    procs = [ctx.Process(target=_party, args=(r, world, port, k, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, frames, sent = q.get(timeout=180)
        assert not (isinstance(out, str) and out == "error"), f"rank {rank}: {frames}"
        res[rank] = (out, frames, sent)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    model, _ = P.build_reference_model(7, pool="max")
    weights = {name: qt.values for name, qt in model.weights.items()}
    scheme = P.SssScheme(P.PrimeField(), k, n)
    x, _ = P.random_input(7, model, index=0)
    ops, _ = P.plan_schedule(model, scheme)
    want = sim.simulate([op.meta() for op in ops], sim.Scheme(k, n), 7, x, weights, record=True)
    assert np.array_equal(res[1][0], want["output"])
    assert transcript_digest([res[r][1] for r in range(world)]) == want["transcript_digest"]
