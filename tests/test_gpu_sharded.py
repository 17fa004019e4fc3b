"""Party-per-GPU batched engine (sharded.PartyShardedEngine): the trusted source and the n
parties as separate torch.distributed ranks (gloo, all on the box's single GPU -- NCCL needs
one GPU per rank).  Every protocol hop crosses a process boundary; decoded outputs must equal
the exact integer plaintext of the residual network."""

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


def _rank(rank, world, port, k, n, verify, q, rotate=True, backend="gloo"):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0 if backend == "gloo" else rank)
    kw = {} if backend == "gloo" else {"device_id": torch.device("cuda", rank)}
    dist.init_process_group(backend, rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120), **kw)
    try:
        import paper_2406_02629_b200 as P
        from paper_2406_02629_b200 import resnet
        from paper_2406_02629_b200.sharded import PartyShardedEngine
        net = resnet.tiny_resnet(seed=3)
        eng = PartyShardedEngine(net, P.SssScheme(P.PrimeField(), k, n), batch=2, seed=11, verify=verify,
                                 rotate_elite=rotate)
        dist.barrier()
        xb = net.random_inputs(seed=5, batch=2)
        outs = [eng.run(xb) for _ in range(2)]          # second run: fresh randomness
        q.put((rank, outs))
    except BaseException as exc:
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


def _run(k, n, verify, rotate, backend):
    from paper_2406_02629_b200 import resnet
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = n + 1
    procs = [ctx.Process(target=_rank, args=(r, world, port, k, n, verify, q, rotate, backend)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, outs = q.get(timeout=240)
        assert not isinstance(outs, str), f"rank {rank}: {outs}"
        res[rank] = outs
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    net = resnet.tiny_resnet(seed=3)
    xb = net.random_inputs(seed=5, batch=2)
    want, _ = resnet.plaintext_forward(net, xb)
    for out in res[1]:
        assert np.array_equal(out, want)
    assert all(o is None for r in range(world) if r != 1 for o in res[r])


@pytest.mark.parametrize("k,n,verify,rotate", [(2, 3, False, True), (3, 5, True, True), (3, 5, True, False)])
def test_party_sharded_matches_plaintext(k, n, verify, rotate):
    """gloo, every rank on cuda:0; rotate: the elite moves over the front ranks op by op."""
    _run(k, n, verify, rotate, "gloo")


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
def test_party_sharded_nccl_one_gpu_per_rank(k, n):
    """The NVLink deployment path: one GPU per protocol rank, every hop one grouped NCCL
    send/recv.  Needs n+1 GPUs (skipped on the single-GPU test box)."""
    import torch
    if torch.cuda.device_count() < n + 1:
        pytest.skip(f"needs {n + 1} GPUs, have {torch.cuda.device_count()}")
    _run(k, n, True, True, "nccl")
