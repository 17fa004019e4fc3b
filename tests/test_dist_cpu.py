"""Party-per-process transport (paper_2406_02629_b200/dist.py) on CPU with the gloo backend,
world_size 2 and 3: addressed FIFO delivery, phase checks (ScheduleDivergence, like
S/transport.py:98-109), the reference's element / frame-byte accounting (S/metrics.py:46-60,
S/wire.py:104-107) and the recorded canonical frames.  No kernels run here."""

import datetime
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=90))
    from paper_2406_02629_b200.dist import DistTransport
    from paper_2406_02629_b200.metrics import CommMetrics
    from paper_2406_02629_b200.transport import ScheduleDivergence
    from paper_2406_02629_b200.wire import Phase, share_frame_bytes, plain_frame_bytes
    m = CommMetrics()
    m.set_op(rank, "t", 0)
    tr = DistTransport(rank, "cpu", m, record=True)
    res = {}
    try:
        if rank == 0:
            x = torch.arange(12, dtype=torch.int64).reshape(3, 4)
            for dst in range(1, world):
                tr.send_share(dst, Phase.RESHARE_OUT, 1, 2, x * dst)
                tr.send_plain(dst, Phase.NONLIN_PLAIN, torch.tensor([5, 6, 7]))
                tr.send_object(dst, Phase.MASK_DIST, None, 40, 3, encode=lambda: b"bundle-bytes")
            # second share with a phase the receiver does not expect
            tr.send_share(1, Phase.TRUNC_MASKED, 1, 1, torch.zeros(2, dtype=torch.int64))
            t = m._tally(0)
            res["sent"] = (t.elements_sent, t.bytes_sent)
            res["frames"] = {k: len(v) for k, v in tr.frames.items()}
        else:
            a = tr.recv(0, Phase.RESHARE_OUT, elements=12)
            res["share"] = (a.meta, a.tensor.tolist())
            b = tr.recv(0, Phase.NONLIN_PLAIN, elements=3)
            res["plain"] = b.tensor.tolist()
            c = tr.recv(0, Phase.MASK_DIST, elements=3)
            res["object"] = c.tensor
            if rank == 1:
                try:
                    tr.recv(0, Phase.SHARE_DIST)
                    res["divergence"] = False
                except ScheduleDivergence:
                    res["divergence"] = True
            t = m._tally(rank)
            res["recv"] = (t.elements_received, t.bytes_received)
        tr.close()                            # complete the in-flight isends
        res["frame_sizes"] = (share_frame_bytes((3, 4)), plain_frame_bytes((3,)))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_transport_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=60) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    share_b, plain_b = out[0]["frame_sizes"]
    assert share_b == 12 + 11 + 8 + 96 and plain_b == 12 + 1 + 4 + 24
    for r in range(1, world):
        meta, vals = out[r]["share"]
        assert meta == (1, 2)
        assert vals == (torch.arange(12).reshape(3, 4) * r).tolist()
        assert out[r]["plain"] == [5, 6, 7]
        assert out[r]["object"] == b"bundle-bytes"
        assert out[r]["recv"] == (12 + 3 + 3, share_b + plain_b + 40)
    assert out[1]["divergence"] is True
    # elements: 12 + 3 + 3 per peer, + 2 for the divergent share
    assert out[0]["sent"][0] == (world - 1) * 18 + 2
    assert out[0]["frames"][(0, 1)] == 4


class _HopStub:
    """The plumbing PartyShardedEngine._exchange needs (host-staged gloo, group base 0)."""
    nccl = False
    base = 0

    def _g(self, role):
        return self.base + role


def _hop_worker(rank, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2, timeout=datetime.timedelta(seconds=90))
    from paper_2406_02629_b200.sharded import PartyShardedEngine
    try:
        other = 1 - rank
        # reshare step 1's pattern: BOTH ranks send a large buffer to the other before either
        # receives -- one grouped hop must complete without deadlock and keep per-peer order
        big = [torch.arange(1 << 20, dtype=torch.int64) * (rank + 1) + i for i in range(3)]
        outs = [torch.empty(1 << 20, dtype=torch.int64) for _ in range(3)]
        PartyShardedEngine._exchange(_HopStub(), [(other, t) for t in big], [(other, o) for o in outs])
        ok = all(torch.equal(outs[i], torch.arange(1 << 20, dtype=torch.int64) * (other + 1) + i) for i in range(3))
        # a hop with only sends on one side and only receives on the other (SHARE_DIST shape)
        buf = torch.empty(7, dtype=torch.int64)
        if rank == 0:
            PartyShardedEngine._exchange(_HopStub(), [(1, torch.full((7,), 42, dtype=torch.int64))], [])
        else:
            PartyShardedEngine._exchange(_HopStub(), [], [(0, buf)])
            ok = ok and buf.tolist() == [42] * 7
        q.put((rank, ok))
    except BaseException as exc:
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


def test_grouped_hop_exchange_gloo_world2():
    """PartyShardedEngine._exchange (one batch_isend_irecv per protocol hop) on CPU gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hop_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(60)
    assert res == {0: True, 1: True}, res
