"""Party-per-process share exchange over torch.distributed -- the multi-GPU counterpart of
the reference's TcpTransport (S/transport.py:146-263) and run-party/run-source drivers
(S/engine.py:215-246).

One process per protocol rank (0 = trusted source, 1..n = parties), one GPU each.  The
transport implements the same duck-typed seam as DeviceTransport / the reference
(`send_share`, `send_plain`, `send_object`, `recv(src, phase, elements)`, `close`): addressed,
FIFO per (src, dst) channel, phase-checked (ScheduleDivergence on mismatch), with
CommMetrics fed the reference's element and frame-byte counts.

Backends: the seam is one blocking, addressed message at a time, and a party sends to several
peers before it receives (reshare step 1: fronts 1 and 2 each send to the other first).  NCCL
pairs a send and a recv between two peers on one stream, so two large ungrouped sends facing
each other wait on each other forever.  This transport therefore always moves its messages over
a gloo group (host-staged); under an NCCL default group run_party_dist creates that gloo group
for it.  The NVLink throughput path is PartyShardedEngine (sharded.py), which issues every
protocol hop as ONE grouped batch_isend_irecv (ncclGroupStart/ncclSend/ncclRecv/ncclGroupEnd).
Every message is a fixed 16-word int64 header followed by the payload (u64 share/plaintext
values, or the u8 bytes of a serialized MaskBundle).
"""

import json
import struct

import numpy as np
import torch
import torch.distributed as dist

from .metrics import CommMetrics
from .transport import Message, PartyTimeout, ScheduleDivergence
from .wire import Phase, ProtocolError, encode_frame, encode_plain_payload, encode_share_payload, \
    plain_frame_bytes, share_frame_bytes

HDR_WORDS = 16
MAGIC = 0x53534E31            # "SSN1"
KIND_SHARE, KIND_PLAIN, KIND_OBJECT = 0, 1, 2
MAX_NDIM = 6


def _header(sender, phase, kind, party_id, degree, nbytes, shape, numel):
    if len(shape) > MAX_NDIM:
        raise ValueError(f"tensor rank {len(shape)} > {MAX_NDIM}")
    h = [MAGIC, sender, int(phase), kind, party_id, degree, nbytes, len(shape)]
    h += list(shape) + [0] * (MAX_NDIM - len(shape))
    h += [numel, 0]
    return h[:HDR_WORDS]


class DistTransport:
    """Transport for rank `rank` of a torch.distributed world whose ranks ARE the protocol
    ranks.  `device` is where received tensors land (a CUDA device for the product path)."""

    def __init__(self, rank, device, metrics=None, record=False, decode_object=None, group=None):
        self.rank = rank
        self.device = torch.device(device)
        self.metrics = metrics
        self.group = group
        self.backend = dist.get_backend(group)
        if self.backend == "nccl":
            raise ValueError("DistTransport needs a gloo group: ungrouped NCCL sends between two parties that "
                             "both send first deadlock (pass group=dist.new_group(backend='gloo'); the NCCL "
                             "path is PartyShardedEngine)")
        self.record = record
        self.frames = {}             # (src, dst) -> [frame bytes]  (sent frames, when recording)
        self.decode_object = decode_object
        self._pending = []           # in-flight isend works (+ their tensors, kept alive)

    # -- wire helpers
    def _comm_device(self):
        return torch.device("cpu")

    def _send_tensor(self, t, dst):
        # Non-blocking: every party sends to several peers before it receives (e.g. reshare
        # step 1), so a blocking send would deadlock two parties sending to each other.
        # Per-(src, dst) FIFO order is preserved by the backend.
        t = t.contiguous()
        if t.device.type != "cpu":
            t = t.cpu()
        self._pending.append((dist.isend(t, dst, group=self.group), t))
        if len(self._pending) > 64:
            self._reap()

    def _reap(self):
        self._pending = [(w, t) for (w, t) in self._pending if not w.is_completed()]

    def flush(self):
        for w, _ in self._pending:
            w.wait()
        self._pending = []

    def _recv_tensor(self, shape, dtype, src):
        t = torch.empty(shape, dtype=dtype, device=self._comm_device())
        dist.recv(t, src, group=self.group)
        return t

    def _send(self, dst, hdr, payload, elements, nbytes, frame=None):
        self._send_tensor(torch.tensor(hdr, dtype=torch.int64, device=self._comm_device()), dst)
        self._send_tensor(payload, dst)
        if self.metrics is not None:
            self.metrics.on_send(self.rank, nbytes, elements)
        if self.record and frame is not None:
            self.frames.setdefault((self.rank, dst), []).append(frame())

    # -- the reference seam (S/protocol.py:111-128)
    def send_share(self, dst, phase, party_id, degree, tensor, elements=None):
        n = tensor.numel() if elements is None else elements
        shape = tuple(tensor.shape)
        nbytes = share_frame_bytes(shape)
        hdr = _header(self.rank, phase, KIND_SHARE, party_id, degree, nbytes, shape, tensor.numel())
        frame = (lambda: encode_frame(self.rank, phase, encode_share_payload(
            party_id, degree, tensor.detach().cpu().numpy().astype(np.uint64))))
        self._send(dst, hdr, tensor.to(torch.int64).reshape(-1), n, nbytes, frame)

    def send_plain(self, dst, phase, tensor, elements=None):
        n = tensor.numel() if elements is None else elements
        shape = tuple(tensor.shape)
        nbytes = plain_frame_bytes(shape)
        hdr = _header(self.rank, phase, KIND_PLAIN, 0, 0, nbytes, shape, tensor.numel())
        frame = (lambda: encode_frame(self.rank, phase, encode_plain_payload(
            tensor.detach().cpu().numpy().astype(np.uint64))))
        self._send(dst, hdr, tensor.to(torch.int64).reshape(-1), n, nbytes, frame)

    def send_object(self, dst, phase, obj, nbytes, elements, encode=None):
        if encode is None:
            raise ValueError("send_object over torch.distributed needs an encoder")
        blob = encode()
        payload = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
        hdr = _header(self.rank, phase, KIND_OBJECT, 0, 0, nbytes, (len(blob),), len(blob))
        self._send(dst, hdr, payload.to(self._comm_device()), elements, nbytes,
                   (lambda: encode_frame(self.rank, phase, blob)))

    def recv(self, src, phase, elements=0):
        hdr = self._recv_tensor((HDR_WORDS,), torch.int64, src).cpu().tolist()
        if hdr[0] != MAGIC:
            raise ProtocolError(f"bad frame magic from {src}")
        sender, got_phase, kind, party_id, degree, nbytes, ndim = hdr[1:8]
        shape = tuple(hdr[8:8 + ndim])
        numel = hdr[8 + MAX_NDIM]
        if sender != src:
            raise ProtocolError(f"frame from {sender} on channel of {src}")
        if kind == KIND_OBJECT:
            blob = self._recv_tensor((numel,), torch.uint8, src).cpu().numpy().tobytes()
            obj = self.decode_object(blob) if self.decode_object is not None else blob
            msg = Message(sender, Phase(got_phase), "object", None, obj, nbytes)
        else:
            vals = self._recv_tensor((numel,), torch.int64, src).to(self.device).reshape(shape)
            msg = Message(sender, Phase(got_phase), "share" if kind == KIND_SHARE else "plain",
                          (party_id, degree) if kind == KIND_SHARE else None, vals, nbytes)
        if got_phase != int(phase):
            raise ScheduleDivergence(
                f"party {self.rank} expected {Phase(phase).name} from {src}, got {Phase(got_phase).name}")
        if self.metrics is not None:
            self.metrics.on_recv(self.rank, nbytes, elements)
        return msg

    def close(self):
        self.flush()


def mask_bundle_decoder(scheme, device):
    """MASK_DIST payload -> MaskBundle on `device` (MaskBundle.decode, S/protocol.py:337-351)."""
    from .protocol import MaskBundle
    return lambda blob: MaskBundle.decode(blob, scheme, device)


def transcript_digest(frames_by_rank):
    """Canonical transcript sha256 (S/transport.py:68-80) from every rank's sent frames
    (list indexed by rank).  Every ordered channel (src != dst) appears, empty ones too."""
    import hashlib
    world = len(frames_by_rank)
    merged = {(s, d): [] for s in range(world) for d in range(world) if s != d}
    for frames in frames_by_rank:
        merged.update(frames)
    parts = []
    for key in sorted(merged):
        parts.append(struct.pack("<HHI", key[0], key[1], len(merged[key])))
        parts.extend(merged[key])
    return hashlib.sha256(b"".join(parts)).hexdigest()


def run_party_dist(model, scheme, seed, input_int, device, ordering="ltn", rng_mode="host", verify=False,
                   record=False, metrics=None):
    """This process's rank of one secure inference (rank 0: trusted source, 1..n: parties)
    -- the reference's run-source / run-party (S/engine.py:215-246) over torch.distributed.
    Every rank must call it.  Returns (decoded output or None, metrics, sent frames)."""
    from .engine import (PURPOSE_PARTY, deal_input_shares, deal_weight_shares, lane_rng, receive_bundle,
                         run_party_online, send_bundles)
    from .layers import plan_schedule
    from .protocol import AuditLog, PartyContext  # noqa: F401
    rank = dist.get_rank()
    if dist.get_world_size() != scheme.n + 1:
        raise ValueError(f"world size {dist.get_world_size()} != n + 1 = {scheme.n + 1}")
    metrics = metrics if metrics is not None else CommMetrics()
    ops, _ = plan_schedule(model, scheme, ordering, verify=verify)
    group = dist.new_group(backend="gloo") if dist.get_backend() == "nccl" else None   # collective
    tr = DistTransport(rank, device, metrics, record=record, decode_object=mask_bundle_decoder(scheme, device),
                       group=group)
    if rank == 0:
        send_bundles(tr, ops, scheme, seed, metrics, rng_mode)
        tr.close()
        return None, metrics, tr.frames
    # model owner / input owner dealing, replayed from the seed (S/engine.py:40-54)
    weight_values = {name: qt.values for name, qt in model.weights.items()}
    w_share = deal_weight_shares(weight_values, scheme, seed, rng_mode)[rank]
    x_share = deal_input_shares(input_int, scheme, seed, 0, rng_mode)[rank - 1]
    ctx = PartyContext(scheme, rank, tr, rng=lane_rng(rng_mode, seed, PURPOSE_PARTY, rank), verify=verify)
    metrics.set_op(rank, "offline", -1)
    receive_bundle(ctx)
    out = run_party_online(ctx, ops, w_share, x_share, metrics)
    tr.close()
    if out is not None:
        out = np.asarray(out, dtype=np.int64)
    return out, metrics, tr.frames
