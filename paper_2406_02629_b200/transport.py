"""Share exchange between parties -- the B200 counterpart of S/transport.py.

Same seam as the reference (S/protocol.py:111-128): addressed, FIFO, phase-checked
point-to-point channels; CommMetrics sees the reference's element and frame-byte counts.
Payloads are device tensors instead of bytes:

* DeviceHub / DeviceTransport: all parties co-resident on one GPU; a send hands the
  receiver the producer's HBM buffer (the send buffer IS the receive buffer).  Ordering is
  stream order: every party enqueues on the same CUDA stream.
* DistTransport (dist.py): one party per process over torch.distributed (the API path), and
  the grouped NCCL hops of PartyShardedEngine (sharded.py, the NVLink throughput path).
* TcpTransport (tcp.py): cross-host parties over the reference's own TCP wire protocol.

A DeviceHub created with record=True serializes every message into the reference frame
format so the canonical transcript (S/transport.py:68-80) can be compared byte for byte.
"""

import hashlib
import queue
import struct
import threading

import numpy as np

from .wire import (Phase, ProtocolError, encode_frame, encode_plain_payload, encode_share_payload,
                   plain_frame_bytes, share_frame_bytes)


class PartyTimeout(ProtocolError):
    pass


class ScheduleDivergence(ProtocolError):
    pass


class HandshakeError(Exception):
    """Configuration disagreement between peers (version, scheme, digests)."""


class Message:
    """kind: 'share' (meta = (party_id, degree)), 'plain', or 'object' (opaque host object
    with an explicit reference frame length)."""
    __slots__ = ("sender", "phase", "kind", "meta", "tensor", "nbytes")

    def __init__(self, sender, phase, kind, meta, tensor, nbytes):
        self.sender, self.phase, self.kind = sender, phase, kind
        self.meta, self.tensor, self.nbytes = meta, tensor, nbytes


def _u64_host(t):
    return t.detach().cpu().numpy().astype(np.uint64)


class DeviceHub:
    def __init__(self, ranks, metrics=None, record=False, timeout=120.0):
        self.ranks = tuple(ranks)
        self.metrics = metrics
        self.record = record
        self.timeout = timeout
        self._queues = {(s, d): queue.SimpleQueue() for s in self.ranks for d in self.ranks if s != d}
        self._transcript = {key: [] for key in self._queues}
        self._lock = threading.Lock()

    def transport(self, rank):
        return DeviceTransport(self, rank)

    def _push(self, src, dst, msg):
        if self.record:
            frame = self._frame(msg)
            with self._lock:
                self._transcript[(src, dst)].append(frame)
        self._queues[(src, dst)].put(msg)

    @staticmethod
    def _frame(msg):
        if msg.kind == "share":
            payload = encode_share_payload(msg.meta[0], msg.meta[1], _u64_host(msg.tensor))
        elif msg.kind == "plain":
            payload = encode_plain_payload(_u64_host(msg.tensor))
        else:
            payload = msg.meta["encode"]()
        return encode_frame(msg.sender, msg.phase, payload)

    def canonical_transcript(self) -> bytes:
        parts = []
        with self._lock:
            for key in sorted(self._transcript):
                frames = self._transcript[key]
                parts.append(struct.pack("<HHI", key[0], key[1], len(frames)))
                parts.extend(frames)
        return b"".join(parts)

    def transcript_digest(self) -> str:
        return hashlib.sha256(self.canonical_transcript()).hexdigest()

    def channel_frames(self, src, dst):
        with self._lock:
            return list(self._transcript[(src, dst)])


class DeviceTransport:
    def __init__(self, hub, rank):
        self.hub = hub
        self.rank = rank

    def _send(self, dst, msg, elements):
        self.hub._push(self.rank, dst, msg)
        if self.hub.metrics is not None:
            self.hub.metrics.on_send(self.rank, msg.nbytes, elements)

    def send_share(self, dst, phase, party_id, degree, tensor, elements=None):
        n = tensor.numel() if elements is None else elements
        self._send(dst, Message(self.rank, Phase(phase), "share", (party_id, degree), tensor,
                                share_frame_bytes(tuple(tensor.shape))), n)

    def send_plain(self, dst, phase, tensor, elements=None):
        n = tensor.numel() if elements is None else elements
        self._send(dst, Message(self.rank, Phase(phase), "plain", None, tensor,
                                plain_frame_bytes(tuple(tensor.shape))), n)

    def send_object(self, dst, phase, obj, nbytes, elements, encode=None):
        self._send(dst, Message(self.rank, Phase(phase), "object", {"encode": encode}, obj, nbytes),
                   elements)

    def recv(self, src, phase, elements=0):
        try:
            msg = self.hub._queues[(src, self.rank)].get(timeout=self.hub.timeout)
        except queue.Empty:
            raise PartyTimeout(f"party {self.rank} timed out waiting for {src}") from None
        if msg.sender != src:
            raise ProtocolError(f"frame from {msg.sender} on channel of {src}")
        if msg.phase != phase:
            raise ScheduleDivergence(
                f"party {self.rank} expected {Phase(phase).name} from {src}, got {msg.phase.name}")
        if self.hub.metrics is not None:
            self.hub.metrics.on_recv(self.rank, msg.nbytes, elements)
        return msg

    def close(self):
        pass
