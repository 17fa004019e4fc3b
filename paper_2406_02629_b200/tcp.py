"""Cross-host parties: a TCP mesh that speaks the reference's wire protocol
(S/transport.py:146-263, S/wire.py) so a party running on a B200 can join a deployment whose
other parties run the reference (or this package on other hosts).

Same duck-typed seam as DeviceTransport / DistTransport (send_share, send_plain, send_object,
recv -> Message, close): addressed, FIFO per (src, dst) channel, phase-checked
(ScheduleDivergence), CommMetrics fed the reference's element and frame-byte counts.  A share
tensor leaves the GPU as ONE device->host copy of its u64 buffer into the frame, and arrives
as one host->device copy of the received payload -- no per-element packing.

Mesh set-up follows the reference: party `rank` (1..n) dials every lower rank, then accepts
every higher rank and, when told to expect it, the trusted source (rank 0), which dials all
parties.  Every connection opens with a HELLO frame (protocol version, k, n, sender, model and
schedule sha256); any disagreement raises HandshakeError before a share moves.
"""

import queue
import socket
import threading
import time

import numpy as np
import torch

from .transport import HandshakeError, Message, PartyTimeout, ScheduleDivergence
from .wire import (FRAME_HEADER_SIZE, PROTOCOL_VERSION, Phase, ProtocolError, decode_hello, decode_plain_payload,
                   decode_share_payload, digest32, encode_frame, encode_hello, encode_plain_payload,
                   encode_share_payload, frame_header, plain_frame_bytes, share_frame_bytes)


def _recv_exact(sock, n):
    buf = bytearray(n)
    view = memoryview(buf)
    got = 0
    while got < n:
        try:
            r = sock.recv_into(view[got:], n - got)
        except socket.timeout:
            raise PartyTimeout("timed out waiting for a frame") from None
        if r == 0:
            raise ProtocolError("connection closed mid-frame")
        got += r
    return buf


def read_frame(sock):
    """One frame from a socket -> (sender, Phase, payload bytearray)."""
    sender, phase, plen = frame_header(_recv_exact(sock, FRAME_HEADER_SIZE))
    return sender, phase, _recv_exact(sock, plen)


def _host_u64(t):
    """A device (or host) int64 tensor as a contiguous uint64 numpy array (one D2H copy)."""
    return t.detach().contiguous().cpu().numpy().view(np.uint64)


class _Writer:
    """Per-connection sender thread: the protocol often sends to a peer that is itself still
    sending (reshare step 1), so a blocking sendall of a multi-MB frame on the protocol thread
    could wait forever on a full socket buffer.  Frames are queued FIFO and written here."""

    def __init__(self, sock):
        self.sock = sock
        self.q = queue.SimpleQueue()
        self.error = None
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        while True:
            frame = self.q.get()
            if frame is None:
                return
            try:
                self.sock.sendall(frame)
            except OSError as exc:
                self.error = exc
                return

    def put(self, frame):
        if self.error is not None:
            raise ProtocolError(f"send failed: {self.error!r}")
        self.q.put(frame)

    def flush(self, timeout):
        self.q.put(None)
        self.thread.join(timeout)
        if self.error is not None:
            raise ProtocolError(f"send failed: {self.error!r}")


class TcpTransport:
    """One party's end of a fully connected TCP mesh.  Received tensors land on `device`."""

    def __init__(self, rank, socks, device="cpu", p=None, metrics=None, decode_object=None, timeout=30.0):
        self.rank = rank
        self._socks = socks
        self._writers = {peer: _Writer(sock) for peer, sock in socks.items()}
        self.device = torch.device(device)
        self.p = p
        self.metrics = metrics
        self.decode_object = decode_object
        self.timeout = timeout

    @classmethod
    def establish(cls, rank, peers, k, n, model_digest, schedule_digest, device="cpu", p=None, metrics=None,
                  expect_source=False, timeout=30.0, dial_deadline=15.0, decode_object=None):
        """Wire up the mesh for party `rank` (1..n) or the source (0).  peers: (host, port) of
        ranks 1..n (S/transport.py:154-236)."""
        mdig, sdig = digest32(model_digest), digest32(schedule_digest)
        hello = encode_frame(rank, Phase.HELLO, encode_hello(k, n, rank, mdig, sdig))

        def check(payload, expect=None):
            version, hk, hn, sender, pm, ps = decode_hello(bytes(payload))
            if version != PROTOCOL_VERSION:
                raise HandshakeError(f"protocol version {version} != {PROTOCOL_VERSION}")
            if (hk, hn) != (k, n):
                raise HandshakeError(f"scheme ({hk},{hn}) != ({k},{n})")
            if pm != mdig:
                raise HandshakeError("model digest mismatch")
            if ps != sdig:
                raise HandshakeError("schedule digest mismatch")
            if expect is not None and sender != expect:
                raise HandshakeError(f"peer claims rank {sender}, expected {expect}")
            return sender

        def tune(sock):
            sock.settimeout(timeout)
            sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)

        socks = {}

        def dial(peer):
            host, port = peers[peer - 1]
            deadline = time.monotonic() + dial_deadline
            while True:
                try:
                    sock = socket.create_connection((host, port), timeout=timeout)
                    break
                except OSError:
                    if time.monotonic() > deadline:
                        raise PartyTimeout(f"cannot reach party {peer}") from None
                    time.sleep(0.05)
            tune(sock)
            sock.sendall(hello)
            _, phase, payload = read_frame(sock)
            if phase != Phase.HELLO:
                raise ProtocolError("expected hello")
            check(payload, expect=peer)
            socks[peer] = sock

        if rank == 0:
            for j in range(1, n + 1):
                dial(j)
            return cls(rank, socks, device, p, metrics, decode_object, timeout)
        host, port = peers[rank - 1]
        server = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        server.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        server.bind((host, port))
        server.listen(n + 1)
        server.settimeout(timeout)
        try:
            for j in range(1, rank):
                dial(j)
            for _ in range((n - rank) + (1 if expect_source else 0)):
                try:
                    conn, _ = server.accept()
                except socket.timeout:
                    raise PartyTimeout("timed out waiting for peers") from None
                tune(conn)
                _, phase, payload = read_frame(conn)
                if phase != Phase.HELLO:
                    raise ProtocolError("expected hello")
                sender = check(payload)
                conn.sendall(hello)
                socks[sender] = conn
        finally:
            server.close()
        return cls(rank, socks, device, p, metrics, decode_object, timeout)

    # ---- the seam (S/protocol.py:111-128)
    def _send_frame(self, dst, phase, payload, elements):
        frame = encode_frame(self.rank, phase, payload)
        self._writers[dst].put(frame)
        if self.metrics is not None:
            self.metrics.on_send(self.rank, len(frame), elements)

    def send_share(self, dst, phase, party_id, degree, tensor, elements=None):
        n = tensor.numel() if elements is None else elements
        self._send_frame(dst, phase, encode_share_payload(party_id, degree, _host_u64(tensor)), n)

    def send_plain(self, dst, phase, tensor, elements=None):
        n = tensor.numel() if elements is None else elements
        self._send_frame(dst, phase, encode_plain_payload(_host_u64(tensor)), n)

    def send_object(self, dst, phase, obj, nbytes, elements, encode=None):
        if encode is None:
            raise ValueError("send_object over TCP needs an encoder")
        self._send_frame(dst, phase, encode(), elements)

    def recv(self, src, phase, elements=0):
        sender, got, payload = read_frame(self._socks[src])
        if sender != src:
            raise ProtocolError(f"frame from {sender} on channel of {src}")
        if got != phase:
            raise ScheduleDivergence(f"party {self.rank} expected {Phase(phase).name} from {src}, got {got.name}")
        nbytes = FRAME_HEADER_SIZE + len(payload)
        if got == Phase.MASK_DIST:
            obj = self.decode_object(bytes(payload)) if self.decode_object is not None else bytes(payload)
            msg = Message(sender, got, "object", None, obj, nbytes)
        elif got == Phase.NONLIN_PLAIN:
            vals = decode_plain_payload(payload)
            msg = Message(sender, got, "plain", None, self._to_device(vals), nbytes)
            if nbytes != plain_frame_bytes(vals.shape):
                raise ProtocolError("plaintext frame size mismatch")
        else:
            pid, degree, vals = decode_share_payload(payload, self.p)
            msg = Message(sender, got, "share", (pid, degree), self._to_device(vals), nbytes)
            if nbytes != share_frame_bytes(vals.shape):
                raise ProtocolError("share frame size mismatch")
        if self.metrics is not None:
            self.metrics.on_recv(self.rank, nbytes, elements)
        return msg

    def _to_device(self, vals_u64):
        t = torch.from_numpy(np.ascontiguousarray(vals_u64).view(np.int64))
        return t.to(self.device) if self.device.type != "cpu" else t.clone()

    def close(self):
        try:
            for w in self._writers.values():
                w.flush(self.timeout)
        finally:
            self._close_socks()

    def _close_socks(self):
        for sock in self._socks.values():
            try:
                sock.shutdown(socket.SHUT_RDWR)
            except OSError:
                pass
            sock.close()
        self._socks.clear()


def run_party_tcp(rank, peers, model, scheme, seed, input_int, device, ordering="ltn", rng_mode="host",
                  input_index=0, metrics=None, timeout=60.0):
    """This host's party `rank` of one secure inference over TCP -- the reference's
    run_tcp_party (S/engine.py:208-229) with this package's kernels: weight and input shares
    are dealt from the seed exactly as the reference deals them (rng_mode="host"), the mask
    bundle arrives from the source in the reference's MASK_DIST frame.  Returns the decoded
    output at the elite (rank 1), None elsewhere."""
    from .dist import mask_bundle_decoder
    from .engine import (PURPOSE_PARTY, deal_input_shares, deal_weight_shares, lane_rng, receive_bundle,
                         run_party_online)
    from .layers import plan_schedule
    from .protocol import PartyContext
    ops, sdig = plan_schedule(model, scheme, ordering)
    tr = TcpTransport.establish(rank, peers, scheme.k, scheme.n, model.digest(), sdig, device=device,
                                p=scheme.field.p, metrics=metrics, expect_source=True, timeout=timeout,
                                decode_object=mask_bundle_decoder(scheme, device))
    try:
        weight_values = {name: qt.values for name, qt in model.weights.items()}
        w_share = deal_weight_shares(weight_values, scheme, seed, rng_mode)[rank]
        x_share = deal_input_shares(input_int, scheme, seed, input_index, rng_mode)[rank - 1]
        ctx = PartyContext(scheme, rank, tr, rng=lane_rng(rng_mode, seed, PURPOSE_PARTY, rank))
        if metrics is not None:
            metrics.set_op(rank, "offline", -1)
        receive_bundle(ctx)
        out = run_party_online(ctx, ops, w_share, x_share, metrics)
        return None if out is None else np.asarray(out, dtype=np.int64)
    finally:
        tr.close()


def run_source_tcp(peers, model, scheme, seed, ordering="ltn", rng_mode="host", metrics=None, timeout=60.0):
    """The trusted source over TCP (S/engine.py:232-246): one MASK_DIST frame per party."""
    from .engine import send_bundles
    from .layers import plan_schedule
    ops, sdig = plan_schedule(model, scheme, ordering)
    tr = TcpTransport.establish(0, peers, scheme.k, scheme.n, model.digest(), sdig, p=scheme.field.p,
                                metrics=metrics, timeout=timeout)
    try:
        send_bundles(tr, ops, scheme, seed, metrics, rng_mode)
    finally:
        tr.close()
