"""Wire formats, the TCP mesh and the file containers (host side, no GPU).

Pinned to tests/golden/wire.json (made by the reference itself, make_wire_golden.py): frame,
HELLO, share / plaintext payloads, MaskBundle encoding, model and share files.  The TCP mesh
is exercised between this package's ranks and -- when the unmodified reference is installed in
baseline/_ref (tools/install_reference.sh) -- between this package and the reference's own
TcpTransport on localhost (S/transport.py:146-263).
"""
import hashlib
import json
import os
import socket
import sys
import threading

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_02629_b200 import containers, wire  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.model import build_reference_model  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402
from paper_2406_02629_b200.tcp import TcpTransport  # noqa: E402
from paper_2406_02629_b200.transport import HandshakeError, ScheduleDivergence  # noqa: E402

G = json.load(open(os.path.join(ROOT, "tests", "golden", "wire.json")))
FILES = os.path.join(ROOT, "tests", "golden", "wire_files")
P = PrimeField().p


def test_frame_and_hello_match_reference_bytes():
    assert wire.encode_frame(3, wire.Phase.RESHARE_OUT, b"\x01\x02\x03").hex() == G["frame"]
    assert wire.decode_frame(bytes.fromhex(G["frame"])) == (3, wire.Phase.RESHARE_OUT, b"\x01\x02\x03")
    hello = wire.encode_hello(3, 5, 2, bytes(range(32)), bytes(range(32, 64)))
    assert hello.hex() == G["hello"]
    assert wire.decode_hello(hello) == (1, 3, 5, 2, bytes(range(32)), bytes(range(32, 64)))
    frame = bytes.fromhex(G["frame"])
    with pytest.raises(wire.ProtocolError):
        wire.decode_frame(b"XXXX" + frame[4:])                     # bad magic
    with pytest.raises(wire.ProtocolError):
        wire.decode_frame(frame[:-1])                             # length mismatch
    with pytest.raises(wire.ProtocolError):
        wire.decode_frame(frame[:6])                              # short
    with pytest.raises(wire.ProtocolError):
        wire.decode_frame(wire.encode_frame(1, 2, b"")[:6] + (99).to_bytes(2, "little") + frame[8:12])
    with pytest.raises(wire.ProtocolError):
        wire.decode_hello(hello[:-1])


def test_payloads_match_reference_bytes():
    vals = np.array([[0, 1, P - 1], [12345678901, 2, 3]], dtype=np.uint64)
    assert wire.encode_plain_payload(vals).hex() == G["plain_payload"]
    assert np.array_equal(wire.decode_plain_payload(bytes.fromhex(G["plain_payload"])), vals)
    pid, deg, got = wire.decode_share_payload(bytes.fromhex(G["share_payload"]), P)
    assert [int(v) for v in got] == G["share_payload_values"]
    assert wire.encode_share_payload(pid, deg, got).hex() == G["share_payload"]
    bad = bytearray(bytes.fromhex(G["share_payload"]))
    bad[-8:] = (P).to_bytes(8, "little")                          # element == p
    with pytest.raises(wire.ProtocolError):
        wire.decode_share_payload(bytes(bad), P)


class _St:                      # host stand-in for a ShareTensor (the real one lives in HBM)
    def __init__(self, party_id, degree, values):
        self.party_id, self.degree, self.values = party_id, degree, torch.from_numpy(values.view(np.int64).copy())
        self.shape, self.size = tuple(values.shape), values.size


def test_mask_bundle_roundtrip_matches_reference_bytes():
    from paper_2406_02629_b200.protocol import MaskBundle
    ents = MaskBundle.decode_entries(bytes.fromhex(G["mask_bundle"]), P)
    assert [(e[0], e[1]) for e in ents] == [(0, "zero"), (2, "alpha")]
    b = MaskBundle({(op, name): _St(pid, deg, vals) for op, name, pid, deg, vals in ents})
    assert b.encode().hex() == G["mask_bundle"]
    with pytest.raises(wire.ProtocolError):
        MaskBundle.decode_entries(bytes.fromhex(G["mask_bundle"])[:-8], P)


def test_model_file_roundtrip_is_byte_identical(tmp_path):
    m = containers.load_model(os.path.join(FILES, "reference_model.ssnm"))
    ours, _ = build_reference_model(7)
    assert m.digest() == ours.digest() == G["model_digest"]
    out = tmp_path / "m.ssnm"
    assert containers.save_model(str(out), m) == G["model_digest"]
    assert hashlib.sha256(out.read_bytes()).hexdigest() == G["model_file_sha256"]
    raw = bytearray(out.read_bytes())
    raw[40] ^= 1
    out.write_bytes(bytes(raw))
    with pytest.raises(wire.ProtocolError):
        containers.load_model(str(out))


def test_share_file_roundtrip_is_byte_identical(tmp_path):
    src = os.path.join(FILES, "party2.shares")
    header, raw = containers.read_share_file(src)
    assert (header["k"], header["n"], header["rank"]) == (2, 3, 2) and "input" in raw
    entries = {name: _St(pid, deg, vals) for name, (pid, deg, vals) in raw.items()}
    out = tmp_path / "party2.shares"
    extra = {kk: header[kk] for kk in ("arch", "ordering", "seed", "input_index", "schedule_digest")}
    containers.save_shares(str(out), SssScheme(PrimeField(), 2, 3), 2, header["model_digest"], entries, extra=extra)
    assert hashlib.sha256(out.read_bytes()).hexdigest() == G["share_files_sha256"]["party2.shares"]
    with pytest.raises(wire.ProtocolError):                       # a share file is not a model file
        wire.read_container(str(out), containers.MODEL_MAGIC)


def _ports(n):
    socks = [socket.socket() for _ in range(n)]
    for s in socks:
        s.bind(("127.0.0.1", 0))
    ports = [s.getsockname()[1] for s in socks]
    for s in socks:
        s.close()
    return [("127.0.0.1", p) for p in ports]


def _mesh(n, k, digests, expect_source=True, timeout=20.0):
    """Rank 0..n of our TcpTransport on localhost threads -> {rank: transport}."""
    peers = _ports(n)
    out, errs = {}, []

    def up(r):
        try:
            out[r] = TcpTransport.establish(r, peers, k, n, digests[r][0], digests[r][1], p=P,
                                            expect_source=expect_source, timeout=timeout)
        except Exception as exc:           # noqa: BLE001 (collected and re-raised below)
            errs.append(exc)
    th = [threading.Thread(target=up, args=(r,)) for r in range(1, n + 1)]
    for t in th:
        t.start()
    if expect_source:
        up(0)
    for t in th:
        t.join()
    return out, errs


def test_tcp_mesh_moves_shares_plain_and_checks_phases():
    d = (hashlib.sha256(b"m").digest(), hashlib.sha256(b"s").digest())
    tr, errs = _mesh(3, 2, {r: d for r in range(4)})
    assert not errs, errs
    x = torch.arange(12, dtype=torch.int64).reshape(3, 4) * 977
    big = torch.randint(0, P, (1 << 19,), dtype=torch.int64)       # 4 MB: bigger than a socket buffer
    # both directions at once before either side receives (reshare step 1's pattern)
    tr[1].send_share(2, wire.Phase.RESHARE_OUT, 1, 2, big)
    tr[2].send_share(1, wire.Phase.RESHARE_OUT, 2, 2, big + 1)
    assert torch.equal(tr[1].recv(2, wire.Phase.RESHARE_OUT).tensor, big + 1)
    m = tr[2].recv(1, wire.Phase.RESHARE_OUT)
    assert m.meta == (1, 2) and torch.equal(m.tensor, big)
    tr[3].send_plain(1, wire.Phase.NONLIN_PLAIN, x)
    assert torch.equal(tr[1].recv(3, wire.Phase.NONLIN_PLAIN).tensor, x)
    tr[0].send_object(2, wire.Phase.MASK_DIST, None, 0, 0, encode=lambda: b"bundle-bytes")
    assert tr[2].recv(0, wire.Phase.MASK_DIST).tensor == b"bundle-bytes"
    tr[1].send_share(3, wire.Phase.TRUNC_MASKED, 1, 1, x)
    with pytest.raises(ScheduleDivergence):
        tr[3].recv(1, wire.Phase.SHARE_DIST)
    for t in tr.values():
        t.close()


def test_tcp_handshake_rejects_mismatched_schedule():
    good = (hashlib.sha256(b"m").digest(), hashlib.sha256(b"s").digest())
    bad = (good[0], hashlib.sha256(b"other").digest())
    tr, errs = _mesh(2, 2, {0: good, 1: good, 2: bad}, expect_source=False, timeout=5.0)
    assert any(isinstance(e, HandshakeError) for e in errs), errs
    for t in tr.values():
        t.close()


def _reference():
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    try:
        import ssnet
        return ssnet
    except ImportError:
        return None


def test_tcp_interoperates_with_reference_transport():
    """Our rank 1 and the reference's ranks 2, 3 (+ its source) form ONE mesh: HELLO digests,
    frames and share payloads cross both ways (S/transport.py:146-263)."""
    ssnet = _reference()
    if ssnet is None:
        pytest.skip("reference not installed in baseline/_ref (tools/install_reference.sh)")
    from ssnet.transport import TcpTransport as RefTcp
    from ssnet import wire as rwire
    mdig, sdig = hashlib.sha256(b"m").digest(), hashlib.sha256(b"s").digest()
    peers = _ports(3)
    tr, errs = {}, []

    def ours():
        try:
            tr[1] = TcpTransport.establish(1, peers, 2, 3, mdig, sdig, p=P, expect_source=True, timeout=20)
        except Exception as exc:          # noqa: BLE001
            errs.append(exc)

    def ref(r):
        try:
            tr[r] = RefTcp.establish(r, peers, 2, 3, mdig, sdig, expect_source=True, timeout=20)
        except Exception as exc:          # noqa: BLE001
            errs.append(exc)
    th = [threading.Thread(target=ours)] + [threading.Thread(target=ref, args=(r,)) for r in (2, 3)]
    for t in th:
        t.start()
    tr[0] = RefTcp.establish(0, peers, 2, 3, mdig, sdig, timeout=20)
    for t in th:
        t.join()
    assert not errs, errs
    s23 = ssnet.SssScheme(ssnet.PrimeField(), 2, 3)
    vals = np.array([[1, 2, 3], [P - 1, 0, 99]], dtype=object)
    st = ssnet.ShareTensor(2, 1, vals, s23)
    tr[2].send(1, rwire.Phase.SHARE_DIST, rwire.encode_share_tensor(st), elements=6)
    m = tr[1].recv(2, wire.Phase.SHARE_DIST)
    assert m.meta == (2, 1) and m.tensor.tolist() == [[1, 2, 3], [P - 1, 0, 99]]
    mine = torch.tensor([[5, 6], [7, P - 2]], dtype=torch.int64)
    tr[1].send_share(3, wire.Phase.RESHARE_BACK, 1, 1, mine)
    back = rwire.decode_share_tensor(tr[3].recv(1, rwire.Phase.RESHARE_BACK), s23)
    assert back.party_id == 1 and back.values.tolist() == [[5, 6], [7, P - 2]]
    tr[1].send_plain(2, wire.Phase.NONLIN_PLAIN, mine)
    assert rwire.decode_plain_tensor(tr[2].recv(1, rwire.Phase.NONLIN_PLAIN)).tolist() == mine.tolist()
    for t in tr.values():
        t.close()
