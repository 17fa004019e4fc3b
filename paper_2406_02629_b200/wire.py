"""Byte formats shared with the reference (S/wire.py): frames, HELLO, tensor payloads, and the
sha256-sealed file containers.

On the B200 path share tensors move as device buffers (co-resident hand-off or NCCL), not
bytes.  Bytes are needed where a party talks to the outside world -- the cross-host TCP
transport (tcp.py, wire-compatible with the reference's TcpTransport), share / mask-bundle /
model files, and recorded transcripts (S/transport.py:68-80).  Element blobs are u64
little-endian, row-major; they are built from and decoded into whole numpy / torch buffers
(one memcpy, no per-element struct packing).
"""

import hashlib
import json
import struct
from enum import IntEnum

import numpy as np

MAGIC = b"SSN1"
PROTOCOL_VERSION = 1
_FRAME = struct.Struct("<4sHHI")          # magic, sender u16, phase u16, payload_len u32 (S/wire.py:23)
_HELLO = struct.Struct("<HHHH32s32s")     # version, k, n, sender, model digest, schedule digest (:24)
_CONTAINER = struct.Struct("<4sHI")       # magic, version u16, header_len u32 (:25)
FRAME_HEADER_SIZE = _FRAME.size           # 12
HELLO_SIZE = _HELLO.size                  # 72


class ProtocolError(Exception):
    """A peer violated the wire protocol."""


class Phase(IntEnum):           # S/wire.py:32-41
    HELLO = 1
    MASK_DIST = 2
    SHARE_DIST = 3
    RESHARE_OUT = 4
    RESHARE_BACK = 5
    TRUNC_MASKED = 6
    NONLIN_MASKED = 7
    NONLIN_PLAIN = 8
    OUTPUT_SHARE = 9


def share_frame_bytes(shape):
    """len(frame) of a share-tensor frame: 12 + (8+2+1) + 4*ndim + 8*numel (S/wire.py:104-107)."""
    n = int(np.prod(shape)) if len(shape) else 1
    return FRAME_HEADER_SIZE + 11 + 4 * len(shape) + 8 * n


def plain_frame_bytes(shape):
    """len(frame) of a plaintext-tensor frame: 12 + 1 + 4*ndim + 8*numel (S/wire.py:95-98)."""
    n = int(np.prod(shape)) if len(shape) else 1
    return FRAME_HEADER_SIZE + 1 + 4 * len(shape) + 8 * n


# ---------------------------------------------------------------- frames and HELLO

def encode_frame(sender, phase, payload):
    return _FRAME.pack(MAGIC, sender, int(phase), len(payload)) + payload


def frame_header(buf):
    """(sender, Phase, payload_len) of a 12-byte frame header (S/wire.py:48-60 checks)."""
    if len(buf) < FRAME_HEADER_SIZE:
        raise ProtocolError("short frame")
    magic, sender, phase, plen = _FRAME.unpack_from(buf)
    if magic != MAGIC:
        raise ProtocolError(f"bad magic {magic!r}")
    try:
        phase = Phase(phase)
    except ValueError:
        raise ProtocolError(f"unknown phase tag {phase}") from None
    return sender, phase, plen


def decode_frame(buf):
    """-> (sender, Phase, payload); the buffer must be exactly one frame."""
    sender, phase, plen = frame_header(buf)
    if len(buf) != FRAME_HEADER_SIZE + plen:
        raise ProtocolError("frame length mismatch")
    return sender, phase, bytes(buf[FRAME_HEADER_SIZE:])


def encode_hello(k, n, sender, model_digest, schedule_digest):
    return _HELLO.pack(PROTOCOL_VERSION, k, n, sender, digest32(model_digest), digest32(schedule_digest))


def decode_hello(payload):
    """-> (version, k, n, sender, model_digest, schedule_digest)."""
    if len(payload) != HELLO_SIZE:
        raise ProtocolError("bad hello size")
    return _HELLO.unpack(payload)


def digest32(value):
    """A 32-byte digest from bytes or a hex string (S/transport.py:132-143)."""
    if isinstance(value, str):
        value = bytes.fromhex(value)
    value = bytes(value)
    if len(value) != 32:
        raise ValueError(f"digest must be 32 bytes, got {len(value)}")
    return value


# ---------------------------------------------------------------- tensor payloads

def _u64(values):
    v = np.asarray(values)
    if v.dtype == object:
        v = v.astype(np.uint64)
    return np.ascontiguousarray(v.astype("<u8", copy=False))


def encode_elements(values):
    """Field elements as u64 LE, row-major (S/wire.py:79-82)."""
    return _u64(values).tobytes()


def decode_elements(buf, count, offset=0):
    """count u64 LE elements at offset -> uint64 ndarray (a view of buf when it is bytes)."""
    if offset + 8 * count > len(buf):
        raise ProtocolError("element blob shorter than its header says")
    return np.frombuffer(buf, dtype="<u8", count=count, offset=offset)


def encode_share_payload(party_id, degree, values_u64):
    v = _u64(values_u64)
    return struct.pack(f"<QHB{v.ndim}I", party_id, degree, v.ndim, *v.shape) + v.tobytes()


def decode_share_payload(buf, p=None):
    """-> (party_id, degree, uint64 ndarray); rejects elements >= p (S/wire.py:110-123)."""
    if len(buf) < 11:
        raise ProtocolError("short share payload")
    party_id, degree, ndim = struct.unpack_from("<QHB", buf)
    shape = struct.unpack_from(f"<{ndim}I", buf, 11)
    count = int(np.prod(shape)) if ndim else 1
    off = 11 + 4 * ndim
    if len(buf) != off + 8 * count:
        raise ProtocolError("share payload length mismatch")
    vals = decode_elements(buf, count, off).reshape(shape)
    if p is not None and count and int(vals.max()) >= p:
        raise ProtocolError("element outside field range")
    return party_id, degree, vals


def encode_plain_payload(values_u64):
    v = _u64(values_u64)
    return struct.pack(f"<B{v.ndim}I", v.ndim, *v.shape) + v.tobytes()


def decode_plain_payload(buf):
    """-> uint64 ndarray (S/wire.py:95-101)."""
    if len(buf) < 1:
        raise ProtocolError("short plaintext payload")
    ndim = buf[0]
    shape = struct.unpack_from(f"<{ndim}I", buf, 1)
    count = int(np.prod(shape)) if ndim else 1
    off = 1 + 4 * ndim
    if len(buf) != off + 8 * count:
        raise ProtocolError("plaintext payload length mismatch")
    return decode_elements(buf, count, off).reshape(shape)


# ---------------------------------------------------------------- file containers

def write_container(path, magic, header, blob):
    """magic | version u16 | header_len u32 | header JSON | blob | sha256 of all before it
    (S/wire.py:129-135).  Returns the digest."""
    head = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
    body = _CONTAINER.pack(magic, 1, len(head)) + head + bytes(blob)
    digest = hashlib.sha256(body).digest()
    with open(path, "wb") as fh:
        fh.write(body)
        fh.write(digest)
    return digest


def read_container(path, magic):
    """-> (header dict, blob bytes, digest); ProtocolError on a bad seal, magic or version."""
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < _CONTAINER.size + 32:
        raise ProtocolError("truncated container")
    body, digest = data[:-32], data[-32:]
    if hashlib.sha256(body).digest() != digest:
        raise ProtocolError("container digest mismatch")
    got, version, hlen = _CONTAINER.unpack_from(body)
    if got != magic:
        raise ProtocolError(f"expected {magic!r} container, found {got!r}")
    if version != 1:
        raise ProtocolError(f"unsupported container version {version}")
    off = _CONTAINER.size
    header = json.loads(body[off:off + hlen].decode())
    return header, body[off + hlen:], digest
