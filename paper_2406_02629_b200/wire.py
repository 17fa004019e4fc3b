"""Wire vocabulary shared with the reference (S/wire.py).

On the B200 path share tensors move as device buffers (co-resident hand-off or NCCL), not
bytes; this module keeps the reference's phase tags, error types and exact frame sizes so
that CommMetrics byte counts match, and can serialize a device tensor into the reference
frame format when a transcript is recorded (tests only; the reference digests every frame,
S/transport.py:68-80).
"""

import struct
from enum import IntEnum

import numpy as np

MAGIC = b"SSN1"
PROTOCOL_VERSION = 1
FRAME_HEADER_SIZE = 12          # "<4sHHI" (S/wire.py:23)


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
    """len(frame) of encode_share_tensor: 12 + (8+2+1) + 4*ndim + 8*numel (S/wire.py:104-107)."""
    n = int(np.prod(shape)) if len(shape) else 1
    return FRAME_HEADER_SIZE + 11 + 4 * len(shape) + 8 * n


def plain_frame_bytes(shape):
    """len(frame) of encode_plain_tensor: 12 + 1 + 4*ndim + 8*numel (S/wire.py:95-98)."""
    n = int(np.prod(shape)) if len(shape) else 1
    return FRAME_HEADER_SIZE + 1 + 4 * len(shape) + 8 * n


def encode_frame(sender, phase, payload):
    return struct.pack("<4sHHI", MAGIC, sender, int(phase), len(payload)) + payload


def encode_share_payload(party_id, degree, values_u64):
    v = np.asarray(values_u64, dtype=np.uint64)
    return struct.pack(f"<QHB{v.ndim}I", party_id, degree, v.ndim, *v.shape) + v.astype("<u8").tobytes()


def encode_plain_payload(values_u64):
    v = np.asarray(values_u64, dtype=np.uint64)
    return struct.pack(f"<B{v.ndim}I", v.ndim, *v.shape) + v.astype("<u8").tobytes()
