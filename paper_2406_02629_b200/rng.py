"""Randomness sources for share generation and masks.

Two modes, chosen by the rng object a caller passes (the reference passes numpy
Generators, S/engine.py:31-32):

* numpy.random.Generator -- *parity mode*: coefficients / masks are drawn on the host with
  exactly the reference's calls (rng.integers(0, p, size, int64), S/field.py:138-142) and
  uploaded, so every share is bit-identical to the reference run with the same seed.
* DeviceRng -- *speed mode*: Philox4x32-10 evaluated inside the kernels
  (csrc/ssn_field.cuh).  Each draw site consumes a fresh stream id from a host counter,
  so runs are deterministic given the seed.  Decoded outputs are RNG-independent
  (T/test_engine.py:66-74), so speed mode still reproduces the reference's outputs.
"""

import hashlib


class DeviceRng:
    def __init__(self, seed, *path):
        h = hashlib.sha256(repr((int(seed),) + tuple(int(x) for x in path)).encode()).digest()
        self.seed = int.from_bytes(h[:8], "little")
        self._stream = int.from_bytes(h[8:12], "little") << 20

    def next_stream(self, count=1):
        s = self._stream
        self._stream += int(count)
        return s

    def spawn(self, *path):
        return DeviceRng(self.seed, *path)

    def __repr__(self):
        return f"DeviceRng(seed={self.seed:#x}, stream={self._stream})"
