"""Tensor-pipe rate of the share GEMM's MMA issue pattern (ssn_mma_probe) against the plain
back-to-back peak: is the int8 GEMM limited by its MMA shape / operand reads, or by its
pipeline?  Usage: python tools/mma_probe.py [out.json]"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02629_b200 import _lib  # noqa: E402

_lib.load()
nsm = torch.cuda.get_device_properties(0).multi_processor_count
ms, ops = ctypes.c_float(), ctypes.c_double()
res = {}
for mode, n in ((0, 256), (0, 192), (0, 128), (0, 96), (0, 64), (0, 32), (1, 192), (1, 96)):
    best = 0.0
    for _ in range(3):
        _lib.call("ssn_mma_probe", mode, n, 120000, nsm, ctypes.byref(ms), ctypes.byref(ops), _lib.stream_ptr())
        best = max(best, ops.value / (ms.value / 1e3) / 1e12)
    res[f"mode{mode}_n{n}"] = round(best, 1)
    print(f"mode {mode} N={n}: {best:.1f} int8 TOP/s", flush=True)
if len(sys.argv) > 1:
    json.dump(res, open(sys.argv[1], "w"), indent=1)
