"""Measure the dense int8 tensor-pipe peak of this B200 with ssn_mma_peak (back-to-back
tcgen05.mma.kind::i8 128x256x32 from resident smem, one CTA per SM): burst = best of 5 single
launches, sustained = launches back to back for ~4 s.  Writes the JSON given as argv[1]
(bench.py reads profiles/r*/int8_peak.json for the share-GEMM roofline)."""
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02629_b200 import _lib  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "int8_peak.json"
L = _lib.load()
nsm = torch.cuda.get_device_properties(0).multi_processor_count
ms, ops = ctypes.c_float(), ctypes.c_double()


def one(iters):
    _lib.call("ssn_mma_peak", iters, nsm, ctypes.byref(ms), ctypes.byref(ops), _lib.stream_ptr())
    return ops.value / (ms.value / 1e3) / 1e12, ms.value


iters = 400000
burst = max(one(iters)[0] for _ in range(5))
t0, vals = time.perf_counter(), []
while time.perf_counter() - t0 < 4.0:
    vals.append(one(iters)[0])
sustained = sum(vals) / len(vals)
res = {"int8_tops_burst": round(burst, 1), "int8_tops_sustained": round(sustained, 1), "sms": nsm,
       "mma": "tcgen05.mma.cta_group::1.kind::i8 M=128 N=256 K=32, one CTA per SM, resident smem operands",
       "iters_per_launch": iters, "gpu": torch.cuda.get_device_name(0)}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
