"""Reshare step 1 fused into the share GEMM's epilogue (ssn_gemm_tc_subshares) vs the GEMM
followed by ssn_gen, on the party-per-GPU path's shapes (one party, a ResNet-152 batch of 32):
device time per layer class.  Usage: python tools/fused_subshares_probe.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02629_b200 import _lib, gemm as G  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402

P = PrimeField().p
_lib.load()
B = 32
res = []
for (O, C, ks, H, stride, pad) in [(256, 256, 3, 14, 1, 1), (1024, 256, 1, 14, 1, 0), (256, 1024, 1, 14, 1, 0),
                                  (64, 64, 3, 56, 1, 1), (256, 64, 1, 56, 1, 0)]:
    for k, n in ((2, 3), (3, 5)):
        sch = SssScheme(PrimeField(), k, n)
        rng = np.random.default_rng(0)
        w = torch.as_tensor(rng.integers(0, P, size=(1, O, C, ks, ks), dtype=np.uint64).astype(np.int64), device="cuda")
        x = torch.as_tensor(rng.integers(0, P, size=(1, B, C, H, H), dtype=np.uint64).astype(np.int64), device="cuda")
        planes = G.weight_planes(w.reshape(1, O, -1), P, 1)
        OH = (H + 2 * pad - ks) // stride + 1
        N = B * O * OH * OH
        SUB = torch.empty((1, k, N), dtype=torch.int64, device="cuda")
        ids = _lib.u64_array(sch.front_ids)

        def unfused():
            acc = G.field_conv(w, x, stride, pad, P, nimg=B, nparty=1, planes=planes, force="tc")
            _lib.call("ssn_gen", _lib.ptr(acc), N, None, 0, 5, 9, k - 1, ids, k, _lib.ptr(SUB), N, N, N, 1, P,
                      _lib.stream_ptr())

        def fused():
            G.field_conv(w, x, stride, pad, P, nimg=B, nparty=1, planes=planes, force="tc",
                         sub=G.SubShares(SUB, 5, 9, k - 1, sch.front_ids))
        row = {"O": O, "C": C, "k": ks, "H": H, "scheme": [k, n]}
        for name, fn in (("unfused_ms", unfused), ("fused_ms", fused)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            row[name] = round(e0.elapsed_time(e1) / 10, 3)
        res.append(row)
        print(json.dumps(row), flush=True)
out = sys.argv[1] if len(sys.argv) > 1 else None
if out:
    json.dump(res, open(out, "w"), indent=1)
