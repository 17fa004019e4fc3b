"""Kernel timeline of one overlapped (two-stream) step: CUDA events around every GEMM and chain
launch on its own stream, relative to one start event.  Prints how much GEMM time of one
sub-batch ran while the other sub-batch was inside a chain kernel, and the gaps.
Usage: python tools/timeline.py [workload] [batch] [out.json]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_02629_b200.batched import StreamPipelinedEngine  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet152-5pc"
kind, k, n, verify, dflt = bench.WORKLOADS[wl]
B = int(sys.argv[2]) if len(sys.argv) > 2 else dflt
model = bench.build_model(kind)
eng = StreamPipelinedEngine(model, SssScheme(PrimeField(), k, n), batch=B, streams=2, seed=7, verify=verify)
for e in eng.engines:
    e.defer_verify = True
x = torch.as_tensor(model.random_inputs(seed=1, batch=B), device="cuda")
eng.run_device(x)
eng.run_device(x)
torch.cuda.synchronize()
eng.enable_profiling()
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
eng.run_device(x)
t1 = torch.cuda.Event(enable_timing=True)
t1.record()
torch.cuda.synchronize()
step = t0.elapsed_time(t1)
iv = []
for si, e in enumerate(eng.engines):
    for cls, rec in e._prof.items():
        for r in rec:
            iv.append((si, cls, t0.elapsed_time(r[0]), t0.elapsed_time(r[1])))
eng.disable_profiling()


def overlap(a, b):
    """total length of the intersection of two interval lists"""
    tot = 0.0
    for s0, e0 in a:
        for s1, e1 in b:
            tot += max(0.0, min(e0, e1) - max(s0, s1))
    return tot


res = {"step_ms": step}
for si in (0, 1):
    g = [(s, e) for (i, c, s, e) in iv if i == si and c == "gemm"]
    ch = [(s, e) for (i, c, s, e) in iv if i == 1 - si and c == "chain"]
    res[f"gemm{si}_ms"] = sum(e - s for s, e in g)
    res[f"gemm{si}_under_chain{1 - si}_ms"] = overlap(g, ch)
busy = sorted((s, e) for (_, _, s, e) in iv)
idle, cur = 0.0, 0.0
for s, e in busy:
    if s > cur:
        idle += s - cur
    cur = max(cur, e)
res["no_kernel_ms"] = idle
res["by_class_ms"] = {}
for (_, c, s, e) in iv:
    res["by_class_ms"][c] = res["by_class_ms"].get(c, 0.0) + e - s
print(json.dumps(res))
if len(sys.argv) > 3:
    json.dump({"summary": res, "intervals": iv}, open(sys.argv[3], "w"))
