"""Batch-1 latency split: host enqueue time of one inference vs its device time with the host
decoupled (a long torch.cuda._sleep is queued first, so the whole inference is enqueued before
the GPU reaches it and its CUDA-event time is pure device time).
Usage: python tools/latency_probe.py [workload] [batch]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_02629_b200 import _lib  # noqa: E402
from paper_2406_02629_b200.batched import BatchedEngine  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet152-5pc"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
kind, k, n, verify, _ = bench.WORKLOADS[wl]
model = bench.build_model(kind)
eng = BatchedEngine(model, SssScheme(PrimeField(), k, n), batch=B, seed=7, verify=verify)
eng.defer_verify = True
x = torch.as_tensor(model.random_inputs(seed=1, batch=B), device="cuda")
for _ in range(3):
    eng.run_device(x)
torch.cuda.synchronize()
res = {"workload": wl, "batch": B}
# 1) back to back (what bench.py's latency_batch1 measures)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    eng.run_device(x)
e1.record()
torch.cuda.synchronize()
res["back_to_back_ms"] = round(e0.elapsed_time(e1) / 5, 3)
# 2) host enqueue time and device-only time of one inference
dev, host = [], []
for _ in range(5):
    torch.cuda._sleep(int(2e9 * 0.2))                    # ~0.2 s of GPU spin at ~2 GHz
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    l0 = _lib.launch_count()
    h0 = time.perf_counter()
    eng.run_device(x)
    host.append((time.perf_counter() - h0) * 1e3)
    launches = _lib.launch_count() - l0
    b.record()
    torch.cuda.synchronize()
    dev.append(a.elapsed_time(b))
res["host_enqueue_ms"] = round(min(host), 3)
res["device_ms"] = round(min(dev), 3)
res["launches"] = launches
print(res)
