"""Run one warm step of the batched engine inside a cudaProfilerStart/Stop range (for ncu
--profile-from-start off).  Usage: python tools/profile_step.py [workload] [batch (default: bench.py's)]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_02629_b200.batched import BatchedEngine  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet152-5pc"
kind, k, n, verify, dflt = bench.WORKLOADS[wl]
# default: one bench engine's batch (the bench splits its batch over DEFAULT_STREAMS engines)
B = int(sys.argv[2]) if len(sys.argv) > 2 else dflt // bench.DEFAULT_STREAMS.get(wl, 1)
model = bench.build_model(kind)
eng = BatchedEngine(model, SssScheme(PrimeField(), k, n), batch=B, seed=7, verify=verify)
if hasattr(model, "random_inputs"):
    xb = model.random_inputs(seed=1, batch=B)
else:                                        # ModelGraph (LeNet-style chain models)
    import numpy as np
    from paper_2406_02629_b200.model import random_input
    xb = np.stack([random_input(1, model, index=i)[0] for i in range(B)])
x = torch.as_tensor(xb, device="cuda")
eng.run_device(x)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.run_device(x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one step:", wl, "batch", B)
