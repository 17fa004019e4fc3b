"""Host-side (Python) profile of one warm ResNet-152 5PC step: where enqueue time goes."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_02629_b200.batched import BatchedEngine  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402

model = bench.build_model("imagenet152")
eng = BatchedEngine(model, SssScheme(PrimeField(), 3, 5), batch=16, seed=7, verify=True)
eng.defer_verify = True
x = torch.as_tensor(model.random_inputs(seed=1, batch=16), device="cuda")
for _ in range(3):
    eng.run_device(x)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    eng.run_device(x)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
