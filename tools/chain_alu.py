"""Calibrate bench.py's CHAIN_ALU: executed thread instructions and FMA-heavy pipe cycles per
chain element for one workload (the chain kernels are bound by the FMA-heavy pipe that executes
IMAD).  Run one warm step under ncu first:
  ncu --metrics smsp__thread_inst_executed.sum,sm__pipe_fmaheavy_cycles_active.sum,\
sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg \
      --profile-from-start off -k regex:k_chain --csv --log-file chain.csv \
      python tools/profile_step.py WORKLOAD BATCH
then: python tools/chain_alu.py WORKLOAD BATCH chain.csv  (needs the GPU for the element count)."""
import csv
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_02629_b200.batched import BatchedEngine  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402

wl, B, path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
kind, k, n, verify, _ = bench.WORKLOADS[wl]
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
eng.enable_profiling()
eng.run_device(x)
stats = eng.profile_summary(1)
eng.disable_profiling()
elems = stats["chain"]["elems_per_launch"] * stats["chain"]["launches_per_step"]
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if "Metric Value" in r)
vi, ni = rows[h].index("Metric Value"), rows[h].index("Metric Name")


def total(metric):
    return sum(float(r[vi].replace(",", "")) for r in rows[h + 1:] if len(r) > vi and r[ni] == metric)


def per_launch(metric):
    return [float(r[vi].replace(",", "")) for r in rows[h + 1:] if len(r) > vi and r[ni] == metric]


inst = total("smsp__thread_inst_executed.sum")
heavy = total("sm__pipe_fmaheavy_cycles_active.sum")
# heavy-pipe slots per SM per cycle, from ncu's own normalisation: sum / (SMs * cycles * pct)
pct, cyc, hv = (per_launch("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                per_launch("sm__cycles_elapsed.avg"), per_launch("sm__pipe_fmaheavy_cycles_active.sum"))
nsm = torch.cuda.get_device_properties(0).multi_processor_count
slots = [h_ / (nsm * c * p / 100.0) for h_, c, p in zip(hv, cyc, pct) if c and p]
print(f"{wl} B={B} (k,n)=({k},{n}): {inst:.4g} thread instructions / {elems:.4g} chain elements = "
      f"{inst / elems:.0f} per element; FMA-heavy pipe {heavy / elems:.1f} cycles per element "
      f"({sum(slots) / max(len(slots), 1):.2f} slots per SM per cycle); mean heavy-pipe busy "
      f"{sum(pct) / max(len(pct), 1):.1f}% of elapsed")
