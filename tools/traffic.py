"""Aggregate an ncu --csv launch list with dram__bytes_{read,write}.sum and
gpu__time_duration.sum into per-kernel-class DRAM traffic per launch (bench.py's
roofline.traffic).  Usage: python tools/traffic.py launches.csv [workload] > profiles/rNN/traffic.json"""
import csv
import json
import sys
from collections import defaultdict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}


def kernel_class(name):
    if "k_gemm_p45" in name or "k_gemm_tc" in name:
        return "gemm"
    if "k_chain" in name:
        return "chain"
    if "k_im2col_limbs" in name or "k_limb_split" in name:
        return "im2col"
    return "other"


rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, ii, mi, ui, vi = (hdr.index(c) for c in ("Kernel Name", "ID", "Metric Name", "Metric Unit", "Metric Value"))
per_launch = defaultdict(dict)
names = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    per_launch[r[ii]][r[mi]] = v
    names[r[ii]] = r[ki]
agg = defaultdict(lambda: [0, 0.0, 0.0])
for lid, m in per_launch.items():
    c = kernel_class(names[lid])
    a = agg[c]
    a[0] += 1
    a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[2] += m.get("gpu__time_duration.sum", 0)
# a protocol-chain CALL (ssn_layer_chain) is one k_chain_plain and, for a nonlinear chain, one
# k_chain_nonlin; every call follows exactly one share GEMM, so per call = per GEMM launch
per_launch_bytes = {c: a[1] / a[0] for c, a in agg.items()}
if "chain" in agg and "gemm" in agg:
    per_launch_bytes["chain"] = agg["chain"][1] / agg["gemm"][0]
out = {"how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum over one "
              "warm step (tools/profile_step.py); cold-cache, serialised launches; chain: per chain call "
              "(plain + nonlinearity kernel), i.e. per share-GEMM launch",
       "workload": sys.argv[2] if len(sys.argv) > 2 else "resnet152-5pc",
       "bytes_per_launch": per_launch_bytes,
       "bytes_per_step": {c: a[1] for c, a in agg.items()},
       "launches": {c: a[0] for c, a in agg.items()},
       "ms_total": {c: a[2] / 1e6 for c, a in agg.items()}}
print(json.dumps(out, indent=1))
