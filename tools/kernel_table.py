"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
unit = "ns"
total = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{name[:60]:60s} {cnt[name]:8d} {t / 1e6:10.3f} {t / total:7.1%}")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {total / 1e6:10.3f}")
