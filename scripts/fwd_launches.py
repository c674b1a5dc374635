"""Per-kernel durations of the last forward in an ncu launch list:
    python scripts/fwd_launches.py gpurun_out/<tag>_fwd_launches.csv"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, vi, ui, mi, gi = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name", "Grid Size"))
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    us = v / 1000 if r[ui] in ("nsecond", "ns") else (v if r[ui] in ("usecond", "us") else v * 1000)
    seq.append((re.sub(r"\(.*", "", r[ki]).replace("void ", "").split("::")[-1][:28], us, r[gi]))
n = len(seq) // 2
tot = 0.0
for name, us, grid in seq[n:]:
    tot += us
    print(f"{us:7.2f} {grid:>14} {name}")
print("total_us", round(tot, 1), "kernels", len(seq) - n)
