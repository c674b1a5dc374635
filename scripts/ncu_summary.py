"""Summarise an ncu capture into profiles/ (tracked):
    python scripts/ncu_summary.py <tag> [--rep gpurun_out/<tag>_transform.ncu-rep]
                                        [--launches gpurun_out/<tag>_launches.csv]
Writes profiles/<tag>_ncu_<name>.json (per-kernel key metrics of the full
capture; bench.py reads dram traffic from it) and profiles/<tag>_launches.md
(the launch list of the bench command grouped by kernel, with the first
timed step spelled out)."""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}


def kname(n):
    n = re.sub(r"^void ", "", n)
    n = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", n)
    return n.split("(")[0]


def full(rep, tag, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        if not r or len(r) != len(h):
            continue
        k = {"kernel": kname(r[h.index("Kernel Name")])}
        for key in KEYS:
            if key in h:
                i = h.index(key)
                v = float(r[i].replace(",", "")) if r[i] else None
                unit = u[i]
                if unit in ("byte", "Kbyte", "Mbyte", "Gbyte") and v is not None:
                    v, unit = v * SCALE[unit], "byte"
                if unit in ("ns", "us", "ms") and v is not None:
                    v, unit = v * SCALE[unit], "us"
                k[key] = v
        kernels.append(k)
    doc = {"source": os.path.relpath(rep, ROOT), "command": "see scripts/gpu_round.sh (ncu --set full)",
           "kernels": kernels,
           # one transform step = one launch: per-launch means over the captured launches
           "step": {"launches_captured": len(kernels),
                    "duration_us": sum(k["gpu__time_duration.sum"] for k in kernels) / max(1, len(kernels)),
                    "dram_bytes": sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in kernels)
                    / max(1, len(kernels))}}
    path = os.path.join(ROOT, "profiles", f"{tag}_ncu_{name}.json")
    json.dump(doc, open(path, "w"), indent=1)
    print("wrote", path)


def launches(path_csv, tag):
    rows = list(csv.reader(open(path_csv)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi, bi = h.index("Grid Size"), h.index("Block Size")
    seq = []
    for r in rows[hi + 1:]:
        if len(r) > vi and r[vi]:
            seq.append((kname(r[ki]), float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1), r[gi], r[bi]))
    agg = collections.OrderedDict()
    for n, us, g, b in seq:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v for _, v in agg.values())
    lines = [f"# {tag}: ncu launch list of the bench command", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv "
             "python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline` (scripts/gpu_round.sh).",
             "Per-launch times are cold-cache and serialised by ncu; compare SHARES, not absolute times.",
             f"Launches captured: {len(seq)} (cap 3000), total {tot:.1f} us.", "",
             "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
    for n, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{n[:90]}` | {c} | {us:.1f} | {100 * us / tot:.1f}% |")
    # the timed transform steps come first in bench.py: show one step
    lines += ["", "First launches (warm-up + timed transform steps, in order):", "",
              "| # | kernel | us | grid | block |", "|---:|---|---:|---|---|"]
    for i, (n, us, g, b) in enumerate(seq[:24]):
        lines.append(f"| {i} | `{n[:80]}` | {us:.2f} | {g} | {b} |")
    path = os.path.join(ROOT, "profiles", f"{tag}_launches.md")
    open(path, "w").write("\n".join(lines) + "\n")
    print("wrote", path)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--rep")
    ap.add_argument("--name", default="transform")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.rep:
        full(a.rep, a.tag, a.name)
    if a.launches:
        launches(a.launches, a.tag)
