"""Per-layer ncu summary of one eager forward (K7 GEMMs + K8 kernels) into profiles/:
    python scripts/ncu_forward_summary.py <csv> <out.json> [--flops-json gpurun_out/<tag>_flops.json]

<csv>: `ncu --metrics <FWD_METRICS> --csv --log-file <csv> python scripts/prof_forward.py <arch> 1 1`
(one eager forward, one launch per kernel; ncu serialises launches and runs
them cold, so durations are per-kernel shares, not the graph's wall time).
Writes per launch: kernel, grid, duration, tensor-pipe instructions (tcgen05
MMA/commit), tensor-pipe active %, DRAM bytes; plus totals per kernel kind."""
import collections
import csv
import json
import sys

FWD_METRICS = ("gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__inst_executed_pipe_tc.sum,"
               "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,"
               "dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3}


def parse(path):
    rows = collections.OrderedDict()
    lines = [l for l in open(path) if l.startswith('"')]
    for r in csv.DictReader(lines):
        k = r["ID"]
        d = rows.setdefault(k, {"kernel": r["Kernel Name"].split("(")[0], "grid": r.get("Grid Size", "")})
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v) * SCALE.get(r["Metric Unit"], 1)
        except ValueError:
            pass
        d[r["Metric Name"]] = v
    return list(rows.values())


def main():
    src, out = sys.argv[1], sys.argv[2]
    rows = parse(src)
    launches = []
    for d in rows:
        launches.append({"kernel": d["kernel"], "grid": d["grid"],
                         "us": round(d.get("gpu__time_duration.sum", 0), 3),
                         "tc_inst": d.get("sm__inst_executed_pipe_tc.sum"),
                         "tensor_active_pct": d.get("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
                         "sm_throughput_pct": d.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                         "dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)})
    kinds = collections.OrderedDict()
    for l in launches:
        k = kinds.setdefault(l["kernel"], {"launches": 0, "us": 0.0})
        k["launches"] += 1
        k["us"] = round(k["us"] + l["us"], 3)
    doc = {"source": src, "launches": len(launches), "total_us_serialised": round(sum(l["us"] for l in launches), 2),
           "by_kernel": kinds, "per_launch": launches}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in doc.items() if k != "per_launch"}, indent=1))


if __name__ == "__main__":
    main()
