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
               "sm__pipe_tensor_cycles_active_realtime.sum,sm__pipe_tensor_cycles_active_realtime.max,"
               "sm__cycles_elapsed.sum,sm__cycles_elapsed.max,"
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


def pct(a, b):
    try:
        return round(100.0 * float(a) / float(b), 3)
    except (TypeError, ValueError, ZeroDivisionError):
        return None


def main():
    src, out = sys.argv[1], sys.argv[2]
    rows = parse(src)
    launches = []
    for d in rows:
        launches.append({"kernel": d["kernel"], "grid": d["grid"],
                         "us": round(d.get("gpu__time_duration.sum", 0), 3),
                         "tc_inst": d.get("sm__inst_executed_pipe_tc.sum"),
                         # tensor pipe busy: over all SMs x the launch, and on the busiest SM
                         "tensor_active_pct_all_sms": pct(d.get("sm__pipe_tensor_cycles_active_realtime.sum"),
                                                          d.get("sm__cycles_elapsed.sum")),
                         "tensor_active_pct_busiest_sm": pct(d.get("sm__pipe_tensor_cycles_active_realtime.max"),
                                                             d.get("sm__cycles_elapsed.max")),
                         "sm_throughput_pct": d.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                         "dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)})
    # Tensor-pipe work issued: every tcgen05.mma (UTCHMMA) here is 128 x BN x 16
    # (cta_group::1, kind::f16), BN from the kernel's template arguments; the
    # issued rate against the 2.25 PFLOP/s dense bf16 peak is the tensor-pipe
    # utilisation (the realtime tensor-active counters read n/a on this ncu).
    import re
    for l in launches:
        # gemm_tc_kernel<BN, STAGES, S, MC> (MC = -2: a 2-SM pair, M = 256
        # per instruction) or gemm_persist_kernel<BN, STAGES>
        m = re.search(r"gemm_(?:tc|persist)_kernel<(\d+),\s*\d+(?:,\s*\d+,\s*(-?\d+))?", l["kernel"])
        if m and l["tc_inst"] and l["us"]:
            bn = int(m.group(1))
            rows = 256 if m.group(2) == "-2" else 128
            fl = float(l["tc_inst"]) * rows * bn * 16 * 2
            l["mma_flop_issued"] = fl
            l["mma_tflops_issued"] = round(fl / (l["us"] * 1e-6) / 1e12, 2)
            l["tensor_pipe_frac_of_2250tf"] = round(fl / (l["us"] * 1e-6) / 2.25e15, 4)
    kinds = collections.OrderedDict()
    for l in launches:
        k = kinds.setdefault(l["kernel"], {"launches": 0, "us": 0.0})
        k["launches"] += 1
        k["us"] = round(k["us"] + l["us"], 3)
    g = [l for l in launches if "mma_flop_issued" in l]
    gemm_us = sum(l["us"] for l in g)
    doc = {"source": src, "launches": len(launches), "total_us_serialised": round(sum(l["us"] for l in launches), 2),
           "gemm_launches": len(g), "gemm_us_serialised": round(gemm_us, 2),
           "gemm_mma_tflops_issued_overall": round(sum(l["mma_flop_issued"] for l in g) / (gemm_us * 1e-6) / 1e12, 2)
           if gemm_us else None,
           "gemm_tensor_pipe_frac_median": sorted(l["tensor_pipe_frac_of_2250tf"] for l in g)[len(g) // 2] if g else None,
           "gemm_tensor_pipe_frac_max": max((l["tensor_pipe_frac_of_2250tf"] for l in g), default=None),
           "by_kernel": kinds, "per_launch": launches}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in doc.items() if k != "per_launch"}, indent=1))


if __name__ == "__main__":
    main()
