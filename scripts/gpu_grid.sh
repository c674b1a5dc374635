#!/bin/bash
# Grid runs: bash scripts/gpu_grid.sh <tag> <catalog> [requests]  (time-sliced and MPS workers)
tag=$1; cat=${2:-tiny}; reqs=${3:-200}
mkdir -p gpurun_out
for mode in nomps mps; do
  timeout ${GRID_TIMEOUT:-900} python scripts/grid.py gpurun_out/${tag}_grid_${cat}_${mode}.json $reqs $cat $mode ${WORLDS:-1,2,4} ${CONCS:-1,4} > /dev/null 2> gpurun_out/${tag}_grid_${cat}_${mode}.err
  echo "$mode exit $?"
done
python - <<PY
import json, glob
for f in sorted(glob.glob("gpurun_out/${tag}_grid_${cat}_*.json")):
    d = json.load(open(f)); print(f, "mps", d["mps"])
    print("gpus frac conc ok speedup pen_mean pen_med open_ms hit peer")
    for c in d["cells"]:
        print(c["gpus"], c["fraction"], c["concurrency"], c["ok"], c["geomean_p95_speedup"], c["mean_latency_penalty_vs_warm"],
              c["median_latency_penalty_vs_warm"], c["open_ms_p50"], c["fast_hit_rate"], c["peer_hits"], c["error"])
PY
