#!/bin/bash
# Shared-clients leg under env settings (inherited by the client processes):
# bash scripts/gpu_mps_env.sh <tag> "<ENV=..>" ...
tag=$1; shift
mkdir -p gpurun_out
for cfg in "$@"; do
  echo "[$cfg] $(env $cfg timeout 600 python scripts/shared_clients.py 16 250 2>&1 | tail -1)" >> gpurun_out/${tag}_mps_env.log
done
python - <<PY
import json, re
for l in open("gpurun_out/${tag}_mps_env.log"):
    tag, _, js = l.partition("] ")
    try:
        d = json.loads(js)
        print(tag + "]", "mps", d["requests_per_s"], "p50", d["p50_ms"], "single", d.get("single_client_requests_per_s"),
              "ratio", d.get("aggregate_over_single_client"), "timesliced", d.get("without_mps", {}).get("requests_per_s"))
    except Exception as e:
        print(tag, "ERR", js[:300])
PY
