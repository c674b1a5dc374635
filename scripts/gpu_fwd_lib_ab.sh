#!/bin/bash
# Same-box A/B of library builds (and env settings) on the forward:
# bash scripts/gpu_fwd_lib_ab.sh <tag> <arch> "<ENV=..>" ...   (ENV may set TRIMS_LIB=...)
tag=$1; arch=$2; shift 2
mkdir -p gpurun_out
for rep in 1 2 3; do
  for cfg in "$@"; do
    echo "[$cfg] $(env $cfg timeout 120 python scripts/time_forward.py $arch 1 2>&1 | tail -1 | grep -o '"fwd_ms_graph": [0-9.]*')" >> gpurun_out/${tag}_fwd_ab.log
  done
done
cat gpurun_out/${tag}_fwd_ab.log
