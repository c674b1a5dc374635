#!/bin/bash
# Forward timing under several env settings: bash scripts/gpu_fwd_env.sh <tag> <arch> "<ENV=..>" "<ENV=..>" ...
tag=$1; arch=$2; shift 2
mkdir -p gpurun_out
for cfg in "$@"; do
  for rep in 1 2; do
    echo "[$cfg] $(env $cfg timeout 300 python scripts/time_forward.py $arch 1 2>&1 | tail -1)" >> gpurun_out/${tag}_fwd_env.log
  done
done
cat gpurun_out/${tag}_fwd_env.log
