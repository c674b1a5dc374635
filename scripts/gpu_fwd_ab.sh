#!/bin/bash
# Forward A/B on one box: graph-replayed forward per arch with an env switch
# on/off, and the per-layer GEMM timeline of the trace build.
# usage: bash scripts/gpu_fwd_ab.sh <tag> <ENVVAR> [archs...]
tag=$1; var=$2; shift 2
archs=${@:-resnet50 vgg16 alexnet}
mkdir -p gpurun_out
for a in $archs; do
  for v in 0 1; do
    echo "[$var=$v] $(env $var=$v timeout 300 python scripts/time_forward.py $a 1 2>&1 | tail -1)" >> gpurun_out/${tag}_fwd_ab.log
  done
done
for a in $archs; do
  TRIMS_LIB=paper_1811_09732_b200/variants/libtrims_gtrace.so timeout 300 python scripts/gemm_trace.py $a 1 > gpurun_out/${tag}_gtrace_$a.jsonl 2>&1
done
cat gpurun_out/${tag}_fwd_ab.log
