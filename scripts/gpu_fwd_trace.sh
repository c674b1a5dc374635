#!/bin/bash
# Forward timing (graph replay) per arch + per-CTA GEMM phase trace of the
# diagnostic build: bash scripts/gpu_fwd_trace.sh <tag> [archs...]
tag=$1; shift
archs=${@:-resnet50 vgg16 alexnet vgg19}
mkdir -p gpurun_out
for a in $archs; do
  echo "$(timeout 300 python scripts/time_forward.py $a 1 2>&1 | tail -1)" >> gpurun_out/${tag}_fwd.log
done
for a in ${TRACE_ARCHS:-resnet50}; do
  TRIMS_LIB=paper_1811_09732_b200/variants/libtrims_gtrace.so timeout 300 python scripts/gemm_trace.py $a 1 > gpurun_out/${tag}_gtrace_$a.jsonl 2>&1
done
cat gpurun_out/${tag}_fwd.log
