#!/bin/bash
# GEMM/forward correctness, forward timing and the GEMM timeline in one box call.
# usage: bash scripts/gpu_fwd_check.sh <tag> [archs...]
tag=$1; shift
archs=${@:-resnet50 vgg16 alexnet}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_forward.py -q -x -p no:cacheprovider > gpurun_out/${tag}_pytest_fwd.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest_fwd.log
tail -3 gpurun_out/${tag}_pytest_fwd.log
for a in $archs; do
  echo "$(timeout 300 python scripts/time_forward.py $a 1 2>&1 | tail -1)" >> gpurun_out/${tag}_fwd.log
done
cat gpurun_out/${tag}_fwd.log
for a in $archs; do
  TRIMS_LIB=paper_1811_09732_b200/variants/libtrims_gtrace.so timeout 300 python scripts/gemm_trace.py $a 1 > gpurun_out/${tag}_gtrace_$a.jsonl 2>&1
done
