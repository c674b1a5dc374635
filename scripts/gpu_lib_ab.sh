#!/bin/bash
# Forward A/B between library builds, alternated on one box:
# bash scripts/gpu_lib_ab.sh <tag> <variant.so> [archs...]  (variant under paper_1811_09732_b200/variants/)
tag=$1; var=$2; shift 2
archs=${@:-resnet50 alexnet vgg16}
mkdir -p gpurun_out
for rep in 1 2 3; do
  for a in $archs; do
    echo "[base] $(timeout 300 python scripts/time_forward.py $a 1 2>&1 | tail -1)" >> gpurun_out/${tag}_lib_ab.log
    echo "[$var] $(TRIMS_LIB=paper_1811_09732_b200/variants/$var timeout 300 python scripts/time_forward.py $a 1 2>&1 | tail -1)" >> gpurun_out/${tag}_lib_ab.log
  done
done
if [ -n "$GTRACE" ]; then
  TRIMS_LIB=paper_1811_09732_b200/variants/$GTRACE timeout 300 python scripts/gemm_trace.py resnet50 1 > gpurun_out/${tag}_gtrace_var.jsonl 2>&1
fi
grep -o '^\[[^]]*\].*"arch": "[a-z0-9]*"\|"fwd_ms_graph": [0-9.]*' gpurun_out/${tag}_lib_ab.log | paste - - 
