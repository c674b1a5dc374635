#!/bin/bash
# Persistent-GEMM A/B on the forward (TRIMS_PERSIST=0/1/2), batch 1 and 32:
# bash scripts/gpu_persist_ab.sh <tag>
tag=$1
mkdir -p gpurun_out
out=gpurun_out/${tag}_persist_ab.log
: > $out
for rep in 1 2; do
  for arch_b in "vgg16 1" "vgg16 32" "resnet50 32" "resnet50 1" "alexnet 1" "vgg19 1"; do
    for m in 0 1 2; do
      echo "[TRIMS_PERSIST=$m $arch_b] $(TRIMS_PERSIST=$m timeout 180 python scripts/time_forward.py $arch_b 2>&1 | tail -1 | grep -o '"fwd_ms_graph": [0-9.]*')" >> $out
    done
  done
done
cat $out
