#!/bin/bash
# Forward times (graph) for a set of (arch, batch), optionally with env:
# bash scripts/gpu_fwd_quick.sh <tag> "<ENV=..>" ...
tag=$1; shift
out=gpurun_out/${tag}_fwd_quick.log
: > $out
for rep in 1 2; do
  for cfg in "${@:-X=1}"; do
    for arch_b in "resnet50 1" "resnet50 32" "vgg16 1" "vgg16 32" "alexnet 1" "alexnet 32"; do
      echo "[$cfg $arch_b] $(env $cfg timeout 180 python scripts/time_forward.py $arch_b 2>&1 | tail -1 | grep -o '"fwd_ms_graph": [0-9.]*')" >> $out
    done
  done
done
cat $out
