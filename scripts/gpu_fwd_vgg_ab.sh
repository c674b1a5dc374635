#!/bin/bash
# VGG forward A/B over env settings: bash scripts/gpu_fwd_vgg_ab.sh <tag> "<ENV=..>" ...
tag=$1; shift
out=gpurun_out/${tag}_vgg_ab.log
: > $out
for rep in 1 2 3; do
  for cfg in "$@"; do
    for arch_b in "vgg16 1" "vgg16 32" "vgg19 1"; do
      echo "[$cfg $arch_b] $(env $cfg timeout 180 python scripts/time_forward.py $arch_b 2>&1 | tail -1 | grep -o '"fwd_ms_graph": [0-9.]*')" >> $out
    done
  done
done
cat $out
