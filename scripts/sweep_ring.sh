#!/bin/bash
# TMA ring geometry sweep for the transform kernel (stage KB, depth, CTAs/SM).
out=${1:-gpurun_out/sweep_ring.log}
for cfg in "32 3 2" "16 6 2" "16 12 1" "32 6 1" "8 12 2" "64 3 1" "16 4 3" "8 8 3"; do
  set -- $cfg
  for a in resnet50 vgg16; do
    TRIMS_TMA_STAGE_KB=$1 TRIMS_TMA_STAGES=$2 TRIMS_TMA_CTAS=$3 python scripts/prof_transform.py $a 3 | sed "s/^/kb=$1 st=$2 ctas=$3 /" >> $out 2>&1
  done
done
for a in resnet50 vgg16; do TRIMS_CVT_PATH=direct TRIMS_PERM_PATH=direct python scripts/prof_transform.py $a 3 | sed "s/^/direct /" >> $out; done
