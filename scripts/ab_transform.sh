#!/bin/bash
# A/B of transform variants (env switches) on resnet50 / vgg16.
for arch in resnet50 vgg16; do
  for v in "A=1" "TRIMS_TRANSFORM_SERIAL=1" "TRIMS_PERM_ONEPASS=1" "TRIMS_TMA_STAGES=2" "TRIMS_TMA_STAGE_KB=32 TRIMS_TMA_STAGES=4" "TRIMS_TMA_STAGE_KB=48"; do
    echo -n "$arch [$v] "
    env $v python scripts/prof_transform.py $arch 3 3
  done
done
