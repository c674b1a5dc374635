#!/bin/bash
# A/B of transform variants on resnet50 / vgg16: env switches and variant
# builds of the library (paper_1811_09732_b200/variants/*.so via TRIMS_LIB).
V=paper_1811_09732_b200/variants
VARIANTS=${VARIANTS:-"A=1 TRIMS_TMA_STAGES=2 TRIMS_TMA_STAGE_KB=72 TRIMS_TMA_STAGE_KB=96,TRIMS_TMA_STAGES=2 TRIMS_TMA_STAGE_KB=112,TRIMS_TMA_STAGES=2 TRIMS_TMA_STAGE_KB=48,TRIMS_TMA_STAGES=4 TRIMS_TMA_STAGE_KB=32,TRIMS_TMA_STAGES=6 TRIMS_CVT_PATH=direct"}
for arch in resnet50 vgg16; do
  for v in $VARIANTS $(for f in $V/*.so; do [ -e "$f" ] && echo "TRIMS_LIB=$f"; done) \
           $(for f in $V/*.so; do [ -e "$f" ] && echo "TRIMS_LIB=$f,TRIMS_TMA_STAGES=2"; done); do
    echo -n "$arch [$v] "
    env ${v//,/ } python scripts/prof_transform.py $arch 3 3
  done
done
