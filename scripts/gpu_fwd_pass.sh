#!/bin/bash
# GEMM/forward parity tests, then forward timing + GEMM phase trace:
# bash scripts/gpu_fwd_pass.sh <tag>
tag=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gemm or forward" > gpurun_out/${tag}_pytest.log 2>&1
echo "exit $?" >> gpurun_out/${tag}_pytest.log
tail -3 gpurun_out/${tag}_pytest.log
bash scripts/gpu_fwd_trace.sh $tag ${ARCHS:-resnet50 vgg16 alexnet vgg19}
