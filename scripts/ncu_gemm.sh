# Source-level stall sampling of a few mid-network GEMM launches (ResNet-50 b1).
# usage: bash scripts/ncu_gemm.sh <tag> [cache-control: all|none]
tag=${1:-r2k}; cc=${2:-none}
mkdir -p gpurun_out
timeout 600 ncu --section WarpStateStats --section SourceCounters --section SpeedOfLight --warp-sampling-interval 0 \
  --import-source on --clock-control none --cache-control $cc -k regex:gemm_tc_kernel --launch-skip 300 --launch-count 4 \
  -f -o gpurun_out/${tag}_gemm python scripts/time_forward.py resnet50 1 > gpurun_out/${tag}_ncu.log 2>&1
tail -3 gpurun_out/${tag}_ncu.log
