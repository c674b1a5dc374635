# ncu per-layer metrics of one eager forward per model (K7/K8 evidence):
#   bash scripts/gpu_fwd_ncu.sh <tag>
tag=${1:-r2a}
M=$(python -c "import sys; sys.path.insert(0,'scripts'); import ncu_forward_summary as s; print(s.FWD_METRICS)")
for a in ${ARCHS:-resnet50 vgg16 alexnet}; do
  ncu --metrics $M --clock-control none -k regex:'gemm|im2col|pool|gemv|input_prep|flatten' --csv --log-file gpurun_out/${tag}_fwd_${a}.csv \
      python scripts/prof_forward.py $a 1 1 > gpurun_out/${tag}_fwd_${a}.log 2>&1
done
