# forward-pass GPU pass: gemm/forward parity tests + timing A/B
tag=${1:-r01m}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gemm or forward or sharing" > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log
for v in ${VARIANTS:-A=1 TRIMS_SPLITK=0}; do
  for a in resnet50 vgg16 alexnet; do echo -n "[$v] "; env ${v//,/ } timeout 300 python scripts/time_forward.py $a 1; done
done > gpurun_out/${tag}_fwd.log 2>&1
if [ -n "$NCU" ]; then
  ncu --metrics gpu__time_duration.sum,launch__grid_size --cache-control none --clock-control none --csv --log-file gpurun_out/${tag}_fwd_launches.csv -k regex:'gemm|im2col|pool|gemv|input_prep|flatten' python scripts/prof_forward.py resnet50 1 2 > gpurun_out/${tag}_fwdprof.log 2>&1
fi
