#!/bin/bash
# One GPU-box pass: gpu tests, a bench line, the ncu launch list of the bench
# command, and one full ncu capture of the transform kernel.
# usage: bash scripts/gpu_round.sh <tag> [tests|bench|reference|multi|ncu ...]
tag=${1:-r01}; shift
what=${@:-tests bench ncu}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
for w in $what; do
  case $w in
    tests)
      timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
      echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err ;;
    reference)
      timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.jsonl 2> gpurun_out/${tag}_bench_reference.err ;;
    multi)
      TRIMS_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --quick \
        > gpurun_out/${tag}_bench_shared2.jsonl 2> gpurun_out/${tag}_bench_shared2.err ;;
    ncu)
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
        --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --quick --no-cpu-baseline \
        > gpurun_out/${tag}_ncu_bench.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:transform -c 2 \
        -f -o gpurun_out/${tag}_transform python scripts/prof_transform.py resnet50 1 \
        > gpurun_out/${tag}_ncu_transform.log 2>&1 ;;
    fwdncu)
      ARCHS="resnet50 vgg16 alexnet vgg19" timeout 1500 bash scripts/gpu_fwd_ncu.sh ${tag}
      for a in resnet50 vgg16 alexnet vgg19; do
        python scripts/ncu_forward_summary.py gpurun_out/${tag}_fwd_${a}.csv gpurun_out/${tag}_ncu_forward_${a}.json > /dev/null 2>&1
      done ;;
    refmaps)  # which shared objects the reference arm's process maps (must be oracle/_ref only)
      timeout 900 python -c "
import runpy, sys, os
sys.argv = ['bench.py', '--impl', 'reference', '--quick', '--steps', '3', '--warmup', '3']
try:
    runpy.run_path('bench.py', run_name='__main__')
finally:
    maps = open('/proc/self/maps').read().split()
    sos = sorted({m for m in maps if m.endswith('.so') and ('repo' in m or 'graft' in m or 'oracle' in m)})
    print('REFERENCE_ARM_MAPS', sos)
" > gpurun_out/${tag}_refmaps.log 2>&1 ;;
  esac
done
ls -la gpurun_out
