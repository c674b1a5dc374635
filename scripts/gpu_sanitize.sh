#!/bin/bash
# compute-sanitizer over the GPU paths: bash scripts/gpu_sanitize.sh <tag>
tag=${1:-r3w}
mkdir -p gpurun_out
out=gpurun_out/${tag}_sanitize.log
: > $out
run() {  # run <tool> <label> <pytest -k expr | smoke>
  echo "### compute-sanitizer --tool $1: $2" >> $out
  if [ "$3" = smoke ]; then
    timeout 900 compute-sanitizer --tool $1 --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> $out 2>&1
  else
    timeout 1500 compute-sanitizer --tool $1 --error-exitcode 9 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$3" >> $out 2>&1
  fi
  echo "exit $?" >> $out
}
run memcheck smoke smoke
run memcheck gemm "test_gemm"
run memcheck forward_modes "test_forward_executor_modes and resnet50"
run memcheck forward_e2e "test_forward_end_to_end and (resnet50-1 or alexnet-1)"
run memcheck direct_io "direct_io"
run racecheck gemm_split "test_gemm_split_k and (49-512-4608 or 196-256-1024)"
run synccheck gemm_split "test_gemm_split_k and 49-512-4608"
grep -E "^###|ERROR SUMMARY|^exit|passed|failed" $out
