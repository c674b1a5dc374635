# full gpu tests + one quick bench line
tag=${1:-r01v}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log
timeout 900 python bench.py ${BENCH_ARGS:---quick --no-cpu-baseline --steps 10 --warmup 3} > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err
