# cold-path A/B: store tests, then bench --quick with and without the prestage overlap
tag=${1:-r01t}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "store or ingest or smoke or sharing or integration" > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log
for v in A=1 TRIMS_PRESTAGE=0; do
  echo "[$v]"; env $v timeout 600 python bench.py --quick --no-cpu-baseline --steps 10 --warmup 3
done > gpurun_out/${tag}_cold.log 2> gpurun_out/${tag}_cold.err
