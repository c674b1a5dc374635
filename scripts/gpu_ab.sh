# quick GPU pass: ingest/store parity tests, transform A/B, one ncu capture
tag=${1:-r01h}; what=${2:-"tests ab ncu"}
mkdir -p gpurun_out
for w in $what; do case $w in
tests) timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "ingest or store or peer or smoke or integration" > gpurun_out/${tag}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${tag}_pytest.log ;;
ab) VARIANTS=${VARIANTS:-"A=1 TRIMS_TILE_SCHED=dynamic TRIMS_TMA_STAGES=2,TRIMS_TMA_STAGE_KB=96 TRIMS_TMA_STAGE_KB=48,TRIMS_TMA_STAGES=4"} timeout 600 bash scripts/ab_transform.sh > gpurun_out/${tag}_ab.log 2>&1 ;;
ncu) timeout 600 ncu --set full --clock-control none --import-source on -k regex:transform -c 1 -f -o gpurun_out/${tag}_transform python scripts/prof_transform.py resnet50 1 > gpurun_out/${tag}_ncu.log 2>&1 ;;
esac; done
