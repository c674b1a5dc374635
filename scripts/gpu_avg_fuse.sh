# Fused global average pool (ResNet's last conv): forward tests, then graph
# timing A/B TRIMS_AVG_FUSE=0/1 alternated:  bash scripts/gpu_avg_fuse.sh <tag>
tag=${1:-r4c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_forward.py -q -x -p no:cacheprovider -rA > gpurun_out/${tag}_fwd_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_fwd_tests.log
bash scripts/gpu_fwd_env.sh ${tag} resnet50 TRIMS_AVG_FUSE=0 TRIMS_AVG_FUSE=1 TRIMS_AVG_FUSE=0 TRIMS_AVG_FUSE=1
