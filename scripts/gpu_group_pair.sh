# Paired group GEMMs (AlexNet conv4/conv5): forward tests, then AlexNet graph
# timing A/B TRIMS_GROUP_PAIR=0/1 alternated:  bash scripts/gpu_group_pair.sh <tag>
tag=${1:-r4i}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_forward.py -q -x -p no:cacheprovider -rA > gpurun_out/${tag}_fwd_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_fwd_tests.log
bash scripts/gpu_fwd_env.sh ${tag} alexnet TRIMS_GROUP_PAIR=0 TRIMS_GROUP_PAIR=1 TRIMS_GROUP_PAIR=0 TRIMS_GROUP_PAIR=1
