cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/p14.log 2>&1; echo "rc=$?" >> gpurun_out/p14.log
for r in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_pairscore.py tests/test_gpu_updates.py -q -p no:cacheprovider -rf 2>&1 | tail -1; done > gpurun_out/p14_file.log
