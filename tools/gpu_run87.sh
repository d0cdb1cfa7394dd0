cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zv
timeout 900 python -m pytest tests/test_gpu_pairscore.py -q -p no:cacheprovider -rf -k wide --durations=5 > gpurun_out/r01zv/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zv/pytest.log
