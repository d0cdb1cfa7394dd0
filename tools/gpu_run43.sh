cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01d
timeout 600 python -m pytest tests/test_gpu_search.py tests/test_gpu_updates.py -q -p no:cacheprovider -rf -x > gpurun_out/r01d/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01d/pytest.log
NRG_DEBUG_LEVELS=1 timeout 600 python tools/dense_ab.py > gpurun_out/r01d/ab.log 2>&1; echo "rc=$?" >> gpurun_out/r01d/ab.log
