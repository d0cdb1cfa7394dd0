cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01t
timeout 900 python -m pytest tests/test_gpu_updates.py tests/test_io.py tests/test_gpu_dropin.py tests/test_gpu_pairscore.py -q -p no:cacheprovider -rf -x > gpurun_out/r01t/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01t/pytest.log
timeout 600 python tools/e2e_parts.py > gpurun_out/r01t/e2e.log 2>&1; echo "rc=$?" >> gpurun_out/r01t/e2e.log
