cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01n
timeout 600 python -m pytest tests/test_gpu_updates.py tests/test_io.py tests/test_gpu_dropin.py -q -p no:cacheprovider -rf -x > gpurun_out/r01n/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01n/pytest.log
timeout 600 python tools/e2e_parts.py > gpurun_out/r01n/e2e.log 2>&1; echo "rc=$?" >> gpurun_out/r01n/e2e.log
timeout 600 python tools/timeline.py gpurun_out/r01n/timeline.json > gpurun_out/r01n/timeline.log 2>&1; echo "rc=$?" >> gpurun_out/r01n/timeline.log
