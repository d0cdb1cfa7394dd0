cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01p
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01p/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01p/pytest.log
timeout 600 python tools/sweeps_trace.py 7 > gpurun_out/r01p/trace.log 2>&1; echo "rc=$?" >> gpurun_out/r01p/trace.log
timeout 600 python tools/timeline.py gpurun_out/r01p/timeline.json > gpurun_out/r01p/timeline.log 2>&1; echo "rc=$?" >> gpurun_out/r01p/timeline.log
