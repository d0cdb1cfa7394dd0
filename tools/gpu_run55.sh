cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01q
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01q/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01q/pytest.log
timeout 600 python tools/sweeps_trace.py 7 > gpurun_out/r01q/trace.log 2>&1; echo "rc=$?" >> gpurun_out/r01q/trace.log
timeout 600 python tools/timeline.py gpurun_out/r01q/timeline.json > gpurun_out/r01q/timeline.log 2>&1; echo "rc=$?" >> gpurun_out/r01q/timeline.log
