cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01j
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01j/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01j/pytest.log
timeout 600 python tools/timeline.py gpurun_out/r01j/timeline.json > gpurun_out/r01j/timeline.log 2>&1; echo "rc=$?" >> gpurun_out/r01j/timeline.log
timeout 900 python bench.py > gpurun_out/r01j/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01j/bench.log
