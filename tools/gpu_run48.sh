cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01i
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01i/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01i/pytest.log
timeout 600 python tools/timeline.py gpurun_out/r01i/timeline.json > gpurun_out/r01i/timeline.log 2>&1; echo "rc=$?" >> gpurun_out/r01i/timeline.log
timeout 600 python tools/dense_ab.py > gpurun_out/r01i/ab.log 2>&1; echo "rc=$?" >> gpurun_out/r01i/ab.log
