cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zm
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r01zm/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zm/pytest.log
for i in 1 2; do timeout 300 python tools/steady_sweep.py > gpurun_out/r01zm/steady$i.log 2>&1; done
timeout 600 python tools/timeline.py gpurun_out/r01zm/timeline.json > gpurun_out/r01zm/timeline.log 2>&1
