cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01mw
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_updates.py -q -p no:cacheprovider -rf > gpurun_out/r01mw/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01mw/pytest.log
for i in 1 2 3; do timeout 300 python tools/steady_sweep.py > gpurun_out/r01mw/steady$i.log 2>&1; done
