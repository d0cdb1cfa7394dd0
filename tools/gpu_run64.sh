cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01z
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_updates.py tests/test_gpu_sharded.py -q -p no:cacheprovider -rf > gpurun_out/r01z/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01z/pytest.log
for i in 1 2; do timeout 300 python tools/steady_sweep.py > gpurun_out/r01z/steady$i.log 2>&1; done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01z/launches_steady.csv python tools/steady_sweep.py > gpurun_out/r01z/ncu_launch.log 2>&1
