cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zzc
timeout 900 python -m pytest tests/test_gpu_exhaustive_tc.py tests/test_gpu_search.py -q -p no:cacheprovider -rf > gpurun_out/r01zzc/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zzc/pytest.log
for i in 1 2; do timeout 300 python tools/steady_sweep.py > gpurun_out/r01zzc/steady$i.log 2>&1; done
timeout 300 python tools/tc_bench.py > gpurun_out/r01zzc/tc_bench.log 2>&1
