cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r01x/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01x/pytest.log
timeout 600 python tools/config_runs.py 3 4 > gpurun_out/r01x/cfg3.log 2>&1; echo rc=$? >> gpurun_out/r01x/cfg3.log
timeout 1200 python tools/config_runs.py 5 3 > gpurun_out/r01x/cfg5.log 2>&1; echo rc=$? >> gpurun_out/r01x/cfg5.log
timeout 300 python tools/tc_bench.py > gpurun_out/r01x/tc_bench.log 2>&1; echo rc=$? >> gpurun_out/r01x/tc_bench.log
