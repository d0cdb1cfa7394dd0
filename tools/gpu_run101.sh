cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01c5b
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01c5b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01c5b/pytest.log
timeout 300 python tools/steady_sweep.py > gpurun_out/r01c5b/steady.log 2>&1
NRG_DEBUG_LEVELS=1 timeout 900 python tools/c5_steady.py > gpurun_out/r01c5b/levels.log 2>&1
timeout 1200 python tools/config_runs.py 5 4 > gpurun_out/r01c5b/cfg5.log 2>&1; echo rc5=$? >> gpurun_out/r01c5b/cfg5.log
