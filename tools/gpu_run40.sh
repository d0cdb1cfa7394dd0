cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/p40.log 2>&1; echo "rc=$?" >> gpurun_out/p40.log
timeout 300 python tools/steady_sweep.py > gpurun_out/steady40.log 2>&1
timeout 1200 python tools/config_runs.py 5 3 > gpurun_out/cfg5.log 2>&1; echo rc5=$? >> gpurun_out/cfg5.log
