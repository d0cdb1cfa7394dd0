cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/steady_sweep.py > gpurun_out/steady36.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/p36.log 2>&1; echo "rc=$?" >> gpurun_out/p36.log
