cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sweep_once.py > gpurun_out/sweep_once.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches30.csv python tools/sweep_once.py > gpurun_out/ncu30.log 2>&1
echo rc=$?
