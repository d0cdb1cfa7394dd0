cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/steady_sweep.py > gpurun_out/steady.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches35.csv python tools/steady_sweep.py > gpurun_out/ncu35.log 2>&1
echo rc=$?
