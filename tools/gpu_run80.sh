cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zo
timeout 900 python bench.py > gpurun_out/r01zo/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01zo/bench.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01zo/launches_steady.csv python tools/steady_sweep.py > gpurun_out/r01zo/ncu_launch.log 2>&1
timeout 600 python tools/timeline.py gpurun_out/r01zo/timeline.json > gpurun_out/r01zo/timeline.log 2>&1
timeout 1200 python tools/config_runs.py 5 3 > gpurun_out/r01zo/cfg5.log 2>&1; echo rc5=$? >> gpurun_out/r01zo/cfg5.log
timeout 600 python tools/config_runs.py 3 4 > gpurun_out/r01zo/cfg3.log 2>&1
