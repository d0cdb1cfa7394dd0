cd $GRAFT_REPO_ROOT
O=gpurun_out/r01v11
mkdir -p $O
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_steady.csv python tools/steady_sweep.py > $O/ncu_launch.log 2>&1
python tools/launch_shares.py /tmp/launches_steady.csv zzzz 45 > $O/launches_steady.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch2.log 2>&1
python tools/launch_shares.py /tmp/launches.csv gibbs_persistent 40 > $O/launches_bench.txt
timeout 600 python tools/config_runs.py 3 4 > $O/cfg3.log 2>&1
timeout 900 python tools/config_runs.py 5 4 > $O/cfg5.log 2>&1
