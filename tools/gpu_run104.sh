cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01v7
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r01v7/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01v7/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01v7/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r01v7/smoke.log
timeout 900 python bench.py > gpurun_out/r01v7/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01v7/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r01v7/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r01v7/bench_ref.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_steady.csv python tools/steady_sweep.py > gpurun_out/r01v7/ncu_launch.log 2>&1
python tools/launch_shares.py /tmp/launches_steady.csv zzzz 45 > gpurun_out/r01v7/launches_steady.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01v7/ncu_launch2.log 2>&1
python tools/launch_shares.py /tmp/launches.csv gibbs_persistent 40 > gpurun_out/r01v7/launches_bench.txt
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ising_screen_pipe_kernel --csv --log-file gpurun_out/r01v7/k1_dram.csv python tools/steady_sweep.py > gpurun_out/r01v7/k1_dram.log 2>&1
timeout 600 python tools/timeline.py /tmp/timeline.json > gpurun_out/r01v7/timeline.log 2>&1
timeout 600 python tools/config_runs.py 3 4 > gpurun_out/r01v7/cfg3.log 2>&1
