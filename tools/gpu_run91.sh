cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zz
timeout 900 python bench.py > gpurun_out/r01zz/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01zz/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r01zz/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r01zz/bench_ref.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01zz/launches_steady.csv python tools/steady_sweep.py > gpurun_out/r01zz/ncu_launch.log 2>&1
timeout 600 python tools/timeline.py gpurun_out/r01zz/timeline.json > gpurun_out/r01zz/timeline.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01zz/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01zz/ncu_launch2.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ising_screen_pipe -s 3 -c 1 -o gpurun_out/r01zz/k1p -f python tools/steady_sweep.py > gpurun_out/r01zz/ncu_k1.log 2>&1
