cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zf
timeout 900 python bench.py > gpurun_out/r01zf/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01zf/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01zf/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01zf/ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/r01zf/ncu_launch.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ising_screen_pipe_kernel --csv --log-file gpurun_out/r01zf/k1_dram.csv python tools/steady_sweep.py > gpurun_out/r01zf/k1_dram.log 2>&1
