cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01r
timeout 900 python bench.py > gpurun_out/r01r/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01r/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r01r/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r01r/bench_ref.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ising_screen_small_kernel --csv --log-file gpurun_out/r01r/k1_dram.csv python tools/steady_sweep.py > gpurun_out/r01r/k1_dram.log 2>&1; echo "rc=$?" >> gpurun_out/r01r/k1_dram.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01r/launches_steady.csv python tools/steady_sweep.py > gpurun_out/r01r/ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/r01r/ncu_launch.log
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ising_screen_small_kernel -s 3 -c 1 -o gpurun_out/r01r/k1s -f python tools/steady_sweep.py > gpurun_out/r01r/ncu_k1s.log 2>&1; echo "rc=$?" >> gpurun_out/r01r/ncu_k1s.log
