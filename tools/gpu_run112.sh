cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01k4n
for spec in "ising_screen_pipe_kernel:2:k1_4bit" "ising_refine_cta_kernel:1:k2_cta"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o /tmp/kt_$name -f python tools/steady_sweep.py > /tmp/ncu_$name.log 2>&1
  python tools/ncu_sum.py /tmp/kt_$name.ncu-rep > gpurun_out/r01k4n/$name.txt 2>&1
  ncu -i /tmp/kt_$name.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__func_cache_config > gpurun_out/r01k4n/$name.csv 2>&1
  ncu -i /tmp/kt_$name.ncu-rep --page source --csv --print-source sass > /tmp/src_$name.csv 2>&1; head -c 3000000 /tmp/src_$name.csv > gpurun_out/r01k4n/src_$name.csv
done
