cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01kt
for spec in "ising_screen_pipe_kernel:1:k1" "knn_gather_warp_kernel:1:gather_warp" "knn_gather_kernel:1:gather256" "knn_gather_bits_kernel:0:gather_bits" "knn_merge_warp_kernel:1:merge_warp" "knn_merge_kernel:0:merge_cta" "update_kernel:0:update" "ising_refine_kernel:1:k2" "tc_screen_kernel:0:tc_screen" "snapshot_ising_kernel:0:snapshot" "theta_kernel:0:theta" "pair_dedup_kernel:0:pair_dedup" "resolve_rows_kernel:0:resolve" "logpost_node_kernel:0:logpost"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:$k -s $s -c 1 -o /tmp/kt_$name -f python tools/steady_sweep.py > /tmp/ncu_$name.log 2>&1
  python tools/ncu_sum.py /tmp/kt_$name.ncu-rep > gpurun_out/r01kt/$name.txt 2>&1
  ncu -i /tmp/kt_$name.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size > gpurun_out/r01kt/$name.csv 2>&1
done
