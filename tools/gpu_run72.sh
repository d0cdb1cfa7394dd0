cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zg
for spec in "snapshot_ising_kernel:0:snap" "logpost_node_kernel:0:logpost" "theta_kernel:0:theta" "update_kernel:0:update"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/r01zg/$name -f python tools/steady_sweep.py > gpurun_out/r01zg/ncu_$name.log 2>&1
done
