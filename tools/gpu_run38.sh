cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01
timeout 300 python tools/steady_sweep.py > gpurun_out/r01/steady.log 2>&1 || exit 1
for spec in "ising_screen_kernel:5:k1" "ising_refine_kernel:3:k2" "knn_gather_kernel:10:gather" "knn_merge_kernel:10:merge" "update_kernel:0:update" "theta_kernel:0:theta" "snapshot_ising_kernel:0:snapshot"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/r01/$name -f python tools/steady_sweep.py > gpurun_out/r01/ncu_$name.log 2>&1
  echo "$name rc=$?"
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01/launches_steady.csv python tools/steady_sweep.py > gpurun_out/r01/ncu_launch.log 2>&1
echo launches rc=$?
