cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01c
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c/launches_steady.csv python tools/steady_sweep.py > gpurun_out/r01c/ncu_launch.log 2>&1
echo launches rc=$?
for spec in "ising_screen_small_kernel:5:k1s" "knn_gather_kernel:3:gather" "knn_gather_bits_kernel:3:gatherbits" "knn_merge_warp_kernel:3:mergewarp" "knn_merge_kernel:3:merge"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o gpurun_out/r01c/$name -f python tools/steady_sweep.py > gpurun_out/r01c/ncu_$name.log 2>&1
  echo "$name rc=$?"
done
