cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01ze
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"knn_gather_kernel" -s 7 -c 1 -o gpurun_out/r01ze/gather256 -f python tools/steady_sweep.py > gpurun_out/r01ze/ncu1.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"knn_merge_warp_kernel" -s 1 -c 1 -o gpurun_out/r01ze/mergew -f python tools/steady_sweep.py > gpurun_out/r01ze/ncu2.log 2>&1
