cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zs
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"knn_gather_kernel" -s 1 -c 1 -o gpurun_out/r01zs/gather32 -f python tools/steady_sweep.py > gpurun_out/r01zs/ncu1.log 2>&1
