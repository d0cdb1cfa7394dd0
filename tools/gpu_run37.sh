cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sweep_once.py > gpurun_out/sweep_once.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:knn_gather_kernel -s 21 -c 1 -o gpurun_out/gather2_full -f python tools/sweep_once.py > gpurun_out/ncu37.log 2>&1
echo rc=$?
