cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sweep_once.py > gpurun_out/sweep_once.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ising_screen_kernel -s 1 -c 1 -o gpurun_out/k1big_full -f python tools/sweep_once.py > gpurun_out/ncu_k1big.log 2>&1
echo rc=$?
