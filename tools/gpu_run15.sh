cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sweep_once.py > gpurun_out/sweep_once.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ising_refine_kernel -s 10 -c 1 -o gpurun_out/k2_full -f python tools/sweep_once.py > gpurun_out/ncu_k2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ising_screen_kernel -s 10 -c 1 -o gpurun_out/k1_full -f python tools/sweep_once.py > gpurun_out/ncu_k1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:update_kernel -c 1 -o gpurun_out/upd_full -f python tools/sweep_once.py > gpurun_out/ncu_upd.log 2>&1
ls -la gpurun_out
