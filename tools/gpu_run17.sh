cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/sweep_once.py > gpurun_out/sweep_once.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ising_refine_kernel --csv --log-file gpurun_out/k2_list.csv python tools/sweep_once.py > gpurun_out/ncu_k2list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ising_refine_kernel -s 27 -c 1 -o gpurun_out/k2big_full -f python tools/sweep_once.py > gpurun_out/ncu_k2big.log 2>&1
