cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01
timeout 300 python tools/tc_bench.py > gpurun_out/r01/tc_bench.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_screen_kernel -s 1 -c 1 -o gpurun_out/r01/tc_screen -f python tools/tc_bench.py > gpurun_out/r01/ncu_tc.log 2>&1
echo rc=$?
