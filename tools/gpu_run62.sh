cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01w
NRG_K1_STAGES=3 timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ising_screen_pipe -s 3 -c 1 -o gpurun_out/r01w/k1p -f python tools/steady_sweep.py > gpurun_out/r01w/ncu.log 2>&1; echo rc=$? >> gpurun_out/r01w/ncu.log
