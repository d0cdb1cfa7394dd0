cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01k
NRG_DEBUG_LEVELS=1 timeout 600 python tools/sweeps_trace.py 8 > gpurun_out/r01k/trace.log 2>&1; echo "rc=$?" >> gpurun_out/r01k/trace.log
