cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01g
NRG_DEBUG_LEVELS=1 timeout 600 python tools/dense_ab.py > gpurun_out/r01g/ab.log 2>&1; echo "rc=$?" >> gpurun_out/r01g/ab.log
