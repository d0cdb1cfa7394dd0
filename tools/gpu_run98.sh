cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zze
timeout 600 python tools/c3twice.py > gpurun_out/r01zze/c3.log 2>&1
NRG_NO_GAUSS_SCREEN=1 timeout 600 python tools/c3twice.py > gpurun_out/r01zze/c3n.log 2>&1
