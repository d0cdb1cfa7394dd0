cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_k1.py > gpurun_out/ab_pool.log 2>&1
NRG_SYNC_ALLOC=1 timeout 600 python tools/ab_k1.py > gpurun_out/ab_sync.log 2>&1
