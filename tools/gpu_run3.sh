cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NRG_DEBUG_UPDATES=1 timeout 120 python tools/debug_updates.py > gpurun_out/dbg_upd.log 2>&1
