cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NRG_DEBUG_UPDATES=1 timeout 120 python tools/debug_updates.py > gpurun_out/dbg_upd.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf -x > gpurun_out/pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest2.log
