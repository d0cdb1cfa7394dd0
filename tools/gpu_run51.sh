cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01l
NRG_DEBUG_LEVELS=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r01l/bench_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/r01l/bench_dbg.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r01l/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01l/bench.log
