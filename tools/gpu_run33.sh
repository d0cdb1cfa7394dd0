cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench33.log 2> gpurun_out/bench33.err || { echo "bench failed"; tail -20 gpurun_out/bench33.err; exit 1; }
