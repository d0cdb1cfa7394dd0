cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/p34.log 2>&1; echo "rc=$?" >> gpurun_out/p34.log
timeout 900 python bench.py > gpurun_out/bench34.log 2> gpurun_out/bench34.err || { echo "bench failed"; tail -20 gpurun_out/bench34.err; exit 1; }
