cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench23.log 2> gpurun_out/bench23.err || { echo "bench failed"; tail -20 gpurun_out/bench23.err; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches23.csv python bench.py --no-cpu-baseline > gpurun_out/ncu23.log 2>&1
echo "ncu rc=$?"
