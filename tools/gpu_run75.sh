cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zj
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/r01zj/memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r01zj/memcheck.log
timeout 600 python bench.py --config config2 --no-cpu-baseline > gpurun_out/r01zj/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r01zj/bench_c2.log
timeout 600 python bench.py --config config1 --no-cpu-baseline > gpurun_out/r01zj/bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/r01zj/bench_c1.log
