cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_k1.py > gpurun_out/ab_new.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest10.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/ncu_launch.log
