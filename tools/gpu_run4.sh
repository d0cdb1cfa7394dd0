cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest4.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"ising_screen|ising_finalize|ising_newton|update_kernel|knn_gather" -s 40 -c 5 -o gpurun_out/prof_r01 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
