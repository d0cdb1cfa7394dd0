cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_k1.py > gpurun_out/ab_new.log 2>&1
cd tools/v2lib && timeout 600 python ../ab_k1.py > ../../gpurun_out/ab_v2.log 2>&1; cd ../..
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
