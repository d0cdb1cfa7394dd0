cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01b
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r01b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01b/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01b/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r01b/smoke.log
timeout 900 python bench.py > gpurun_out/r01b/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01b/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01b/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r01b/bench_ref.log
timeout 300 python tools/steady_sweep.py > gpurun_out/r01b/steady.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01b/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r01b/ncu_launch.log
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ising_screen_kernel -s 5 -c 1 -o gpurun_out/r01b/k1 -f python tools/steady_sweep.py > gpurun_out/r01b/ncu_k1.log 2>&1; echo "k1 rc=$?" >> gpurun_out/r01b/ncu_k1.log
