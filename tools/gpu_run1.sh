cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt; lscpu | head -20 >> gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py --config config2 --steps 2 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c2.log
