cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01c5d
timeout 1200 python tools/config_runs.py 5 5 > gpurun_out/r01c5d/cfg5.log 2>&1; echo rc5=$? >> gpurun_out/r01c5d/cfg5.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r01c5d/bench.log 2>&1; echo rc5=$? >> gpurun_out/r01c5d/cfg5_32k.log
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> gpurun_out/r01c5d/cfg5.log
