cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01c5c
timeout 1200 python tools/config_runs.py 5 5 > gpurun_out/r01c5c/cfg5.log 2>&1; echo rc5=$? >> gpurun_out/r01c5c/cfg5.log
NRG_DENSE_N=32768 timeout 1200 python tools/config_runs.py 5 5 > gpurun_out/r01c5c/cfg5_32k.log 2>&1; echo rc5=$? >> gpurun_out/r01c5c/cfg5_32k.log
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> gpurun_out/r01c5c/cfg5.log
