cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t17
mkdir -p $O
NRG_DEBUG_ALLOC=1 NRG_DEBUG_LEVELS=1 timeout 900 python tools/config_runs.py 5 4 > $O/cfg5.log 2> $O/cfg5.err; echo "rc=$?" >> $O/cfg5.log
nvidia-smi --query-gpu=memory.total,memory.used --format=csv >> $O/cfg5.log
