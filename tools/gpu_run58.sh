cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01s
for i in 1 2; do timeout 300 python tools/steady_sweep.py > gpurun_out/r01s/steady$i.log 2>&1; done
