cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01h
timeout 600 python tools/timeline.py gpurun_out/r01h/timeline.json > gpurun_out/r01h/timeline.log 2>&1; echo "rc=$?" >> gpurun_out/r01h/timeline.log
