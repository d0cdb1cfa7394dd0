cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01t8
timeout 600 python tools/timeline.py /tmp/timeline.json > gpurun_out/r01t8/timeline.log 2>&1
