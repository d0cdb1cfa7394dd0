cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01e2
timeout 600 python tools/e2e_parts.py > gpurun_out/r01e2/e2e.log 2>&1; echo "rc=$?" >> gpurun_out/r01e2/e2e.log
