cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/upd_depth2.py > gpurun_out/depth4.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/p21.log 2>&1; echo "rc=$?" >> gpurun_out/p21.log
