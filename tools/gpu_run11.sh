cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_k1.py > gpurun_out/ab_new.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest11.log
