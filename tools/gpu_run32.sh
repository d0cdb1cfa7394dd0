cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_k1.py > gpurun_out/ab32.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/p32.log 2>&1; echo "rc=$?" >> gpurun_out/p32.log
