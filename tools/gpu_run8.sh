cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_dropin.py -q --timeout 300 -p no:cacheprovider -rf -x > gpurun_out/pytest8a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest8a.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -rf > gpurun_out/pytest8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest8.log
