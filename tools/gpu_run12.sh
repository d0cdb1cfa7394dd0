cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pairscore.py -q -p no:cacheprovider -rf > gpurun_out/p12a.log 2>&1; echo "rc=$?" >> gpurun_out/p12a.log
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_pairscore.py -q -p no:cacheprovider -x > gpurun_out/p12b.log 2>&1; echo "rc=$?" >> gpurun_out/p12b.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/dbg_mixed.py > gpurun_out/p12c.log 2>&1; echo "rc=$?" >> gpurun_out/p12c.log
