cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/p13_$r.log 2>&1; echo "rc=$?" >> gpurun_out/p13_$r.log
done
for r in 1 2 3 4 5; do timeout 300 python -m pytest tests/test_gpu_pairscore.py -q -p no:cacheprovider -rf 2>&1 | tail -2; done > gpurun_out/p13_file.log
