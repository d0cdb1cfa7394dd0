cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01k4e
timeout 600 python -m pytest tests/test_gpu_pairscore.py tests/test_gpu_search.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01k4e/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01k4e/pytest.log
for v in "NRG_X=1" "NRG_K1_STAGES=3" "NRG_K1_STAGES=4" "NRG_X=1" "NRG_K1_STAGES=3"; do env $v timeout 300 python tools/steady_sweep.py > "gpurun_out/r01k4e/steady_${v// /_}.$RANDOM.log" 2>&1; done
