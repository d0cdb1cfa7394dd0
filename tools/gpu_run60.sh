cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01v
timeout 900 python -m pytest tests/test_gpu_pairscore.py tests/test_gpu_search.py -q -p no:cacheprovider -rf -x > gpurun_out/r01v/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01v/pytest.log
for v in "NRG_K1_STAGES=2" "NRG_K1_STAGES=3" "NRG_K1_STAGES=4"; do env $v timeout 300 python tools/steady_sweep.py > gpurun_out/r01v/steady_$v.log 2>&1; done
