cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01k4d
timeout 600 python -m pytest tests/test_gpu_pairscore.py tests/test_gpu_search.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01k4d/pytest16.log 2>&1; echo "rc=$?" >> gpurun_out/r01k4d/pytest16.log
NRG_K1_G4=8 timeout 600 python -m pytest tests/test_gpu_pairscore.py tests/test_gpu_search.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01k4d/pytest8.log 2>&1; echo "rc=$?" >> gpurun_out/r01k4d/pytest8.log
NRG_K1_G4=4 timeout 600 python -m pytest tests/test_gpu_pairscore.py tests/test_gpu_search.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01k4d/pytest4.log 2>&1; echo "rc=$?" >> gpurun_out/r01k4d/pytest4.log
for v in "NRG_K1_G4=16" "NRG_K1_G4=8" "NRG_K1_G4=4" "NRG_K1_G4=8 NRG_K1_STAGES=3" "NRG_K1_G4=16" "NRG_K1_G4=8" "NRG_K1_G4=4"; do env $v timeout 300 python tools/steady_sweep.py > "gpurun_out/r01k4d/steady_${v// /_}.$RANDOM.log" 2>&1; done
