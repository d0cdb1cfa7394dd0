cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zw
for v in "NRG_UPD_NT=256" "NRG_UPD_NT=128" "NRG_UPD_NT=256" "NRG_UPD_NT=128"; do env $v timeout 300 python tools/steady_sweep.py > gpurun_out/r01zw/steady_$v.$RANDOM.log 2>&1; done
NRG_UPD_NT=128 timeout 600 python -m pytest tests/test_gpu_updates.py -q -p no:cacheprovider -rf > gpurun_out/r01zw/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zw/pytest.log
