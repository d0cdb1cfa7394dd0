cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01k4c
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01k4c/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01k4c/pytest.log
for v in "NRG_X=1" "NRG_K1_STAGES=3" "NRG_X=1" "NRG_K1_STAGES=3"; do env $v timeout 300 python tools/steady_sweep.py > gpurun_out/r01k4c/steady_$v.$RANDOM.log 2>&1; done
