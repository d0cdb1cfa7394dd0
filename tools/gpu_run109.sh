cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01k2s
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01k2s/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01k2s/pytest.log
for v in "NRG_X=1" "NRG_K2_WARP=1" "NRG_X=1" "NRG_K2_WARP=1"; do env $v timeout 300 python tools/steady_sweep.py > gpurun_out/r01k2s/steady_$v.$RANDOM.log 2>&1; done
