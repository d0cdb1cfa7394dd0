cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01ud
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01ud/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01ud/pytest.log
for v in "NRG_X=1" "NRG_UPD_NO_SNAP=1" "NRG_X=1" "NRG_UPD_NO_SNAP=1"; do env $v timeout 300 python tools/steady_sweep.py > "gpurun_out/r01ud/steady_${v// /_}.$RANDOM.log" 2>&1; done
