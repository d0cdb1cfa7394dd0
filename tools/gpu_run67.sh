cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zb
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r01zb/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zb/pytest.log
for i in 1 2; do NRG_DEBUG_UPD=1 NRG_DEBUG_TAIL=1 timeout 300 python tools/steady_sweep.py > gpurun_out/r01zb/steady$i.log 2>&1; done
