cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zp
timeout 900 python -m pytest tests/test_gpu_search.py -q -p no:cacheprovider -rf > gpurun_out/r01zp/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zp/pytest.log
for v in "NRG_MERGE_BUF=256" "NRG_MERGE_BUF=1024" "NRG_MERGE_BUF=2048" "NRG_MERGE_BUF=512"; do env $v timeout 300 python tools/steady_sweep.py > gpurun_out/r01zp/steady_$v.log 2>&1; done
