cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zc
timeout 900 python -m pytest tests/test_gpu_search.py -q -p no:cacheprovider -rf > gpurun_out/r01zc/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zc/pytest.log
for v in "NRG_BITS_MAXN=16384" "NRG_BITS_MAXN=32768" "NRG_BITS_MAXN=16384" "NRG_BITS_MAXN=32768"; do env $v timeout 300 python tools/steady_sweep.py > gpurun_out/r01zc/steady_$v.$RANDOM.log 2>&1; done
