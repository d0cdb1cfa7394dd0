cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t9
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_k1_passes.py -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/config_runs.py 5 5 > $O/cfg5.log 2>&1; echo "rc=$?" >> $O/cfg5.log
