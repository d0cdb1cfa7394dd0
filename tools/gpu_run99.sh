cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zzf
timeout 900 python -m pytest tests/test_gpu_pairscore.py -q -p no:cacheprovider -rf -k "gaussian" > gpurun_out/r01zzf/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zzf/pytest.log
