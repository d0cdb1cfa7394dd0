cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zzd
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r01zzd/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zzd/pytest.log
timeout 600 python tools/config_runs.py 3 4 > gpurun_out/r01zzd/cfg3.log 2>&1
NRG_NO_GAUSS_SCREEN=1 timeout 600 python tools/config_runs.py 3 4 > gpurun_out/r01zzd/cfg3_noscreen.log 2>&1
