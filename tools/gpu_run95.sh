cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zzb
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r01zzb/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zzb/pytest.log
for i in 1 2; do timeout 300 python tools/steady_sweep.py > gpurun_out/r01zzb/steady$i.log 2>&1; done
