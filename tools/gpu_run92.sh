cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zza
timeout 900 python -m pytest tests/test_gpu_updates.py tests/test_io.py -q -p no:cacheprovider -rf > gpurun_out/r01zza/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01zza/pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r01zza/bench.log 2>&1; echo "rc=$?" >> gpurun_out/r01zza/bench.log
