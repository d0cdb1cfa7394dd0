cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01f
timeout 600 python -m pytest tests/test_gpu_search.py tests/test_gpu_updates.py -q -p no:cacheprovider -rf -x > gpurun_out/r01f/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01f/pytest.log
NRG_DEBUG_LEVELS=1 timeout 600 python tools/dense_ab.py > gpurun_out/r01f/ab.log 2>&1; echo "rc=$?" >> gpurun_out/r01f/ab.log
NRG_DENSE_N=16384 timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"knn_gather_bits|knn_merge_kernel" -s 0 -c 4 -o gpurun_out/r01f/dense -f python tools/steady_sweep.py > gpurun_out/r01f/ncu_dense.log 2>&1
