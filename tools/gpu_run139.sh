cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t27
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_updates.py tests/test_gpu_dropin.py -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in "NRG_X=1" "NRG_UPD_NT=128" "NRG_X=1" "NRG_UPD_NT=128"; do env $v timeout 300 python tools/steady_sweep.py > "$O/steady_${v// /_}.$RANDOM.log" 2>&1; done
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
NRG_FB_LEVEL_ORDER=1 timeout 900 python bench.py --no-cpu-baseline > $O/bench_level.log 2>&1; echo "rc=$?" >> $O/bench_level.log
