cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t10
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in "NRG_X=1" "NRG_KNN_NO_SPEC_U=1" "NRG_X=1" "NRG_KNN_NO_SPEC_U=1"; do env $v timeout 300 python tools/steady_sweep.py > "$O/steady_${v// /_}.$RANDOM.log" 2>&1; done
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 900 python tools/config_runs.py 5 4 > $O/cfg5.log 2>&1; echo "rc=$?" >> $O/cfg5.log
