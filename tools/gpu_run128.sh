cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t18
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in "NRG_X=1" "NRG_X=1"; do env $v timeout 300 python tools/steady_sweep.py > "$O/steady_${v// /_}.$RANDOM.log" 2>&1; done
NRG_DEBUG_ALLOC=1 timeout 900 python tools/config_runs.py 5 5 > $O/cfg5.log 2> $O/cfg5.err; echo "rc=$?" >> $O/cfg5.log
