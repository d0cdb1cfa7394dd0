cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t29
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in "NRG_X=1" "NRG_X=1" "NRG_X=1"; do env $v timeout 300 python tools/steady_sweep.py > "$O/steady_${v// /_}.$RANDOM.log" 2>&1; done
