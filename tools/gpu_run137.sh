cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t25
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 600 python tools/e2e_parts.py > $O/e2e.log 2>&1
