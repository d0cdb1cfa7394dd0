cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01za
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r01za/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01za/pytest.log
for i in 1 2; do timeout 300 python tools/steady_sweep.py > gpurun_out/r01za/steady$i.log 2>&1; done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01za/launches_steady.csv python tools/steady_sweep.py > gpurun_out/r01za/ncu_launch.log 2>&1
