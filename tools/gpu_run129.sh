cd $GRAFT_REPO_ROOT
O=gpurun_out/r01v9
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
timeout 300 python tools/steady_sweep.py > $O/steady.json 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_steady.csv python tools/steady_sweep.py > $O/ncu_launch.log 2>&1
python tools/launch_shares.py /tmp/launches_steady.csv zzzz 45 > $O/launches_steady.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch2.log 2>&1
python tools/launch_shares.py /tmp/launches.csv gibbs_persistent 40 > $O/launches_bench.txt
timeout 600 python tools/timeline.py /tmp/timeline.json > $O/timeline.log 2>&1
timeout 600 python tools/e2e_parts.py > $O/e2e.log 2>&1
