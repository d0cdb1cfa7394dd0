cd $GRAFT_REPO_ROOT
O=gpurun_out/r01v10
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
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ising_screen_pipe_kernel --csv --log-file $O/k1_dram.csv python tools/steady_sweep.py > $O/k1_dram.log 2>&1
python tools/k1_traffic.py $O/k1_dram.csv $O/steady.json $O/k1_traffic.json > $O/k1_traffic.log 2>&1
for spec in "ising_screen_pipe_kernel:2:k1_4bit" "update_kernel:0:update" "theta_kernel:0:theta"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o /tmp/kt_$name -f python tools/steady_sweep.py > /tmp/ncu_$name.log 2>&1
  python tools/ncu_sum.py /tmp/kt_$name.ncu-rep > $O/$name.txt 2>&1
done
timeout 600 python tools/timeline.py /tmp/timeline.json > $O/timeline.log 2>&1
timeout 600 python tools/e2e_parts.py > $O/e2e.log 2>&1
timeout 600 python tools/config_runs.py 3 4 > $O/cfg3.log 2>&1
timeout 900 python tools/config_runs.py 5 5 > $O/cfg5.log 2>&1
