cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t20
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for v in "NRG_X=1" "NRG_X=1"; do env $v timeout 300 python tools/steady_sweep.py > "$O/steady_${v// /_}.$RANDOM.log" 2>&1; done
timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:snapshot_ising -s 0 -c 1 -o /tmp/kt_snap -f python tools/steady_sweep.py > /tmp/ncu_snap.log 2>&1
python tools/ncu_sum.py /tmp/kt_snap.ncu-rep > $O/snapshot.txt 2>&1
