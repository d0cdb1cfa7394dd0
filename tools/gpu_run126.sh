cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t16
mkdir -p $O
TIMELINE_CFG=5 timeout 900 python tools/timeline.py /tmp/timeline5.json > $O/timeline5.log 2>&1; echo "rc=$?" >> $O/timeline5.log
