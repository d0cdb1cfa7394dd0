cd $GRAFT_REPO_ROOT
O=gpurun_out/r01t26
mkdir -p $O
for v in "NRG_X=1" "NRG_LIST_ORDER_TICKETS=1" "NRG_X=1" "NRG_LIST_ORDER_TICKETS=1"; do env $v timeout 300 python tools/steady_sweep.py > "$O/steady_${v// /_}.$RANDOM.log" 2>&1; done
