cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01c5
NRG_DEBUG_LEVELS=1 timeout 900 python tools/c5_steady.py > gpurun_out/r01c5/levels.log 2>&1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c5/launches.csv python tools/c5_steady.py > gpurun_out/r01c5/ncu.log 2>&1
python tools/launch_shares.py gpurun_out/r01c5/launches.csv zzzz 30 > gpurun_out/r01c5/shares.txt
rm -f gpurun_out/r01c5/launches.csv
