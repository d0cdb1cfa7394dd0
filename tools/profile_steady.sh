#!/bin/bash
# ncu evidence for one steady-state config-4 GCD sweep (tools/steady_sweep.py: sweeps
# 0-2 unprofiled, sweep 3 inside cudaProfilerStart/Stop).  Usage (on the GPU box):
#   bash tools/profile_steady.sh <out_dir>
# 1. the plain run (must exit 0 before any ncu run of the same command);
# 2. the launch list with per-launch time, DRAM bytes and executed instructions;
# 3. ncu --set full of the first four K1 launches of the sweep (4-bit + 8-bit passes).
set -e
out=${1:-gpurun_out/prof}
mkdir -p "$out"
python tools/steady_sweep.py > "$out/steady_plain.json"
ncu --profile-from-start off --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__cycles_active.avg \
    --csv --log-file "$out/steady_launches.csv" python tools/steady_sweep.py > "$out/steady_ncu.json"
ncu --profile-from-start off --clock-control none --set full --import-source on \
    -k regex:ising_screen_pipe_kernel -s 0 -c 4 -o "$out/k1_full" python tools/steady_sweep.py > "$out/k1_ncu.json"
