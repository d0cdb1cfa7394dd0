cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01zx
for v in "NRG_UPD_NT=256" "NRG_UPD_NT=128"; do env $v timeout 300 python tools/sweeps_trace.py 4 > gpurun_out/r01zx/trace_$v.log 2>&1; env $v timeout 300 python tools/cd_bench.py > gpurun_out/r01zx/cd_$v.log 2>&1; done
