cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/ab_k1.py > gpurun_out/ab_new.log 2>&1
cd tools/v1lib && timeout 600 python ../ab_k1.py > ../../gpurun_out/ab_old.log 2>&1
