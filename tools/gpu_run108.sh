cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01k2
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r01k2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r01k2/pytest.log
for v in 0 1 2 3 4 0 1; do NRG_K2_CTA=$v timeout 300 python tools/steady_sweep.py > gpurun_out/r01k2/steady_$v.$RANDOM.log 2>&1; done
