#!/bin/bash
# Same-box A/B of two builds: steady config-4 sweeps alternating between the current
# library and paper_2401_01404_b200/libnetrec_b200_prev.so (NRG_LIB), N rounds.
n=${1:-4}
for i in $(seq $n); do
  echo -n "new  "; python tools/steady_sweep.py | tail -1
  echo -n "prev "; NRG_LIB=$PWD/paper_2401_01404_b200/libnetrec_b200_prev.so python tools/steady_sweep.py | tail -1
done
