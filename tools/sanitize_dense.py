"""A small GCD run (N=4000, M=300, kappa 6 so the deep levels have wide rows) exercising the
dense levels' bit-set gathers, short lists, covered levels, the persistent tensor-core
screen and the radix select; meant to run under compute-sanitizer."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
n, M = 4000, 300
m = P.Model(n, M, P.NRG_ISING, float(2 * np.sqrt(M * np.log(n))))
m.generate_ising(mean_deg=4.0, seed=1, burn_in=100, thin=3)
m.reset_state()
for it in range(2):
    rec, c = m.gcd_iteration(it, kappa=6.0, seed=3, want_candidates=True)
print("ok", rec["objective"], m.kernel_stats()["tc_launches"])
