"""A config-1-sized GCD run (N=1000, M=500, 3 sweeps) exercising the dense levels, lazy K2,
tie tails, bulk set_edges and get_state; meant to run under compute-sanitizer."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
n, M = 1000, 500
m = P.Model(n, M, P.NRG_ISING, float(2 * np.sqrt(M * np.log(n))))
X = m.generate_ising(mean_deg=4.0, seed=1, burn_in=200, thin=5, want_samples=True)
m.reset_state()
for it in range(3):
    rec, c = m.gcd_iteration(it, kappa=2.0, seed=3, want_candidates=True)
th, ei, ej, w = m.get_state()
m2 = P.Model.from_samples(X, P.NRG_ISING, m.lam if hasattr(m, "lam") else float(2 * np.sqrt(M * np.log(n))))
m2.set_theta(th)
m2.set_edges(ei, ej, w)
rec2, _ = m2.gcd_iteration(3, kappa=2.0, seed=3, want_candidates=True)
print("ok", len(ei), rec["objective"], rec2["objective"])
