"""One config-4 GCD sweep (for ncu captures): prints kernel stats."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
N, M = 100000, 1000
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
m.generate_ising(mean_deg=5.0, seed=1)
m.reset_counters()
m.reset_state()
m.gcd_iteration(1, kappa=2.0, seed=1000)
print(json.dumps({**m.kernel_stats(), **m.counters()}), flush=True)
