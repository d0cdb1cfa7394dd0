import os, sys
sys.path.insert(0, os.getcwd())
os.environ["NRG_DEBUG_TAIL"] = "1"
import numpy as np
import paper_2401_01404_b200 as P
N, M = 100000, 1000
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
m.generate_ising(mean_deg=5.0, seed=1)
rec, cand = m.gcd_iteration(0, kappa=2.0, seed=1000, want_candidates=True)
d = cand["dist"]; tail = int(np.sum(d == d[-1]))
print("tail length", tail, "first tail pair", cand[len(d) - tail], file=sys.stderr)
