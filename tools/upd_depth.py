"""Dependency depth of the update list of one config-4 sweep (critical path of apply_updates)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
N, M = 100000, 1000
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
m.generate_ising(mean_deg=5.0, seed=1)
for it in range(2):
    m.reset_counters()
    rec, cand = m.gcd_iteration(it, kappa=2.0, seed=1000 + it, want_candidates=True)
    i, j = cand["i"], cand["j"]
    last = np.full(N, 0, np.int64)
    depth = np.zeros(len(i), np.int64)
    for p in range(len(i)):
        d = max(last[i[p]], last[j[p]]) + 1
        depth[p] = d
        last[i[p]] = d
        last[j[p]] = d
    ph = m.phase_times()
    print("iter", it, "updates", len(i), "depth", depth.max(), "update_ms", round(ph["update"], 1),
          "us/level", round(1e3 * ph["update"] / depth.max(), 2), "rec", rec, flush=True)
