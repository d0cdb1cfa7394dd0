"""Structure of the update chains of config-4 sweeps: node frequencies, run lengths."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
N, M = 100000, 1000
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
m.generate_ising(mean_deg=5.0, seed=1)
for it in range(3):
    rec, cand = m.gcd_iteration(it, kappa=2.0, seed=1000 + it, want_candidates=True)
    i, j, d = cand["i"], cand["j"], cand["dist"]
    cnt = np.bincount(np.concatenate([i, j]), minlength=N)
    top = np.argsort(-cnt)[:8]
    last = np.zeros(N, np.int64); depth = np.zeros(len(i), np.int64)
    for p in range(len(i)):
        dd = max(last[i[p]], last[j[p]]) + 1; depth[p] = dd; last[i[p]] = dd; last[j[p]] = dd
    th, ei, ej, w = m.get_state()
    print("iter", it, "depth", depth.max(), "top nodes", top.tolist(), "counts", cnt[top].tolist(),
          "nodes touched", int((cnt > 0).sum()), "edges", len(ei), "theta range", float(th.min()), float(th.max()),
          "dist range", float(d.min()), float(d.max()), "phase", {k: round(v, 1) for k, v in m.phase_times().items()}, "tail_rounds", m.kernel_stats()["tail_rounds"], flush=True)
    m.reset_counters()
