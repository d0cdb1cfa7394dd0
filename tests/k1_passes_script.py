"""Helper for test_gpu_k1_passes.py (run in a subprocess so the A/B switches, read once
per process, take effect): scores a fixed pair list at a converging state and saves the
distances.  usage: k1_passes_script.py out.npz"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2401_01404_b200 as P  # noqa: E402

N, M = 3000, 1000
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
m.generate_ising(mean_deg=5.0, seed=11)
m.reset_state()
cands = None
for it in range(2):
    _, cands = m.gcd_iteration(it, kappa=2.0, seed=3, want_candidates=True)
th, ei, ej, w = m.get_state()
rng = np.random.default_rng(5)
ri = rng.integers(0, N, 200000)
rj = rng.integers(0, N, 200000)
keep = ri != rj
# the last sweep's FindBest candidates: the pairs nearest the kink threshold
si, sj = cands["i"], cands["j"]
I = np.concatenate([ei, ej[:5000], ri[keep], np.asarray(si, np.int32)]).astype(np.int32)
J = np.concatenate([ej, ei[:5000], rj[keep], np.asarray(sj, np.int32)]).astype(np.int32)
d = m.distance(P.NRG_EXACT, I, J)
np.savez(sys.argv[1], i=I, j=J, d=d, edges=len(ei))
print("pairs", len(I), "edges", len(ei), "unpruned", int((d != d.max()).sum()))
