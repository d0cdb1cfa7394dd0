"""Debug: the mixed edges + random pairs batch of test_config1_after_gcd_iteration_vs_checker."""
import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O
from paper_2401_01404_b200 import _lib as gpu
from test_gpu_pairscore import _config1
X, lam = _config1(seed=2, n=600, M=300)
n, M = X.shape
ref = O.CpuModel("orc", X, 0, lam)
ref.reconstruct_gcd(kappa=2.0, max_iters=1, seed=9)
th, ei, ej, w = ref.get_state()
dev = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
dev.set_theta(th); dev.set_edges(ei, ej, w)
rng = np.random.default_rng(1)
ri, rj = rng.integers(0, n, 6000), rng.integers(0, n, 6000)
keep = ri != rj
i = np.concatenate([ei, ri[keep]]); j = np.concatenate([ej, rj[keep]])
ref.begin_generation()
d_ref = ref.distance(0, i, j)
for rep in range(3):
    d_dev = dev.distance(gpu.NRG_EXACT, i, j)
    rel = np.abs(d_dev - d_ref) / np.abs(d_ref)
    bad = np.nonzero(rel > 1e-6)[0]
    print("rep", rep, "bad", len(bad), bad[:10])
    for k in bad[:6]:
        a, b = min(i[k], j[k]), max(i[k], j[k])
        dup = np.nonzero((np.minimum(i, j) == a) & (np.maximum(i, j) == b))[0]
        print("  ", k, i[k], j[k], d_dev[k], d_ref[k], "dups", dup, d_dev[dup])
    dev.begin_generation()
# single-pair queries
k = 561
for rep in range(2):
    print("single", dev.distance(gpu.NRG_EXACT, i[k:k+1], j[k:k+1]), d_ref[k]); dev.begin_generation()
