"""Debug: existing-edge scores after one GCD iteration (dist vs live vs checker)."""
import sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
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
ref.begin_generation()
d_ref = ref.distance(0, ei, ej)
d_dev = dev.distance(gpu.NRG_EXACT, ei, ej)
w_ref, g_ref, _ = ref.optimize_edge(ei, ej)
w_dev, g_dev, _ = dev.optimize_edge(ei, ej)
base = dev.log_posterior()
gd = -(d_dev + base)
bad = np.nonzero(np.abs(gd - g_ref) > 1e-4 * np.maximum(1, np.abs(g_ref)))[0]
badl = np.nonzero(np.abs(g_dev - g_ref) > 1e-4 * np.maximum(1, np.abs(g_ref)))[0]
print("edges", len(ei), "bad cached", len(bad), "bad live", len(badl))
for k in list(bad[:8]) + list(badl[:4]):
    print(k, ei[k], ej[k], "wcur", w[k], "ref", w_ref[k], g_ref[k], "live", w_dev[k], g_dev[k], "cached gain", gd[k])
