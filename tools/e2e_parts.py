"""Wall time of each public-API call of bench.py's e2e step (config 4, after 3 sweeps)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2401_01404_b200 as P
N, M = 100000, 1000
m = P.Model(N, M, P.NRG_ISING, float(2 * np.sqrt(M * np.log(N))))
Xh = m.generate_ising(mean_deg=5.0, seed=1, want_samples=True)
Xpin = torch.from_numpy(np.packbits((Xh > 0).astype(np.uint8), axis=1, bitorder="little")).pin_memory().numpy()
m.reset_state()
for it in range(3):
    m.gcd_iteration(it, kappa=2.0, seed=1)
th, ei, ej, w = m.get_state()
for rep in range(3):
    t = {}
    def T(name, f, *a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); t[name] = round((time.perf_counter() - t0) * 1e3, 2); return r
    T("upload", m.upload_spins_packed, Xpin)
    T("set_theta", m.set_theta, th)
    T("set_edges", m.set_edges, ei, ej, w)
    m.reset_counters()
    T("gcd_iteration", m.gcd_iteration, 3, kappa=2.0, seed=1, want_candidates=True)
    ph = {k: round(v, 1) for k, v in m.phase_times().items()}
    T("get_state", m.get_state)
    print(json.dumps({**t, "phases": ph, "phase_sum": round(sum(ph.values()), 1)}), flush=True)
m.reset_counters()
for it in range(4, 7):
    t0 = time.perf_counter(); m.reset_counters(); m.gcd_iteration(it, kappa=2.0, seed=1, want_candidates=True)
    ph = {k: round(v, 1) for k, v in m.phase_times().items()}
    print(json.dumps({"steady_gcd_iteration": round((time.perf_counter() - t0) * 1e3, 2), "phases": ph}), flush=True)
