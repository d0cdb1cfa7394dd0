"""A/B timing helper: config-4 sweeps, per-step wall/device time and K1 per-launch time."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
N, M = 100000, 1000
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
m.generate_ising(mean_deg=5.0, seed=1)
for mode in ("reset", "reset", "reset", "reset", "reset"):
    m.reset_counters()
    t = time.perf_counter(); m.timer_start()
    m.reset_state()
    rec, _ = m.gcd_iteration(1, kappa=2.0, seed=1000)
    dev = m.timer_stop(); wall = time.perf_counter() - t
    k = m.kernel_stats(); ph = m.phase_times()
    print(json.dumps({"wall_ms": round(wall * 1e3, 1), "dev_ms": round(dev, 1),
                      "k1_ms_per_launch": round(k["k1_ms"] / max(1, k["k1_launches"]), 3),
                      "k1_total": round(k["k1_ms"], 1), "k2_total": round(k["k2_ms"], 1),
                      "phases": {a: round(b, 1) for a, b in ph.items()}}), flush=True)
