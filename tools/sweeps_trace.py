"""Per-sweep device time and phases of the first config-4 sweeps."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
N, M = 100000, 1000
m = P.Model(N, M, P.NRG_ISING, float(2 * np.sqrt(M * np.log(N))))
m.generate_ising(mean_deg=5.0, seed=1)
m.reset_state()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    m.reset_counters(); m.timer_start()
    m.gcd_iteration(it, kappa=2.0, seed=1)
    ms = m.timer_stop()
    ks = m.kernel_stats()
    print(json.dumps({"sweep": it, "ms": round(ms, 1), "tail_rounds": ks["tail_rounds"], "flushes": ks["cache_flushes"],
                      "phases": {k: round(v, 1) for k, v in m.phase_times().items()}}), flush=True)
