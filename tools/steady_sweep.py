"""Config-4 reconstruction: 3 sweeps, then sweep 3 inside cudaProfilerStart/Stop (ncu
--profile-from-start off captures only the steady-state sweep)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2401_01404_b200 as P
N, M = 100000, 1000
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
m.generate_ising(mean_deg=5.0, seed=1)
m.reset_state()
for it in range(3):
    m.gcd_iteration(it, kappa=2.0, seed=1)
m.reset_counters()
if os.environ.get("NRG_DEBUG_ALLOC"):
    print("=== measured sweep", file=sys.stderr, flush=True)
torch.cuda.cudart().cudaProfilerStart()
m.timer_start()
m.gcd_iteration(3, kappa=2.0, seed=1)
ms = m.timer_stop()
torch.cuda.cudart().cudaProfilerStop()
print(json.dumps({"ms": ms, **m.kernel_stats(), **m.counters(), "phases": m.phase_times()}), flush=True)
