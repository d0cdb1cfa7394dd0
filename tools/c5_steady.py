"""Config 5 (Ising N=1e6, M=200, power-law): 2 sweeps, then sweep 2 inside
cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import json, math, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2401_01404_b200 as P
n, M = 1_000_000, 200
m = P.Model(n, M, P.NRG_ISING, 2.0 * math.sqrt(M * math.log(n)))
m.generate_ising_powerlaw(gamma=2.5, dmin=2, w_sigma=0.2, th_sigma=0.1, burn_in=1000, thin=10, seed=5)
for it in range(2):
    m.gcd_iteration(it, kappa=2.0, seed=7)
m.reset_counters()
torch.cuda.cudart().cudaProfilerStart()
m.timer_start()
m.gcd_iteration(2, kappa=2.0, seed=7)
ms = m.timer_stop()
torch.cuda.cudart().cudaProfilerStop()
print(json.dumps({"ms": ms, **m.kernel_stats(), **m.counters(), "phases": m.phase_times()}), flush=True)
