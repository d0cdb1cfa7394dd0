import json, math, os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
import paper_2401_01404_b200 as P
for rep in range(2):
    n, M = 10000, 1000
    m = P.Model(n, M, P.NRG_GAUSSIAN, 1.0)
    X = m.generate_gaussian(degree=4, amp=0.2, burn_in=1000, thin=10, seed=3, want_samples=True)
    var = float(np.mean(X.var(axis=1))); lam = 2.0 * math.sqrt(M * math.log(n)) * var
    m.close(); m = P.Model.from_samples(X, P.NRG_GAUSSIAN, lam)
    for it in range(2):
        m.reset_counters(); m.timer_start(); rec, _ = m.gcd_iteration(it, kappa=2.0, seed=7); ms = m.timer_stop()
        print(rep, it, round(ms,1), {k: round(v,1) for k,v in m.phase_times().items()}, m.kernel_stats()["k2_pairs"], flush=True)
