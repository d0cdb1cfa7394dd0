"""GCD sweeps on configs 3 (Gaussian N=1e4, M=1000) and 5 (Ising N=1e6, M=200) with the
device generators: generation time, per-sweep device time and phases."""
import json, math, os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
import paper_2401_01404_b200 as P
which = sys.argv[1] if len(sys.argv) > 1 else "3"
if which == "3":
    n, M = 10000, 1000
    m = P.Model(n, M, P.NRG_GAUSSIAN, 1.0)
    t = time.perf_counter(); X = m.generate_gaussian(degree=4, amp=0.2, burn_in=1000, thin=10, seed=3, want_samples=True)
    gen = time.perf_counter() - t
    var = float(np.mean(X.var(axis=1)))
    lam = 2.0 * math.sqrt(M * math.log(n)) * var   # Gaussian lambda = 2 sqrt(M ln N) * mean sample variance
    m.close()
    m = P.Model.from_samples(X, P.NRG_GAUSSIAN, lam)
else:
    n, M = 1_000_000, 200
    lam = 2.0 * math.sqrt(M * math.log(n))
    m = P.Model(n, M, P.NRG_ISING, lam)
    t = time.perf_counter(); m.generate_ising_powerlaw(gamma=2.5, dmin=2, w_sigma=0.2, th_sigma=0.1, burn_in=1000, thin=10, seed=5)
    gen = time.perf_counter() - t
print(json.dumps({"config": which, "n": n, "M": M, "lambda": lam, "gen_s": round(gen, 2)}), flush=True)
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    m.reset_counters(); m.timer_start()
    rec, _ = m.gcd_iteration(it, kappa=2.0, seed=7)
    ms = m.timer_stop()
    print(json.dumps({"sweep": it, "ms": round(ms, 1), "pairs": m.counters()["misses"], "edges": int(len(m.get_state()[1])),
                      "objective": float(rec["objective"]), "flushes": m.kernel_stats()["cache_flushes"], "phases": {k: round(v, 1) for k, v in m.phase_times().items()}}), flush=True)
