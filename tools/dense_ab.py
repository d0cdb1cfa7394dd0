"""A/B of the dense FindBest levels on config 4: three sweeps from the empty state, then
sweep 3 re-run from the same state with NRG_DENSE_N in {0, 16384, 32768, 65535}; prints
time, phases, misses and whether the candidate lists agree."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
N, M = int(os.environ.get("AB_N", 100000)), 1000
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
m.generate_ising(mean_deg=5.0, seed=1)
m.reset_state()
os.environ["NRG_DENSE_N"] = "0"
for it in range(3):
    m.gcd_iteration(it, kappa=2.0, seed=1)
st = m.get_state()
ref = None
for dn, ratio in [(0, 4), (16384, 4), (32768, 32), (65535, 64), (0, 4), (16384, 4), (32768, 32)]:
    os.environ["NRG_DENSE_N"] = str(dn)
    os.environ["NRG_DENSE_RATIO"] = str(ratio)
    m.reset_state(); m.set_theta(st[0]); m.set_edges(st[1], st[2], st[3])
    m.reset_counters()
    m.timer_start()
    rec, cands = m.gcd_iteration(3, kappa=2.0, seed=1, want_candidates=True)
    ms = m.timer_stop()
    same = None if ref is None else bool(np.array_equal(ref, cands))
    if ref is None:
        ref = cands
    print(json.dumps({"dense_n": dn, "ratio": ratio, "ms": round(ms, 2), "same": same, **m.counters(),
                      "phases": {k: round(v, 2) for k, v in m.phase_times().items()},
                      "tc": m.kernel_stats()["tc_launches"]}), flush=True)
