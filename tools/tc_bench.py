"""Config 2 exhaustive screen (N=1e4, M=1000, 5e7 pairs): tensor-core vs CUDA-core."""
import json, os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
import paper_2401_01404_b200 as P
import oracle_lib as O
n, M = 10000, 1000
m = P.Model(n, M, P.NRG_ISING, O.ising_lambda(n, M))
m.generate_ising(mean_deg=4.0, seed=2)
nodes = np.arange(n, dtype=np.int32)
for state in ("empty", "after 2 sweeps"):
    if state != "empty":
        for it in range(2):
            m.gcd_iteration(it, kappa=2.0, seed=2)
    for tc in (True, False, True):
        if tc: os.environ.pop("NRG_NO_TC", None)
        else: os.environ["NRG_NO_TC"] = "1"
        m.begin_generation(); m.reset_counters()
        m.timer_start()
        ids, d, sw, ch = m.find_knn(P.NRG_EXACT, 8, nodes, exhaustive=True)
        ms = m.timer_stop()
        ph = m.phase_times(); ks = m.kernel_stats()
        print(json.dumps({"state": state, "tc": tc, "knn_exhaustive_ms": round(ms, 2), "score_ms": round(ph["score"], 2),
                          "k2_ms": round(ks["k2_ms"], 2), "k2_pairs": ks["k2_pairs"], "tc_launches": ks["tc_launches"],
                          "pairs": n * (n - 1) // 2}), flush=True)
