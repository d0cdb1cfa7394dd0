import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2401_01404_b200 as P
N, M = 100000, 1000
m = P.Model(N, M, P.NRG_ISING, float(2 * np.sqrt(M * np.log(N))))
m.generate_ising(mean_deg=5.0, seed=1)
m.reset_state()
def edges():
    th, ei, ej, w = m.get_state()
    return dict(zip((ei.astype(np.int64) << 32 | ej).tolist(), w.tolist())), th.copy()
check = {5, 10, 25, 50, 100, 200, 400, 800}
for it in range(801):
    if it in check:
        e0, t0 = edges()
    m.gcd_iteration(it, kappa=2.0, seed=1)
    if it in check:
        e1, t1 = edges()
        ch = [k for k in set(e0) | set(e1) if e0.get(k) != e1.get(k)]
        nodes = set()
        for k in ch:
            nodes.add(k >> 32); nodes.add(k & 0xffffffff)
        print(json.dumps({"sweep": it, "edges_changed": len(ch), "nodes_touched": len(nodes),
                          "theta_changed": int((t0 != t1).sum()), "edges": len(e1)}), flush=True)
