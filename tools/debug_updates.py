"""Debug helper: set_edges with a duplicated pair (golden ising_state) on the GPU."""
import os
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2401_01404_b200 as P
g = dict(np.load("tests/golden/ising_state.npz"))
for serial in (False, True):
    if serial:
        os.environ["NRG_DEBUG_SERIAL"] = "1"
    m = P.Model.from_samples(g["X"], 0, float(g["lam"]))
    m.set_theta(g["theta_in"])
    m.set_edges(g["e_i"], g["e_j"], g["e_w"])
    d = np.abs(m.get_sums() - g["sums"]).max(axis=1)
    print("serial" if serial else "parallel", "rows wrong:", np.flatnonzero(d > 1e-12), d.max(), flush=True)
    th, ei, ej, w = m.get_state()
    print(" W equal:", np.array_equal(w, g["state_w"]), flush=True)
