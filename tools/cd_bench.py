"""reconstruct_cd at config 1 (N=1000, M=500): device vs the compiled reference (first sweep)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
import paper_2401_01404_b200 as P
import oracle_lib as O
X, _ = O.gen_ising(1000, 500, seed=1)
lam = O.ising_lambda(1000, 500)
dev = P.Model.from_samples(X.astype(np.int8), P.NRG_ISING, lam)
t = time.perf_counter(); recs, conv = dev.reconstruct_cd(max_iters=30); td = time.perf_counter() - t
print(json.dumps({"device_sweeps": len(recs), "converged": conv, "device_s": round(td, 3),
                  "sweep_s": [round(float(x), 4) for x in recs["seconds"]],
                  "objective": [float(x) for x in recs["objective"]][-3:]}), flush=True)
ref = O.CpuModel("ref", X, 0, lam)
t = time.perf_counter(); rr, cr = ref.reconstruct_cd(max_iters=1); tr = time.perf_counter() - t
print(json.dumps({"reference_first_sweep_s": round(tr, 2), "device_first_sweep_s": round(float(recs["seconds"][0]), 4),
                  "obj_ref": float(rr["objective"][0]), "obj_dev": float(recs["objective"][0])}), flush=True)
