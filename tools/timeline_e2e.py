"""GPU timeline of one e2e step of bench.py (config 4): upload the bit-packed samples and
the state S_W, one GCD sweep with candidates, download the state -- device busy time, the
operations outside the sweep and the largest idle gaps."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2401_01404_b200 as P

N, M = 100000, 1000
m = P.Model(N, M, P.NRG_ISING, float(2 * np.sqrt(M * np.log(N))))
Xh = m.generate_ising(mean_deg=5.0, seed=1, want_samples=True)
Xpin = torch.from_numpy(np.packbits(Xh > 0, axis=1, bitorder="little")).pin_memory().numpy()
m.reset_state()
for it in range(5):
    m.gcd_iteration(it, kappa=2.0, seed=1)
th, ei, ej, w = m.get_state()
for warm in range(2):
    m.upload_spins_packed(Xpin)
    m.set_theta(th)
    m.set_edges(ei, ej, w)
    m.gcd_iteration(5, kappa=2.0, seed=1, want_candidates=True)
    m.get_state()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    m.timer_start()
    m.upload_spins_packed(Xpin)
    m.set_theta(th)
    m.set_edges(ei, ej, w)
    m.gcd_iteration(5, kappa=2.0, seed=1, want_candidates=True)
    m.get_state()
    ms = m.timer_stop()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline_e2e.json"
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
busy = sum(e["dur"] for e in k)
span = k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]
print(f"e2e step ms (events) {ms:.2f}; ops {len(k)}; busy {busy / 1e3:.2f} ms; span {span / 1e3:.2f} ms")
print("first 25 ops:")
t0 = k[0]["ts"]
for e in k[:25]:
    print(f"  {(e['ts'] - t0) / 1e3:8.3f} ms {e['dur'] / 1e3:7.3f} ms  {e['name'][:90]}")
print("last 25 ops:")
for e in k[-25:]:
    print(f"  {(e['ts'] - t0) / 1e3:8.3f} ms {e['dur'] / 1e3:7.3f} ms  {e['name'][:90]}")
gaps = sorted(((b["ts"] - a["ts"] - a["dur"], a["name"][:50], b["name"][:50]) for a, b in zip(k, k[1:])), reverse=True)
print("largest gaps:")
for g, a, b in gaps[:15]:
    print(f"  {g / 1e3:7.3f} ms  {a} -> {b}")
