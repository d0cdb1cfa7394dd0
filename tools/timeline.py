"""GPU timeline of one steady-state config-4 sweep through torch.profiler (CUPTI): kernel
busy time vs wall, and the largest idle gaps with the kernels either side of them."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2401_01404_b200 as P
CFG5 = os.environ.get("TIMELINE_CFG") == "5"  # config 5 (N = 1e6, M = 200, power law) instead
N, M = (1000000, 200) if CFG5 else (100000, 1000)
lam = float(2 * np.sqrt(M * np.log(N)))
m = P.Model(N, M, P.NRG_ISING, lam)
if CFG5:
    m.generate_ising_powerlaw(gamma=2.5, dmin=2, w_sigma=0.2, th_sigma=0.1, burn_in=1000, thin=10, seed=5)
else:
    m.generate_ising(mean_deg=5.0, seed=1)
m.reset_state()
PRE = int(os.environ.get("TIMELINE_SWEEP", "3"))  # sweeps before the profiled one
for it in range(PRE):
    m.gcd_iteration(it, kappa=2.0, seed=1)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    m.timer_start()
    m.gcd_iteration(PRE, kappa=2.0, seed=1)
    ms = m.timer_stop()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.json"
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
rt = [e for e in ev if e.get("cat") == "cuda_runtime"]
busy = sum(e["dur"] for e in k)
span = (k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]) if k else 0
print(f"sweep ms (events) {ms:.2f}; kernels+copies {len(k)}; busy {busy/1e3:.2f} ms; span {span/1e3:.2f} ms")
gaps = []
for a, b in zip(k, k[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    gaps.append((g, a["name"][:50], b["name"][:50]))
gaps.sort(reverse=True)
tot = sum(g for g, _, _ in gaps if g > 0)
print(f"idle total {tot/1e3:.2f} ms over {sum(1 for g, _, _ in gaps if g > 5)} gaps > 5us")
hist = {}
for g, a, b in gaps:
    key = (a.split('<')[0].split('(')[0], b.split('<')[0].split('(')[0])
    hist.setdefault(key, [0, 0.0])
    hist[key][0] += 1
    hist[key][1] += max(g, 0)
for key, (n_, t) in sorted(hist.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{t/1e3:8.2f} ms {n_:5d}x  {key[0]:40s} -> {key[1]}")
print("largest single gaps:")
for g, a, b in gaps[:10]:
    print(f"    {g/1e3:8.2f} ms  {a:50s} -> {b}")
rc = {}
for e in rt:
    rc.setdefault(e["name"], [0, 0.0])
    rc[e["name"]][0] += 1
    rc[e["name"]][1] += e["dur"]
print("runtime API:")
for name, (n_, t) in sorted(rc.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{t/1e3:8.2f} ms {n_:6d}x {name}")
agg = {}
for e in k:
    n = e["name"].replace("void ", "").replace("nrg::", "")
    if "cub::" in n:
        n = "cub::" + n.split("::")[-1].split("<")[0][:24] + ("<TriKey>" if "TriKey" in n or "Key128" in n else "")
    else:
        full = n.split("(")[0]
        n = full.split("<")[0] + (("[4-bit]" if "true>" in full else "[8-bit]") if "screen_pipe" in full else "")
    agg.setdefault(n, [0, 0.0])
    agg[n][0] += 1
    agg[n][1] += e["dur"]
print("kernels:")
for n, (c_, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{t/1e3:8.3f} ms {c_:5d} {n}")
