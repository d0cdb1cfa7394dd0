"""DRAM traffic per screened pair of K1 (both passes) from an ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum capture of every
ising_screen_pipe_kernel launch of one steady-state sweep (tools/steady_sweep.py).
usage: k1_traffic.py capture.csv steady_sweep.json out.json"""
import csv, json, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
st = json.load(open(sys.argv[2]))
agg = {}
for r in rows:
    name = r[4]
    tag = "4-bit" if (", true>" in name or ", 1>(" in name) else "8-bit"
    a = agg.setdefault(tag, {"launches": set(), "read": 0.0, "write": 0.0, "ms": 0.0})
    a["launches"].add(r[0])
    unit, val = r[13], float(r[14].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "ns": 1e-6, "us": 1e-3, "ms": 1.0}[unit]
    if r[12] == "dram__bytes_read.sum": a["read"] += val * scale
    elif r[12] == "dram__bytes_write.sum": a["write"] += val * scale
    elif r[12] == "gpu__time_duration.sum": a["ms"] += val * scale
pairs = st["k1_pairs"]
out = {"kernel": "ising_screen_pipe_kernel (K1: 4-bit pass over every pair, 8-bit recheck pass)",
       "capture": sys.argv[1], "pairs": pairs}
tot = 0.0
for tag, a in agg.items():
    out[tag] = {"launches": len(a["launches"]), "dram_bytes_read": a["read"], "dram_bytes_write": a["write"],
                "ncu_serialized_ms": a["ms"], "dram_bytes_per_screened_pair": (a["read"] + a["write"]) / pairs}
    tot += a["read"] + a["write"]
out["dram_bytes_per_pair"] = tot / pairs
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out, indent=1))
