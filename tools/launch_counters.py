"""Per-kernel totals from an ncu --csv launch list with several --metrics (one row per
launch and metric): time, DRAM bytes, executed warp instructions; plus the K1 summary
(bytes and instructions per scored pair) that bench.py's roofline reads.

usage: launch_counters.py launches.csv steady_sweep.json [k1_counters.json]"""
import collections
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "cycle": 1,
        "Kcycle": 1e3, "Mcycle": 1e6, "": 1}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
st = json.load(open(sys.argv[2]))
per = collections.defaultdict(lambda: collections.defaultdict(float))
names = {}
for r in rows:
    lid, name, metric, unit, val = r[0], r[4], r[12], r[13], r[14].replace(",", "")
    try:
        v = float(val) * UNIT.get(unit, 1)
    except ValueError:
        continue
    per[lid][metric] += v
    names[lid] = name
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for lid, m in per.items():
    n = names[lid]
    short = n.split("(")[0].replace("void ", "")
    a = agg[short]
    a["launches"] += 1
    for k, v in m.items():
        a[k] += v
tot_ms = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"{'ms':>8} {'share':>6} {'n':>4} {'DRAM GB/s':>9} {'GB':>7} {'Ginst':>7}  kernel")
for k, a in sorted(agg.items(), key=lambda t: -t[1]["gpu__time_duration.sum"])[:40]:
    ms = a["gpu__time_duration.sum"]
    by = a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]
    print(f"{ms:8.3f} {100 * ms / tot_ms:5.1f}% {int(a['launches']):4d} {by / (ms / 1e3) / 1e9 if ms else 0:9.0f} "
          f"{by / 1e9:7.3f} {a['smsp__inst_executed.sum'] / 1e9:7.3f}  {k[:100]}")
print(f"total {tot_ms:.2f} ms over {len(per)} launches")
k1 = [a for k, a in agg.items() if "ising_screen_pipe_kernel" in k]
if len(sys.argv) > 3 and k1:
    pairs = st["k1_pairs"]
    ms = sum(a["gpu__time_duration.sum"] for a in k1)
    rd = sum(a["dram__bytes_read.sum"] for a in k1)
    wr = sum(a["dram__bytes_write.sum"] for a in k1)
    inst = sum(a["smsp__inst_executed.sum"] for a in k1)
    out = {"kernel": "ising_screen_pipe_kernel (K1, both passes)", "capture": sys.argv[1], "pairs": pairs,
           "launches": int(sum(a["launches"] for a in k1)), "ncu_serialized_ms": ms,
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_pair": (rd + wr) / pairs,
           "inst_executed": inst, "inst_per_pair": inst / pairs,
           "per_variant": {k: {"ms": a["gpu__time_duration.sum"], "dram_bytes": a["dram__bytes_read.sum"] +
                               a["dram__bytes_write.sum"], "inst": a["smsp__inst_executed.sum"]}
                           for k, a in agg.items() if "ising_screen_pipe_kernel" in k}}
    json.dump(out, open(sys.argv[3], "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "per_variant"}))
