"""Summarise an .ncu-rep: SOL, occupancy, pipes, stall reasons, SASS opcode stalls."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))
r = page("raw")
h, u, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]
d = dict(zip(h, zip(u, v)))
for k in want:
    if k in d: print(f"{k:60s} {d[k][1]:>16s} {d[k][0]}")
st = [(k, float(d[k][1].replace(',', ''))) for k in d if k.startswith("smsp__average_warp_latency_issue_stalled") or
      (k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"))]
st.sort(key=lambda x: -x[1])
print("stalls (warps per issue):")
for k, x in st[:10]: print(f"   {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):30s} {x:.3f}")
rows = page("source", ["--print-source", "sass"])
hh = rows[1]; data = rows[2:]
iS = hh.index("Warp Stall Sampling (All Samples)"); iE = hh.index("Instructions Executed"); iSrc = hh.index("Source")
tot = sum(float(x[iS] or 0) for x in data) or 1; totE = sum(float(x[iE] or 0) for x in data) or 1
c, ce = Counter(), Counter()
for x in data:
    t = x[iSrc].split()
    if not t: continue
    op = t[1] if t[0].startswith('@') and len(t) > 1 else t[0]
    op = op.split('.')[0]
    c[op] += float(x[iS] or 0); ce[op] += float(x[iE] or 0)
print("opcode stall% / inst%:")
for op, x in c.most_common(14): print(f"   {op:10s} {100*x/tot:5.1f} {100*ce[op]/totE:5.1f}")
