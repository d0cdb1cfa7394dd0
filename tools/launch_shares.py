"""Kernel shares from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iN, iV = h.index("Kernel Name"), h.index("Metric Value")
skip = sys.argv[2].split(",") if len(sys.argv) > 2 else []
tot = defaultdict(float); cnt = defaultdict(int)
for r in rows[1:]:
    try: v = float(r[iV].replace(",", ""))
    except ValueError: continue
    n = r[iN]
    if any(s in n for s in skip): continue
    tot[n] += v; cnt[n] += 1
T = sum(tot.values())
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{v/1e6:10.2f} ms {100*v/T:6.2f}% {cnt[n]:7d}  {n[:110]}")
print(f"total {T/1e6:.1f} ms")
