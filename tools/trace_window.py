"""Print the device operations around a kernel in a timeline.json (tools/timeline.py):
name, start offset and duration of the `before`/`after` operations around the first
launch whose name contains PATTERN.   usage: trace_window.py timeline.json PATTERN [after]"""
import json
import sys

ev = json.load(open(sys.argv[1]))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
pat = sys.argv[2]
after = int(sys.argv[3]) if len(sys.argv) > 3 else 30
i0 = next(i for i, e in enumerate(k) if pat in e["name"])
t0 = k[i0]["ts"]
for e in k[max(0, i0 - 3): i0 + after]:
    print(f"{(e['ts'] - t0) / 1e3:9.3f} ms  {e['dur'] / 1e3:8.3f} ms  {e['name'][:100]}")
