"""Same-box A/B of two builds on steady config-4 sweeps: alternating fresh processes of
tools/steady_sweep.py with the current library and with libnetrec_b200_prev.so (NRG_LIB);
prints each arm's median sweep and phase times.   usage: python tools/ab_lib.py [reps]"""
import json
import os
import statistics
import subprocess
import sys

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prev = os.path.join(os.getcwd(), "paper_2401_01404_b200", "libnetrec_b200_prev.so")
res = {"new": [], "prev": []}
for r in range(reps):
    for arm in ("new", "prev"):
        env = dict(os.environ)
        env.pop("NRG_LIB", None)
        if arm == "prev":
            env["NRG_LIB"] = prev
        out = subprocess.run([sys.executable, "tools/steady_sweep.py"], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if out.returncode or not line:
            print(arm, "failed", out.stderr[-2000:])
            continue
        res[arm].append(json.loads(line[-1]))
for arm, v in res.items():
    if not v:
        continue
    ph = {k: round(statistics.median(x["phases"][k] for x in v), 3) for k in v[0]["phases"]}
    print(f"{arm}: sweep ms {[round(x['ms'], 2) for x in v]} median {statistics.median(x['ms'] for x in v):.2f}; "
          f"k1 {statistics.median(x['k1_ms'] for x in v):.3f}; phases {ph}; misses {v[0]['misses']} hits {v[0]['hits']}")
