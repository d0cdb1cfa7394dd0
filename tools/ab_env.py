"""A/B of a run-time switch on steady config-4 sweeps: runs tools/steady_sweep.py N times
with and without ENV=1 (alternating, fresh processes) and prints the median sweep time
and phase times of each arm.   usage: python tools/ab_env.py NRG_SWITCH [reps]"""
import json
import os
import statistics
import subprocess
import sys

env_name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
res = {"off": [], "on": []}
for r in range(reps):
    for arm in ("off", "on"):
        env = dict(os.environ)
        env.pop(env_name, None)
        if arm == "on":
            env[env_name] = "1"
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
    print(f"{env_name}={'1' if arm == 'on' else 'unset'}: sweep ms {[round(x['ms'], 2) for x in v]} median "
          f"{statistics.median(x['ms'] for x in v):.2f}; phases {ph}; misses {v[0]['misses']}")
