"""The fast paths of the dense FindBest levels against the plain ones, each in its own
process (the switches are read once per process): the persistent tensor-core screen vs one
tile per CTA, short candidate lists vs full lists, the covered-level shortcut vs the sweeps,
and the per-node staleness flags vs recomputing every row.  Same candidate lists, traces,
misses, hits, deltas and objectives."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np
import paper_2401_01404_b200 as P
import oracle_lib as O
n, M = 6000, 400
m = P.Model(n, M, P.NRG_ISING, O.ising_lambda(n, M))
m.generate_ising(mean_deg=4.0, seed=11)
m.reset_state()
out = []
for it in range(3):
    m.reset_counters()
    rec, cands = m.gcd_iteration(it, kappa=2.0, seed=7, want_candidates=True)
    c = m.counters()
    out.append([hashlib.sha256(np.ascontiguousarray(cands).tobytes()).hexdigest(), repr(float(rec["delta"])),
                repr(float(rec["objective"])), int(c["misses"]), int(c["hits"])])
m.begin_generation(); m.reset_counters()
fb, tr, sc = m.find_best(P.NRG_EXACT, 2 * n, np.arange(n, dtype=np.int32), seed=3)
c = m.counters()
out.append([hashlib.sha256(np.ascontiguousarray(fb).tobytes()).hexdigest(), [list(map(int, t)) for t in tr],
            int(c["misses"]), int(c["hits"])])
th, ei, ej, w = m.get_state()
out.append(hashlib.sha256(th.tobytes() + ei.tobytes() + ej.tobytes() + w.tobytes()).hexdigest())
print("RESULT " + json.dumps(out))
""" % (str(ROOT), str(ROOT / "tests"))


def _run(env_extra):
    env = dict(os.environ)
    for k in ("NRG_TC_ONE_TILE", "NRG_NO_SHORT_LISTS", "NRG_NO_COVER_LEVEL", "NRG_NO_ROW_FLAGS", "NRG_DENSE_EAGER"):
        env.pop(k, None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


def test_dense_fast_paths_equal_plain_paths():
    base = _run({})
    for switch in ("NRG_TC_ONE_TILE", "NRG_NO_SHORT_LISTS", "NRG_NO_COVER_LEVEL", "NRG_DENSE_EAGER"):
        assert _run({switch: "1"}) == base, switch


def test_row_flags_equal_full_recompute_up_to_theta_rounding():
    """Without the flags every theta is re-run from its optimum each sweep and may move by
    an ulp, so the comparison is numeric: same candidate lists in the first sweep, objectives
    within 1e-12 relative, same miss counts."""
    a, b = _run({}), _run({"NRG_NO_ROW_FLAGS": "1"})
    assert a[0] == b[0]
    for x, y in zip(a[:3], b[:3]):
        assert abs(float(x[2]) - float(y[2])) <= 1e-12 * abs(float(y[2]))
