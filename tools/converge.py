"""Run one configuration of BASELINE.json end to end on the device: data from the
device generator, reconstruct_gcd from the empty state to convergence (eps = 1e-6 N,
inc/reconstruct.hpp:148-181), time to convergence, and the reconstruction against the
generator's truth with the reference's metrics (eval_reconstruction,
inc/bench.hpp:254-284: support precision / recall / F1, RMSE over the union support).

    python tools/converge.py --config config4 > profiles/r02_config4_convergence.json
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2401_01404_b200 as P  # noqa: E402

CONFIGS = {"config1": (1000, 500, 4.0, 0.3, "er"), "config2": (10_000, 1000, 4.0, 0.3, "er"),
           "config4": (100_000, 1000, 5.0, 0.3, "er"), "config5": (1_000_000, 200, 0.0, 0.2, "powerlaw")}


def eval_reconstruction(est, truth):
    """inc/bench.hpp:254-284: any stored (nonzero) entry is an edge; RMSE over the union."""
    e = {(int(min(a, b)), int(max(a, b))): float(w) for a, b, w in zip(*est) if w != 0.0}
    t = {(int(min(a, b)), int(max(a, b))): float(w) for a, b, w in zip(*truth) if w != 0.0}
    common = len(e.keys() & t.keys())
    union = e.keys() | t.keys()
    sq = sum((e.get(k, 0.0) - t.get(k, 0.0)) ** 2 for k in union)
    prec = common / len(e) if e else 1.0
    rec = common / len(t) if t else 1.0
    f1 = 2 * prec * rec / (prec + rec) if prec + rec > 0 else 0.0
    return {"precision": prec, "recall": rec, "f1": f1, "rmse": math.sqrt(sq / len(union)) if union else 0.0,
            "truth_edges": len(t), "estimate_edges": len(e), "common_edges": common}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config4", choices=list(CONFIGS))
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--burn-in", type=int, default=1000)
    ap.add_argument("--max-iters", type=int, default=1000)
    ap.add_argument("--kappa", type=float, default=2.0)
    a = ap.parse_args()
    n, M, deg, wsig, kind = CONFIGS[a.config]
    lam = 2.0 * math.sqrt(M * math.log(n))
    m = P.Model(n, M, P.NRG_ISING, lam)
    t0 = time.perf_counter()
    if kind == "er":
        m.generate_ising(mean_deg=deg, w_sigma=wsig, th_sigma=0.1, burn_in=a.burn_in, thin=10, seed=a.seed)
    else:
        m.generate_ising_powerlaw(gamma=2.5, dmin=2, w_sigma=wsig, th_sigma=0.1, burn_in=a.burn_in, thin=10,
                                  seed=a.seed)
    gen_s = time.perf_counter() - t0
    ti, tj, tw, tth = m.generated_truth()
    m.timer_start()
    t0 = time.perf_counter()
    recs, conv = m.reconstruct_gcd(kappa=a.kappa, max_iters=a.max_iters, seed=a.seed)
    wall = time.perf_counter() - t0
    dev_ms = m.timer_stop()
    th, ei, ej, w = m.get_state()
    q = eval_reconstruction((ei, ej, w), (ti, tj, tw))
    q["theta_rmse"] = float(np.sqrt(np.mean((th - tth) ** 2)))
    out = {"config": a.config, "n": n, "M": M, "lambda": lam, "kappa": a.kappa, "eps": 1e-6 * n,
           "converged": conv, "iterations": int(len(recs)),
           "time_to_convergence_s": float(recs["seconds"].sum()), "wall_s": wall, "device_ms": dev_ms,
           "first_sweeps_s": [round(float(x), 4) for x in recs["seconds"][:5]],
           "steady_sweep_s_median": float(np.median(recs["seconds"][5:])) if len(recs) > 5 else None,
           "objective": [float(x) for x in recs["objective"][:: max(1, len(recs) // 50)]],
           "final_objective": float(recs["objective"][-1]), "final_delta": float(recs["delta"][-1]),
           "gen_seconds": gen_s, "eval_reconstruction": q}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
