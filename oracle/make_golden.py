"""Generate tests/golden/*.npz by running the REFERENCE itself (oracle/_ref/libnetrec_ref.so,
the unmodified netrec headers compiled behind ref_shim.cpp).  Test infrastructure only.

    make -C oracle && python oracle/make_golden.py

Inputs are seeded and stored in the fixtures, so the fixtures are self-contained and
the GPU box (which has no /root/reference) can check against them.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
import oracle_lib as O  # noqa: E402

OUT = ROOT / "tests" / "golden"


def pairs_of(n, count, rng):
    i = rng.integers(0, n, count * 2)
    j = rng.integers(0, n, count * 2)
    keep = i != j
    return i[keep][:count].astype(np.int32), j[keep][:count].astype(np.int32)


def model_case(name, X, kind, lam, theta, edges, seed, m_gcd_kappa=2.0, gcd_iters=3):
    rng = np.random.default_rng(seed)
    n, M = X.shape
    R = O.CpuModel("ref", X, kind, lam, theta)
    if edges is not None:
        R.set_edges(*edges)
    out = dict(X=X, kind=np.int32(kind), lam=np.float64(lam),
               theta_in=np.asarray(theta if theta is not None else R.get_state()[0], dtype=np.float64))
    if edges is not None:
        out.update(e_i=edges[0], e_j=edges[1], e_w=edges[2])
    th, ei, ej, w = R.get_state()
    out.update(state_theta=th, state_i=ei, state_j=ej, state_w=w, sums=R.get_sums())
    out["log_posterior"] = np.float64(R.log_posterior())
    # pair scores: random pairs + every existing edge
    pi, pj = pairs_of(n, 400, rng)
    if len(ei):
        pi = np.concatenate([pi, ei, ej[: len(ej) // 2]])
        pj = np.concatenate([pj, ej, ei[: len(ei) // 2]])
    out.update(pair_i=pi, pair_j=pj)
    R.begin_generation()
    out["dist_exact"] = R.distance(0, pi, pj)
    R.begin_generation()
    out["dist_grad"] = R.distance(1, pi, pj)
    wv, gv, warn = R.optimize_edge(pi, pj)
    out.update(opt_w=wv, opt_gain=gv, opt_warn=warn)
    out["edge_grad"] = R.edge_gradient(pi, pj)
    out["opt_theta"] = R.optimize_theta()
    # NNDescent + FindBest on the model distance (exact mode)
    nodes = np.arange(n, dtype=np.int32)
    R.begin_generation()
    ids, dists, sweeps, churn = R.find_knn(0, 8, nodes, seed=seed + 1)
    out.update(knn_ids=ids, knn_dists=dists, knn_sweeps=np.int32(sweeps), knn_churn=churn)
    R.begin_generation()
    fb, tr, sc = R.find_best(0, 2 * n, nodes, seed=seed + 2)
    out.update(fb_i=fb["i"], fb_j=fb["j"], fb_dist=fb["dist"], fb_levels=tr)
    # one round of updates on the find_best candidates, then a theta pass
    delta = R.apply_updates(fb)
    out["upd_delta"] = np.float64(delta)
    th, ei, ej, w = R.get_state()
    out.update(upd_i=ei, upd_j=ej, upd_w=w, upd_sums=R.get_sums())
    R.theta_pass()
    out["upd_theta"] = R.get_state()[0]
    out["upd_log_posterior"] = np.float64(R.log_posterior())
    # full GCD from the input state
    R2 = O.CpuModel("ref", X, kind, lam, theta)
    if edges is not None:
        R2.set_edges(*edges)
    recs, conv, cand = R2.reconstruct_gcd(kappa=m_gcd_kappa, max_iters=gcd_iters, seed=seed + 3,
                                          cand_cap=gcd_iters * int(round(m_gcd_kappa * n)) + 8)
    th, ei, ej, w = R2.get_state()
    out.update(gcd_delta=recs["delta"], gcd_objective=recs["objective"], gcd_candidates=recs["candidates"],
               gcd_cand_i=cand["i"], gcd_cand_j=cand["j"], gcd_cand_dist=cand["dist"],
               gcd_theta=th, gcd_i=ei, gcd_j=ej, gcd_w=w)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, {k: np.asarray(v).shape for k, v in list(out.items())[:3]}, "fb levels", len(tr))


def table_case(name, n, seed):
    """TableMetric (test_findbest.cpp:20-37) and LineMetric (test_knn.cpp:16-29) searches."""
    rng = np.random.default_rng(seed)
    t = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    t[iu] = rng.standard_normal(len(iu[0]))
    pos = rng.random(n)
    X = np.ones((n, 2))
    R = O.CpuModel("ref", X, 0, 0.0)
    R.set_table(t)
    nodes = np.arange(n, dtype=np.int32)
    out = dict(table=t, pos=pos)
    for k in (1, 3, 8):
        ids, dists, sw, churn = R.find_knn(2, k, nodes, seed=seed + k)
        out[f"knn{k}_ids"], out[f"knn{k}_dists"], out[f"knn{k}_sweeps"] = ids, dists, np.int32(sw)
    ids, dists, sw, churn = R.find_knn(2, 4, nodes, seed=seed, width_floor=4, scan_floor=8)
    out["knn4_ids"], out["knn4_sweeps"], out["knn4_churn"] = ids, np.int32(sw), churn
    for m in (5, n // 2, 2 * n, n * n):
        fb, tr, sc = R.find_best(2, m, nodes, seed=seed + m)
        out[f"fb{m}_i"], out[f"fb{m}_j"], out[f"fb{m}_dist"] = fb["i"], fb["j"], fb["dist"]
        out[f"fb{m}_levels"], out[f"fb{m}_short"] = tr, np.int32(sc)
    out["ms"] = np.array([5, n // 2, 2 * n, n * n], dtype=np.int64)
    # line metric kNN: store as a full table so both sides read the same values
    lt = np.abs(pos[:, None] - pos[None, :])
    R.set_table(lt)
    ids, dists, sw, churn = R.find_knn(2, 6, nodes, seed=seed + 99)
    out["line_ids"], out["line_sweeps"] = ids, np.int32(sw)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name)


def rng_case():
    out = {}
    out["mix"] = np.array([O.mix64(a, b, "ref") for a, b in [(0, 0), (1, 2), (2 ** 63, 7), (12345, 2 ** 40)]],
                          dtype=np.uint64)
    out["stream"] = O.rng_stream(42, 7, 64, 0, "ref")
    out["below"] = O.rng_stream(42, 0, 64, 1000, "ref")
    np.savez_compressed(OUT / "rng.npz", **out)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng_case()
    # Ising: seeded ER truth + Gibbs samples (checker generator), lambda = 2 sqrt(M ln N)
    X, truth = O.gen_ising(80, 60, seed=11, burn_in=200, thin=5)
    model_case("ising_small", X, 0, O.ising_lambda(80, 60), None, None, seed=5)
    # Ising from a non-empty state: a few scattered edges + nonzero thetas
    rng = np.random.default_rng(3)
    ei = rng.integers(0, 80, 30).astype(np.int32)
    ej = ((ei + 1 + rng.integers(0, 79, 30)) % 80).astype(np.int32)
    ew = 0.2 * rng.standard_normal(30)
    th = 0.1 * rng.standard_normal(80)
    model_case("ising_state", X, 0, 0.5 * O.ising_lambda(80, 60), th, (ei, ej, ew), seed=6)
    # Gaussian: correlated data from a random sparse precision matrix (numpy)
    n, M = 50, 40
    P = np.eye(n) * 1.5
    for _ in range(60):
        a, b = rng.integers(0, n, 2)
        if a != b:
            v = rng.uniform(-0.2, 0.2)
            P[a, b] += v
            P[b, a] += v
    P += np.eye(n) * np.abs(P - np.diag(np.diag(P))).sum(1)
    L = np.linalg.cholesky(np.linalg.inv(P))
    Xg = (L @ rng.standard_normal((n, M)))
    model_case("gauss_small", Xg, 1, 2.0, None, None, seed=7)
    table_case("table", 40, seed=21)


if __name__ == "__main__":
    main()
