"""Generate tests/golden/gcd_config2.npz: three GCD iterations of the REFERENCE on config 2
of BASELINE.json (Ising ER N=1e4 mean degree 4, w ~ N(0, 0.3^2), theta ~ N(0, 0.1^2),
M=1000 samples from the device data pipeline's chain, lambda = 2 sqrt(M ln N) = 191.9,
kappa = 2: 20000 candidates per iteration).  Test infrastructure only.

The loop is reconstruct_gcd's body (inc/reconstruct.hpp:162-176) driven through the
compiled reference's own functions so FindBest and the theta pass can use 8 threads
(thread-count invariant, test_findbest.cpp:176-189) while apply_edge_updates runs its
sequential branch (threads = 1, inc/reconstruct.hpp:74-82): begin_generation, find_best
with seed mix64(seed, iter), apply_edge_updates, theta_pass, log_posterior.

    make -C oracle && python oracle/make_gcd_trace_c2.py
"""
from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
import oracle_lib as O  # noqa: E402

N, M, SEED, GCD_SEED, KAPPA, ITERS = 10_000, 1000, 2, 3, 2.0, 3


def main():
    X, _ = O.gen_ising_colored(N, M, SEED, mean_deg=4.0, w_sigma=0.3, th_sigma=0.1, burn_in=1000, thin=10)
    lam = O.ising_lambda(N, M)
    m = int(round(KAPPA * N))
    R = O.CpuModel("ref", X.astype(np.float64), 0, lam)
    nodes = np.arange(N, dtype=np.int32)
    cands, objs, deltas = [], [], []
    for it in range(1, ITERS + 1):
        t = time.time()
        R.begin_generation()
        fb, _, _ = R.find_best(0, m, nodes, seed=O.mix64(GCD_SEED, it), threads=8)
        d = R.apply_updates(fb, threads=1)
        R.theta_pass(threads=8)
        objs.append(R.log_posterior())
        deltas.append(d)
        cands.append(fb)
        print(f"iteration {it}: {time.time() - t:.0f} s, delta {d:.6f}, objective {objs[-1]:.6f}", flush=True)
    th, ei, ej, w = R.get_state()
    np.savez_compressed(ROOT / "tests" / "golden" / "gcd_config2.npz",
                        n=np.int32(N), M=np.int32(M), seed=np.uint64(SEED), gcd_seed=np.uint64(GCD_SEED),
                        kappa=np.float64(KAPPA), lam=np.float64(lam),
                        digest=np.array(hashlib.sha256(np.packbits(X > 0, axis=1).tobytes()).hexdigest()),
                        rec_objective=np.array(objs), rec_delta=np.array(deltas),
                        cand_i=np.stack([c["i"] for c in cands]).astype(np.uint16),
                        cand_j=np.stack([c["j"] for c in cands]).astype(np.uint16),
                        cand_dist=np.stack([c["dist"] for c in cands]),
                        final_theta=th, final_i=ei, final_j=ej, final_w=w)


if __name__ == "__main__":
    main()
