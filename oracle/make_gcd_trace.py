"""Generate tests/golden/gcd_config1.npz: the REFERENCE's reconstruct_gcd
(oracle/_ref, inc/reconstruct.hpp:148-181) run to convergence on config 1 of
BASELINE.json -- Ising, Erdos-Renyi N=1000 mean degree 4, w ~ N(0, 0.3^2),
theta ~ N(0, 0.1^2), M=500 Gibbs samples (burn-in 1000, thin 10) from the device
data pipeline's chain (orc_gen_ising_colored, bit-identical to gen.cu), lambda =
2 sqrt(M ln N) = 117.5, kappa = 2 (2000 candidates per iteration, NNDescent k = 8),
eps = 1e-6 N.  Test infrastructure only.

    make -C oracle && python oracle/make_gcd_trace.py

threads = 1: the reference's apply_edge_updates is the sequential Gauss-Seidel loop only
for threads <= 1 (inc/reconstruct.hpp:74-82; more threads take try-locks with deferral,
a nondeterministic order).  The fixture stores every iteration's candidate list (the candidate_hook), the
iteration records and the final state; the samples are regenerated from the seed
(and checked by digest) on the GPU box.
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

N, M, SEED, GCD_SEED, KAPPA = 1000, 500, 1, 3, 2.0
MAX_ITERS = 400


def main():
    X, truth = O.gen_ising_colored(N, M, SEED, mean_deg=4.0, w_sigma=0.3, th_sigma=0.1, burn_in=1000, thin=10)
    lam = O.ising_lambda(N, M)
    m = int(round(KAPPA * N))
    R = O.CpuModel("ref", X.astype(np.float64), 0, lam)
    t = time.time()
    recs, conv, cands = R.reconstruct_gcd(kappa=KAPPA, eps=-1.0, max_iters=MAX_ITERS, seed=GCD_SEED, threads=1,
                                          cand_cap=MAX_ITERS * m)
    secs = time.time() - t
    assert conv, "reference did not converge"
    th, ei, ej, w = R.get_state()
    assert len(cands) == len(recs) * m
    out = dict(n=np.int32(N), M=np.int32(M), seed=np.uint64(SEED), gcd_seed=np.uint64(GCD_SEED),
               kappa=np.float64(KAPPA), lam=np.float64(lam),
               digest=np.array(hashlib.sha256(np.packbits(X > 0, axis=1).tobytes()).hexdigest()),
               rec_objective=recs["objective"], rec_delta=recs["delta"], rec_candidates=recs["candidates"],
               cand_i=cands["i"].astype(np.uint16).reshape(len(recs), m),
               cand_j=cands["j"].astype(np.uint16).reshape(len(recs), m),
               cand_dist=cands["dist"].reshape(len(recs), m),
               final_theta=th, final_i=ei, final_j=ej, final_w=w,
               truth_i=truth["i"], truth_j=truth["j"], truth_w=truth["w"], truth_theta=truth["theta"])
    np.savez_compressed(ROOT / "tests" / "golden" / "gcd_config1.npz", **out)
    print(f"{len(recs)} iterations, converged={conv}, {secs:.0f} s, {len(ei)} couplings")


if __name__ == "__main__":
    main()
