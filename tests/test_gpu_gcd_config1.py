"""Config 1 of BASELINE.json end to end against the compiled reference:
reconstruct_gcd to convergence (inc/reconstruct.hpp:148-181) on N=1000, M=500,
lambda=117.5, kappa=2 (k=8), eps=1e-6 N.

The reference's run is the fixture tests/golden/gcd_config1.npz (oracle/make_gcd_trace.py:
every iteration's candidate list from the candidate_hook, the iteration records and
the final state); the samples are regenerated from the seed by the C restatement of
the device chain and checked by digest.

* Lock-step: each iteration the device runs FindBest (same seed mix64(seed, iter)) on
  the state both sides share, its list is compared with the reference's list, then
  the REFERENCE's list is applied on the device (so the two states stay the same up to
  rounding) and the objective after the theta pass is compared.  Lists: same length,
  shared pairs with the same distance to 1e-9 relative, and every pair in the
  symmetric difference a near-tie at the cut (|gain - gain_cut| <= 1e-5 * max(|gain_cut|,
  1e-8 M) plus the rounding of base + gain).  Objective per iteration within 1e-6
  relative (north_star), final couplings within 1e-4 with identical support.
* Free-running: the device's own reconstruct_gcd from the empty state converges in
  the reference's number of iterations to the same objective (1e-6 relative) and
  couplings (1e-4)."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle_lib as O
from helpers import assert_lists_tie_aware, assert_rel, assert_same_couplings

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _setup(gpu, golden):
    g = golden("gcd_config1")
    n, M = int(g["n"]), int(g["M"])
    X, _ = O.gen_ising_colored(n, M, int(g["seed"]), mean_deg=4.0, w_sigma=0.3, th_sigma=0.1, burn_in=1000,
                               thin=10)
    assert hashlib.sha256(np.packbits(X > 0, axis=1).tobytes()).hexdigest() == str(g["digest"])
    dev = gpu.Model.from_samples(X, gpu.NRG_ISING, float(g["lam"]))
    return g, n, M, dev


def _pairs(i, j, d):
    out = np.zeros(len(i), dtype=O.PAIR_DT)
    out["i"], out["j"], out["dist"] = i, j, d
    return out


def test_gcd_config1_lockstep_vs_reference(gpu, golden):
    g, n, M, dev = _setup(gpu, golden)
    m = int(round(float(g["kappa"]) * n))
    nodes = np.arange(n, dtype=np.int32)
    iters = len(g["rec_objective"])
    base = dev.log_posterior()
    assert_rel(base, -n * M * np.log(2.0), 1e-12, "empty-state objective")
    n_diff, beyond = [], []
    for it in range(1, iters + 1):
        dev.begin_generation()
        fb, _, _ = dev.find_best(gpu.NRG_EXACT, m, nodes, seed=O.mix64(int(g["gcd_seed"]), it))
        ref = _pairs(g["cand_i"][it - 1], g["cand_j"][it - 1], g["cand_dist"][it - 1])
        try:
            n_diff.append(assert_lists_tie_aware(fb, ref, base, M, f"iteration {it}"))
        except AssertionError as e:
            beyond.append((it, str(e)[:300]))
            ka = set(zip(fb["i"].tolist(), fb["j"].tolist()))
            kb = set(zip(ref["i"].tolist(), ref["j"].tolist()))
            n_diff.append(len(ka ^ kb))
        delta = dev.apply_updates(ref)
        dev.theta_pass()
        base = dev.log_posterior()
        assert_rel(base, g["rec_objective"][it - 1], 1e-6, f"objective after iteration {it}")
        assert_rel(delta, g["rec_delta"][it - 1], 1e-6, f"delta of iteration {it}") if g["rec_delta"][it - 1] > 1e-9 \
            else None
    st = dev.get_state()
    assert_same_couplings(st, (None, g["final_i"], g["final_j"], g["final_w"]), tol=1e-4)
    np.testing.assert_allclose(st[0], g["final_theta"], rtol=0, atol=1e-4)
    print(f"config-1 lock-step: {iters} iterations, lists identical in {n_diff.count(0)}, "
          f"differing candidates per iteration {n_diff}; beyond near-ties: {beyond}")
    assert not beyond


def test_gcd_config1_free_running_converges_like_reference(gpu, golden):
    g, n, M, dev = _setup(gpu, golden)
    iters = len(g["rec_objective"])
    recs, conv = dev.reconstruct_gcd(kappa=float(g["kappa"]), max_iters=2 * iters + 20, seed=int(g["gcd_seed"]))
    assert conv
    print(f"device converged in {len(recs)} iterations (reference {iters}); final objective "
          f"{recs['objective'][-1]:.6f} vs {g['rec_objective'][-1]:.6f}")
    assert_rel(recs["objective"][-1], g["rec_objective"][-1], 1e-6, "converged objective")
    k = min(len(recs), iters)
    assert_rel(recs["objective"][:k], g["rec_objective"][:k], 1e-6, "objective per iteration")
    assert_same_couplings(dev.get_state(), (None, g["final_i"], g["final_j"], g["final_w"]), tol=1e-4)
