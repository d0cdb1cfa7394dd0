"""The device data pipeline's chain (coloured Gibbs, restated in C as
orc_gen_ising_colored and pinned bit-exactly to the device by
tests/test_gpu_generators.py) against the reference's sequential single-site sampler
(sample_ising, inc/synth.hpp:133-158, restated as orc_gen_ising): same truth, same
stationary law.  Per-node magnetisations and truth-edge correlations agree: every
standardised difference below 5 (sigma estimated from 40 batch means per chain, so
the statistic is t-distributed with ~39 dof: P(|t| > 5) ~ 1e-5 per node) and the mean
squared one near 1.  CPU only."""
from __future__ import annotations

import numpy as np

import oracle_lib as O


def _batch_sigma(v, nb=40):
    """standard error of the mean of each row of v [rows, M] from nb batch means"""
    M = v.shape[1] - v.shape[1] % nb
    b = v[:, :M].reshape(v.shape[0], nb, -1).mean(axis=2)
    return b.std(axis=1, ddof=1) / np.sqrt(nb)


def test_colored_chain_has_the_reference_law():
    n, M, seed = 400, 4000, 17
    Xs, ts = O.gen_ising(n, M, seed=seed, mean_deg=4.0, burn_in=500, thin=5)
    Xc, tc = O.gen_ising_colored(n, M, seed, mean_deg=4.0, burn_in=500, thin=5)
    # identical truth (the reference's ER scheme on SplitRng(mix64(seed, 0)))
    for k in ("i", "j", "w", "theta"):
        np.testing.assert_array_equal(ts[k], tc[k])
    assert not np.array_equal(Xs.astype(np.int8), Xc)  # different chains...
    Xs = Xs.astype(np.float64)
    Xc = Xc.astype(np.float64)
    # ...same law: magnetisations
    sig = np.sqrt(_batch_sigma(Xs) ** 2 + _batch_sigma(Xc) ** 2)
    z = (Xs.mean(axis=1) - Xc.mean(axis=1)) / np.maximum(sig, 1e-3)
    assert np.abs(z).max() < 5.0, np.abs(z).max()
    assert 0.3 < np.mean(z ** 2) < 2.0, np.mean(z ** 2)
    # truth-edge correlations <x_i x_j>
    ei, ej = ts["i"], ts["j"]
    cs, cc = Xs[ei] * Xs[ej], Xc[ei] * Xc[ej]
    sig = np.sqrt(_batch_sigma(cs) ** 2 + _batch_sigma(cc) ** 2)
    z = (cs.mean(axis=1) - cc.mean(axis=1)) / np.maximum(sig, 1e-3)
    assert np.abs(z).max() < 5.0, np.abs(z).max()
    assert 0.3 < np.mean(z ** 2) < 2.0, np.mean(z ** 2)
    # and the correlations carry the couplings' signs (the data is informative)
    strong = np.abs(ts["w"]) > 0.3
    assert np.mean(np.sign(cs.mean(axis=1)[strong]) == np.sign(ts["w"][strong])) > 0.9


def test_colored_chain_is_thread_count_invariant():
    a, _ = O.gen_ising_colored(500, 64, 3, burn_in=50, thin=2, threads=1)
    b, _ = O.gen_ising_colored(500, 64, 3, burn_in=50, thin=2, threads=7)
    np.testing.assert_array_equal(a, b)
