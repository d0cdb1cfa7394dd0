"""Pair-score parity on the B200: distance() / optimize_edge / edge_gradient /
optimize_theta / log_posterior through the C-ABI vs the reference's golden vectors and
the C checker.  Tolerances in tests/helpers.py (w* 1e-4, gain 1e-5 rel with a 1e-8*M
floor, dist 1e-5 rel)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from helpers import assert_gains, assert_rel, assert_w

pytestmark = pytest.mark.gpu
CASES = ["ising_small", "ising_state", "gauss_small"]


def dev_model(P, g):
    m = P.Model.from_samples(g["X"], int(g["kind"]), float(g["lam"]))
    m.set_theta(g["theta_in"])
    if "e_i" in g:
        m.set_edges(g["e_i"], g["e_j"], g["e_w"])
    return m


@pytest.mark.parametrize("case", CASES)
def test_state_sums_and_log_posterior(gpu, golden, case):
    g = golden(case)
    m = dev_model(gpu, g)
    th, ei, ej, w = m.get_state()
    assert (ei == g["state_i"]).all() and (ej == g["state_j"]).all()
    np.testing.assert_array_equal(w, g["state_w"])
    np.testing.assert_allclose(m.get_sums(), g["sums"], rtol=0, atol=1e-12)
    assert_rel(m.log_posterior(), g["log_posterior"], 1e-11, "log_posterior")


@pytest.mark.parametrize("case", CASES)
def test_distance_exact_and_gradient(gpu, golden, case):
    g = golden(case)
    m = dev_model(gpu, g)
    M = g["X"].shape[1]
    i, j = g["pair_i"], g["pair_j"]
    m.begin_generation()
    d = m.distance(gpu.NRG_EXACT, i, j)
    assert_rel(d, g["dist_exact"], 1e-5, "exact distance")
    gain_ref = -(g["dist_exact"] + g["log_posterior"])
    gain_dev = -(d + m.log_posterior())
    assert_gains(gain_dev, np.maximum(gain_ref, 0.0), M, "gain from dist")
    # symmetric and memoized: d(j,i) == d(i,j) bitwise within the generation
    np.testing.assert_array_equal(m.distance(gpu.NRG_EXACT, j, i), d)
    m.begin_generation()
    dg = m.distance(gpu.NRG_GRADIENT, i, j)
    assert_rel(dg, g["dist_grad"], 1e-5, "gradient distance")


@pytest.mark.parametrize("case", CASES)
def test_optimize_edge(gpu, golden, case):
    g = golden(case)
    m = dev_model(gpu, g)
    M = g["X"].shape[1]
    i, j = g["pair_i"], g["pair_j"]
    w, gain, warn = m.optimize_edge(i, j)
    assert_w(w, g["opt_w"])
    assert_gains(gain, g["opt_gain"], M)
    assert (warn == g["opt_warn"]).all()
    np.testing.assert_allclose(m.edge_gradient(i, j), g["edge_grad"], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("case", CASES)
def test_optimize_theta(gpu, golden, case):
    g = golden(case)
    m = dev_model(gpu, g)
    np.testing.assert_allclose(m.optimize_theta(), g["opt_theta"], rtol=0, atol=1e-6)


def _config1(seed=1, n=1000, M=500):
    X, truth = O.gen_ising(n, M, seed=seed)
    return X, O.ising_lambda(n, M)


def test_config1_random_pairs_vs_checker(gpu):
    """Config 1 (Ising N=1000, M=500) at the empty state: 20k random pairs, exact mode."""
    X, lam = _config1()
    n, M = X.shape
    rng = np.random.default_rng(0)
    i = rng.integers(0, n, 22000)
    j = rng.integers(0, n, 22000)
    keep = i != j
    i, j = i[keep][:20000], j[keep][:20000]
    ref = O.CpuModel("orc", X, 0, lam)
    dev = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
    d_ref = ref.distance(0, i, j)
    d_dev = dev.distance(gpu.NRG_EXACT, i, j)
    assert_rel(d_dev, d_ref, 1e-5, "dist")
    g_ref = -(d_ref + ref.log_posterior())
    g_dev = -(d_dev + dev.log_posterior())
    assert_gains(g_dev, np.maximum(g_ref, 0), M)
    # pruned pairs are exact ties at -base on both sides
    assert ((g_ref == 0) == (g_dev == 0)).mean() > 0.999


def test_config1_after_gcd_iteration_vs_checker(gpu):
    """State transferred from the checker after one GCD iteration: existing edges,
    nonzero thetas — exact scores for all edges + random pairs."""
    X, lam = _config1(seed=2, n=600, M=300)
    n, M = X.shape
    ref = O.CpuModel("orc", X, 0, lam)
    ref.reconstruct_gcd(kappa=2.0, max_iters=1, seed=9)
    th, ei, ej, w = ref.get_state()
    dev = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
    dev.set_theta(th)
    dev.set_edges(ei, ej, w)
    np.testing.assert_allclose(dev.get_sums(), ref.get_sums(), rtol=0, atol=1e-12)
    rng = np.random.default_rng(1)
    ri, rj = rng.integers(0, n, 6000), rng.integers(0, n, 6000)
    keep = ri != rj
    i = np.concatenate([ei, ri[keep]])
    j = np.concatenate([ej, rj[keep]])
    ref.begin_generation()
    d_ref = ref.distance(0, i, j)
    d_dev = dev.distance(gpu.NRG_EXACT, i, j)
    assert_rel(d_dev, d_ref, 1e-5, "dist")
    w_ref, g_ref, _ = ref.optimize_edge(i, j)
    w_dev, g_dev, _ = dev.optimize_edge(i, j)
    assert_w(w_dev, w_ref)
    assert_gains(g_dev, g_ref, M)
    # the cached exact score equals -(base + live gain) in the same frozen state
    assert_gains(-(d_dev + dev.log_posterior()), g_ref, M, "cached gain")


def test_gaussian_vs_checker(gpu):
    rng = np.random.default_rng(5)
    n, M = 200, 120
    A = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.02)
    X = rng.standard_normal((n, M)) + 0.5 * A @ rng.standard_normal((n, M))
    lam = 5.0
    ref = O.CpuModel("orc", X, 1, lam)
    dev = gpu.Model.from_samples(X, gpu.NRG_GAUSSIAN, lam)
    np.testing.assert_allclose(dev.get_state()[0], ref.get_state()[0], rtol=1e-14)
    ref.reconstruct_gcd(kappa=1.0, max_iters=1, seed=3)
    th, ei, ej, w = ref.get_state()
    dev.set_theta(th)
    dev.set_edges(ei, ej, w)
    i = np.concatenate([ei, rng.integers(0, n, 3000)])
    j = np.concatenate([ej, rng.integers(0, n, 3000)])
    keep = i != j
    i, j = i[keep], j[keep]
    w_ref, g_ref, _ = ref.optimize_edge(i, j)
    w_dev, g_dev, _ = dev.optimize_edge(i, j)
    assert_w(w_dev, w_ref)
    assert_gains(g_dev, g_ref, M)
    ref.begin_generation()
    assert_rel(dev.distance(gpu.NRG_EXACT, i, j), ref.distance(0, i, j), 1e-5, "gauss dist")
    np.testing.assert_allclose(dev.optimize_theta(), ref.optimize_theta(), rtol=1e-6, atol=1e-9)


# ---- known answers of the reference suite (test_model.cpp), on the device
def test_ising_empty_state_log_posterior(gpu):
    rng = np.random.default_rng(1)
    X = np.where(rng.random((64, 50)) < 0.5, -1, 1).astype(np.int8)
    m = gpu.Model.from_samples(X, gpu.NRG_ISING, 1.0)
    assert abs(m.log_posterior() - (-64 * 50 * np.log(2))) <= 1e-12 * 64 * 50


def test_gaussian_unit_theta_log_posterior(gpu):
    rng = np.random.default_rng(2)
    X = rng.standard_normal((10, 15))
    m = gpu.Model.from_samples(X, gpu.NRG_GAUSSIAN, 0.5)
    m.set_theta(np.ones(10))
    assert abs(m.log_posterior() + 0.5 * (X ** 2).sum()) <= 1e-12 * (X ** 2).sum()


def test_huge_lambda_gives_exact_zero(gpu):
    rng = np.random.default_rng(3)
    X = np.where(rng.random((6, 40)) < 0.5, -1, 1).astype(np.int8)
    X[1] = X[0]
    m = gpu.Model.from_samples(X, gpu.NRG_ISING, 1e12)
    w, g, _ = m.optimize_edge([0], [1])
    assert w[0] == 0.0 and g[0] == 0.0


def test_aligned_columns_vanishing_derivative(gpu):
    """test_model.cpp:190-207: lambda = 0, aligned columns: w* > 0 and the slice is
    flat there (central difference of the checker's objective < 1e-6)."""
    M = 30
    rng = np.random.default_rng(4)
    x0 = np.where(rng.random(M) < 0.5, -1.0, 1.0)
    x1 = x0.copy()
    x1[:3] *= -1
    X = np.stack([x0, x1])
    m = gpu.Model.from_samples(X, gpu.NRG_ISING, 0.0)
    w, g, _ = m.optimize_edge([0], [1])
    assert w[0] > 0.0
    ref = O.CpuModel("orc", X, 0, 0.0)
    h = 1e-4
    fd = (ref.edge_objective(0, 1, w[0] + h) - ref.edge_objective(0, 1, w[0] - h)) / (2 * h)
    assert abs(fd) < 1e-6


def test_theta_known_answers(gpu):
    M = 25
    X = np.stack([np.ones(M), np.where(np.arange(M) % 2 == 0, 1.0, -1.0)])
    m = gpu.Model.from_samples(X, gpu.NRG_ISING, 0.0)
    th = m.optimize_theta()
    assert abs(th[0] - 20.0) <= 1e-6 and abs(th[1] - np.log(13 / 12) / 2) < 1e-9
    Xg = np.zeros((2, 10))
    Xg[1] = 1.0
    g = gpu.Model(2, 10, gpu.NRG_GAUSSIAN, 0.0)
    with pytest.raises(ValueError):
        g.upload_samples(Xg * np.nan)
    g.upload_samples(Xg)
    g.set_theta(np.ones(2))
    before = g.counters()["warnings"]
    th = g.optimize_theta()
    assert th[0] == 1e-8 and g.counters()["warnings"] == before + 1


def test_validation_errors(gpu):
    X = np.where(np.random.default_rng(0).random((5, 8)) < 0.5, -1.0, 1.0)
    with pytest.raises(ValueError):
        gpu.Model.from_samples(X * 0.5, gpu.NRG_ISING, 1.0)
    with pytest.raises(ValueError):
        gpu.Model(5, 8, gpu.NRG_ISING, -1.0)
    m = gpu.Model.from_samples(X, gpu.NRG_ISING, 1.0)
    with pytest.raises(ValueError):
        m.distance(gpu.NRG_EXACT, [1], [1])
    with pytest.raises(IndexError):
        m.distance(gpu.NRG_EXACT, [1], [7])
    gm = gpu.Model.from_samples(X, gpu.NRG_GAUSSIAN, 1.0)
    with pytest.raises(ValueError):
        gm.set_theta(np.zeros(5))  # gaussian model requires theta > 0


@pytest.mark.parametrize("M", [1000, 1024, 1500, 2048])
def test_wide_rows_vs_checker(gpu, M):
    """The screen variants by row width — M = 1000/1024 (the headline's shape: the
    shared-memory-staged K1), 1500 (partial words), 2048 (two words per lane): scores,
    couplings and gains vs the checker, at the empty state and after one checker GCD
    iteration (existing edges, nonzero fields)."""
    n = 200
    X, _ = O.gen_ising(n, M, seed=M, burn_in=200, thin=3)
    lam = O.ising_lambda(n, M)
    ref = O.CpuModel("orc", X, 0, lam)
    dev = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
    rng = np.random.default_rng(M)
    ri, rj = rng.integers(0, n, 4000), rng.integers(0, n, 4000)
    keep = ri != rj
    ri, rj = ri[keep], rj[keep]
    d_ref = ref.distance(0, ri, rj)
    d_dev = dev.distance(gpu.NRG_EXACT, ri, rj)
    assert_rel(d_dev, d_ref, 1e-5, "dist (empty state)")
    assert_gains(-(d_dev + dev.log_posterior()), np.maximum(-(d_ref + ref.log_posterior()), 0), M)
    ref.reconstruct_gcd(kappa=2.0, max_iters=1, seed=4)
    th, ei, ej, w = ref.get_state()
    dev.set_theta(th)
    dev.set_edges(ei, ej, w)
    i = np.concatenate([ei, ri])
    j = np.concatenate([ej, rj])
    ref.begin_generation()
    dev.begin_generation()
    d_ref = ref.distance(0, i, j)
    d_dev = dev.distance(gpu.NRG_EXACT, i, j)
    assert_rel(d_dev, d_ref, 1e-5, "dist (after a GCD iteration)")
    w_ref, g_ref, _ = ref.optimize_edge(i, j)
    w_dev, g_dev, _ = dev.optimize_edge(i, j)
    assert_w(w_dev, w_ref)
    assert_gains(g_dev, g_ref, M)
    assert_gains(-(d_dev + dev.log_posterior()), g_ref, M, "cached gain")


@pytest.mark.parametrize("M", [120, 1000])
def test_gaussian_screen_at_the_threshold(gpu, M):
    """The fp32 Gaussian screen (gauss_screen_kernel) only settles pairs its bound proves
    to be at the kink: with lambda at the median |P| (half the pairs within a hair of the
    threshold) the kink set and the distances equal the checker's."""
    rng = np.random.default_rng(M)
    n = 300
    X = rng.standard_normal((n, M)) + 0.3 * rng.standard_normal((1, M))
    i, j = rng.integers(0, n, 6000), rng.integers(0, n, 6000)
    keep = i != j
    i, j = i[keep], j[keep]
    th = np.sqrt((X * X).mean(axis=1))  # make_empty_state's theta (row RMS); sums are 0
    U = X  # u = x + theta^2 s with s = 0
    P = np.einsum("ij,ij->i", U[i], X[j]) + np.einsum("ij,ij->i", U[j], X[i])
    lam = float(np.median(np.abs(P)))
    ref = O.CpuModel("orc", X, 1, lam)
    dev = gpu.Model.from_samples(X, gpu.NRG_GAUSSIAN, lam)
    np.testing.assert_allclose(dev.get_state()[0], th, rtol=1e-12)
    ref.begin_generation()
    d_ref = ref.distance(0, i, j)
    d_dev = dev.distance(gpu.NRG_EXACT, i, j)
    base_ref = -ref.log_posterior()
    base_dev = -dev.log_posterior()
    kink_ref = d_ref == base_ref
    kink_dev = d_dev == base_dev
    assert 0.3 < kink_ref.mean() < 0.7
    np.testing.assert_array_equal(kink_dev, kink_ref)
    assert_rel(d_dev, d_ref, 1e-5, "gauss dist at the threshold")
