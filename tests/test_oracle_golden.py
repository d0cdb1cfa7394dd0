"""Pin the C restatement (oracle/nrg_oracle.c) against golden vectors produced by the
reference itself (oracle/make_golden.py over oracle/_ref).  CPU only.

Integer/set outputs must be identical; floating outputs agree to 1e-12 relative (both
are fp64 C/C++ with the same libm; residual differences come from summation order
in the prior and unordered_map iteration)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from helpers import assert_rel, row_sets

CASES = ["ising_small", "ising_state", "gauss_small"]


def _orc_model(g):
    kind = int(g["kind"])
    th = g["theta_in"]
    m = O.CpuModel("orc", g["X"], kind, float(g["lam"]), th)
    if "e_i" in g:
        m.set_edges(g["e_i"], g["e_j"], g["e_w"])
    return m


@pytest.mark.parametrize("case", CASES)
def test_state_and_objective(golden, case):
    g = golden(case)
    m = _orc_model(g)
    th, ei, ej, w = m.get_state()
    assert (ei == g["state_i"]).all() and (ej == g["state_j"]).all()
    np.testing.assert_array_equal(w, g["state_w"])
    np.testing.assert_allclose(m.get_sums(), g["sums"], rtol=0, atol=1e-12)
    assert_rel(m.log_posterior(), g["log_posterior"], 1e-12, "log_posterior")


@pytest.mark.parametrize("case", CASES)
def test_pair_scores(golden, case):
    g = golden(case)
    m = _orc_model(g)
    i, j = g["pair_i"], g["pair_j"]
    m.begin_generation()
    assert_rel(m.distance(0, i, j), g["dist_exact"], 1e-12, "exact distance")
    m.begin_generation()
    assert_rel(m.distance(1, i, j), g["dist_grad"], 1e-12, "gradient distance")
    w, gain, warn = m.optimize_edge(i, j)
    np.testing.assert_allclose(w, g["opt_w"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(gain, g["opt_gain"], rtol=1e-9, atol=1e-9)
    assert (warn == g["opt_warn"]).all()
    np.testing.assert_allclose(m.edge_gradient(i, j), g["edge_grad"], rtol=1e-12, atol=1e-9)
    # golden_max on a flat maximum is sensitive to last-bit differences (FMA contraction
    # moved theta by ~4e-8), so the checker is built with the reference's
    # -ffp-contract=off numerics and must agree to 1e-12
    np.testing.assert_allclose(m.optimize_theta(), g["opt_theta"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("case", CASES)
def test_search(golden, case):
    g = golden(case)
    m = _orc_model(g)
    n = g["X"].shape[0]
    nodes = np.arange(n, dtype=np.int32)
    seed = {"ising_small": 5, "ising_state": 6, "gauss_small": 7}[case]
    m.begin_generation()
    ids, dists, sweeps, churn = m.find_knn(0, 8, nodes, seed=seed + 1)
    assert sweeps == int(g["knn_sweeps"])
    assert row_sets(ids) == row_sets(g["knn_ids"])
    np.testing.assert_allclose(churn, g["knn_churn"], rtol=0, atol=0)
    m.begin_generation()
    fb, tr, sc = m.find_best(0, 2 * n, nodes, seed=seed + 2)
    assert (fb["i"] == g["fb_i"]).all() and (fb["j"] == g["fb_j"]).all()
    assert_rel(fb["dist"], g["fb_dist"], 1e-12, "find_best dist")
    assert (tr == g["fb_levels"]).all()


@pytest.mark.parametrize("case", CASES)
def test_updates_theta_gcd(golden, case):
    g = golden(case)
    m = _orc_model(g)
    n = g["X"].shape[0]
    nodes = np.arange(n, dtype=np.int32)
    seed = {"ising_small": 5, "ising_state": 6, "gauss_small": 7}[case]
    m.begin_generation()
    fb, _, _ = m.find_best(0, 2 * n, nodes, seed=seed + 2)
    delta = m.apply_updates(fb)
    assert_rel(delta, g["upd_delta"], 1e-9, "delta")
    th, ei, ej, w = m.get_state()
    assert (ei == g["upd_i"]).all() and (ej == g["upd_j"]).all()
    np.testing.assert_allclose(w, g["upd_w"], rtol=0, atol=1e-12)
    m.theta_pass()
    np.testing.assert_allclose(m.get_state()[0], g["upd_theta"], rtol=0, atol=1e-12)
    # GCD trajectory
    m2 = _orc_model(g)
    recs, conv, cand = m2.reconstruct_gcd(kappa=2.0, max_iters=3, seed=seed + 3, cand_cap=len(g["gcd_cand_i"]) + 8)
    assert_rel(recs["objective"], g["gcd_objective"], 1e-9, "gcd objective")
    assert_rel(recs["delta"], g["gcd_delta"], 1e-6, "gcd delta")
    th, ei, ej, w = m2.get_state()
    assert (ei == g["gcd_i"]).all() and (ej == g["gcd_j"]).all()
    np.testing.assert_allclose(w, g["gcd_w"], rtol=0, atol=1e-9)


def test_table_metric_search(golden):
    g = golden("table")
    t = g["table"]
    n = t.shape[0]
    m = O.CpuModel("orc", np.ones((n, 2)), 0, 0.0)
    m.set_table(t)
    nodes = np.arange(n, dtype=np.int32)
    for k in (1, 3, 8):
        ids, dists, sw, churn = m.find_knn(2, k, nodes, seed=21 + k)
        assert row_sets(ids) == row_sets(g[f"knn{k}_ids"]) and sw == int(g[f"knn{k}_sweeps"])
    ids, dists, sw, churn = m.find_knn(2, 4, nodes, seed=21)
    assert row_sets(ids) == row_sets(g["knn4_ids"])
    np.testing.assert_array_equal(churn, g["knn4_churn"])
    for mm in g["ms"]:
        fb, tr, sc = m.find_best(2, int(mm), nodes, seed=21 + int(mm))
        assert (fb["i"] == g[f"fb{mm}_i"]).all() and (fb["j"] == g[f"fb{mm}_j"]).all()
        np.testing.assert_array_equal(fb["dist"], g[f"fb{mm}_dist"])
        assert (tr == g[f"fb{mm}_levels"]).all() and int(sc) == int(g[f"fb{mm}_short"])
    lt = np.abs(g["pos"][:, None] - g["pos"][None, :])
    m.set_table(lt)
    ids, _, sw, _ = m.find_knn(2, 6, nodes, seed=21 + 99)
    assert row_sets(ids) == row_sets(g["line_ids"]) and sw == int(g["line_sweeps"])


def test_rng(golden):
    g = golden("rng")
    mix = [O.mix64(a, b) for a, b in [(0, 0), (1, 2), (2 ** 63, 7), (12345, 2 ** 40)]]
    np.testing.assert_array_equal(np.array(mix, dtype=np.uint64), g["mix"])
    np.testing.assert_array_equal(O.rng_stream(42, 7, 64, 0), g["stream"])
    np.testing.assert_array_equal(O.rng_stream(42, 0, 64, 1000), g["below"])


@pytest.mark.skipif(not O.available("ref"), reason="reference not compiled here")
@pytest.mark.parametrize("case", CASES)
def test_reference_reproduces_golden(golden, case):
    """The compiled reference regenerates its own fixtures (fixtures are current)."""
    g = golden(case)
    m = O.CpuModel("ref", g["X"], int(g["kind"]), float(g["lam"]), g["theta_in"])
    if "e_i" in g:
        m.set_edges(g["e_i"], g["e_j"], g["e_w"])
    m.begin_generation()
    np.testing.assert_array_equal(m.distance(0, g["pair_i"], g["pair_j"]), g["dist_exact"])


# ---- known-answer tests of the reference suite (test_model.cpp), against the checker
def test_ising_empty_state_is_minus_NM_log2():
    rng = np.random.default_rng(1)
    X = np.where(rng.random((30, 20)) < 0.5, -1.0, 1.0)
    m = O.CpuModel("orc", X, 0, 1.0)
    assert abs(m.log_posterior() - (-30 * 20 * np.log(2))) <= 1e-12 * 30 * 20


def test_gaussian_unit_theta_is_minus_half_sum_sq():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((10, 15))
    m = O.CpuModel("orc", X, 1, 0.5, np.ones(10))
    assert abs(m.log_posterior() + 0.5 * (X ** 2).sum()) <= 1e-12 * (X ** 2).sum()


def test_huge_lambda_forces_exact_zero():
    rng = np.random.default_rng(3)
    X = np.where(rng.random((6, 40)) < 0.5, -1.0, 1.0)
    X[1] = X[0]
    m = O.CpuModel("orc", X, 0, 1e12)
    w, g, _ = m.optimize_edge([0], [1])
    assert w[0] == 0.0 and g[0] == 0.0
