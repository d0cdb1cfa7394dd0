"""Coordinate updates, theta pass and whole GCD iterations on the B200 vs the
reference: for the same candidate list, identical support and couplings within 1e-4;
GCD trajectories (objective per iteration) within 1e-6 relative."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from helpers import assert_rel, assert_same_couplings

pytestmark = pytest.mark.gpu
CASES = ["ising_small", "ising_state", "gauss_small"]


def dev_model(P, g):
    m = P.Model.from_samples(g["X"], int(g["kind"]), float(g["lam"]))
    m.set_theta(g["theta_in"])
    if "e_i" in g:
        m.set_edges(g["e_i"], g["e_j"], g["e_w"])
    return m


@pytest.mark.parametrize("case", CASES)
def test_updates_on_reference_candidates(gpu, golden, case):
    g = golden(case)
    m = dev_model(gpu, g)
    cands = np.zeros(len(g["fb_i"]), gpu.PAIR_DT)
    cands["i"], cands["j"], cands["dist"] = g["fb_i"], g["fb_j"], g["fb_dist"]
    delta = m.apply_updates(cands)
    assert_rel(delta, g["upd_delta"], 1e-6, "delta")
    st = m.get_state()
    assert_same_couplings(st, (None, g["upd_i"], g["upd_j"], g["upd_w"]))
    np.testing.assert_allclose(m.get_sums(), g["upd_sums"], rtol=0, atol=1e-6)
    m.theta_pass()
    np.testing.assert_allclose(m.get_state()[0], g["upd_theta"], rtol=0, atol=1e-6)
    assert_rel(m.log_posterior(), g["upd_log_posterior"], 1e-9, "objective after updates")


@pytest.mark.parametrize("case", CASES)
def test_gcd_trajectory(gpu, golden, case):
    g = golden(case)
    m = dev_model(gpu, g)
    seed = {"ising_small": 5, "ising_state": 6, "gauss_small": 7}[case]
    recs, conv = m.reconstruct_gcd(kappa=2.0, max_iters=3, seed=seed + 3)
    assert_rel(recs["objective"], g["gcd_objective"], 1e-6, "objective per iteration")
    np.testing.assert_array_equal(recs["candidates"], g["gcd_candidates"])
    assert_same_couplings(m.get_state(), (None, g["gcd_i"], g["gcd_j"], g["gcd_w"]), tol=1e-3,
                          allow_support_diff=2)


def test_updates_config1_candidates_from_checker(gpu):
    """Config-1 shape: the checker's FindBest candidates (2N pairs, many sharing hubs)
    applied on both sides from the same state."""
    X, _ = O.gen_ising(1000, 500, seed=1)
    lam = O.ising_lambda(1000, 500)
    n = X.shape[0]
    ref = O.CpuModel("orc", X, 0, lam)
    ref.begin_generation()
    fb, _, _ = ref.find_best(1, 2 * n, np.arange(n, dtype=np.int32), seed=4)
    dev = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
    d_dev = dev.apply_updates(fb)
    d_ref = ref.apply_updates(fb)
    assert_rel(d_dev, d_ref, 1e-6, "delta")
    assert_same_couplings(dev.get_state(), ref.get_state())
    dev.theta_pass()
    ref.theta_pass()
    np.testing.assert_allclose(dev.get_state()[0], ref.get_state()[0], atol=1e-6)
    assert_rel(dev.log_posterior(), ref.log_posterior(), 1e-9, "objective")


def test_set_edges_sequential_semantics(gpu):
    """set_edge list applied in order (later writes win, zero deletes), sums rebuilt."""
    rng = np.random.default_rng(0)
    X = np.where(rng.random((30, 40)) < 0.5, -1.0, 1.0)
    ei = np.array([0, 1, 0, 2, 5, 0], np.int32)
    ej = np.array([1, 0, 3, 4, 6, 3], np.int32)
    w = np.array([0.5, 0.25, 0.1, -0.3, 0.2, 0.0])
    dev = gpu.Model.from_samples(X, gpu.NRG_ISING, 1.0)
    ref = O.CpuModel("orc", X, 0, 1.0)
    dev.set_edges(ei, ej, w)
    ref.set_edges(ei, ej, w)
    th, a, b, ww = dev.get_state()
    assert list(zip(a, b, ww)) == list(zip(*ref.get_state()[1:]))
    np.testing.assert_allclose(dev.get_sums(), ref.get_sums(), rtol=0, atol=1e-15)


@pytest.mark.parametrize("kind", ["ising", "gauss"])
def test_bulk_set_edges_equals_sequential(gpu, monkeypatch, kind):
    """set_edges into an empty table with distinct pairs takes the per-node incidence
    pass (update.cu set_edges_bulk); its sums, couplings and objective are bitwise those
    of the sequential set_edge path, and the reference's."""
    rng = np.random.default_rng(3)
    n, M = 400, 300
    X = np.where(rng.random((n, M)) < 0.5, -1.0, 1.0) if kind == "ising" else rng.standard_normal((n, M))
    K = gpu.NRG_ISING if kind == "ising" else gpu.NRG_GAUSSIAN
    i = rng.integers(0, n, 5000)
    j = rng.integers(0, n, 5000)
    keep = i != j
    key = np.minimum(i, j)[keep] * n + np.maximum(i, j)[keep]
    _, first = np.unique(key, return_index=True)
    first.sort()
    ei, ej = i[keep][first].astype(np.int32), j[keep][first].astype(np.int32)
    w = rng.normal(0, 0.2, len(ei))
    w[::17] = 0.0
    out = []
    for bulk in (True, False):
        if bulk:
            monkeypatch.delenv("NRG_NO_BULK_SET", raising=False)
        else:
            monkeypatch.setenv("NRG_NO_BULK_SET", "1")
        m = gpu.Model.from_samples(X, K, 1.0)
        m.set_edges(ei, ej, w)
        out.append((m.get_sums(), m.get_state(), m.log_posterior()))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    for a, b in zip(out[0][1][1:], out[1][1][1:]):
        np.testing.assert_array_equal(a, b)
    assert out[0][2] == out[1][2]
    ref = O.CpuModel("orc", X, 0 if kind == "ising" else 1, 1.0)
    ref.set_edges(ei, ej, w)
    np.testing.assert_array_equal(out[0][0], ref.get_sums())


def test_device_generator_and_full_iteration(gpu):
    """Device Gibbs data (config-1 shape) + two GCD iterations run end to end; the
    objective increases and the edge count is plausible."""
    m = gpu.Model(1000, 500, gpu.NRG_ISING, O.ising_lambda(1000, 500))
    X = m.generate_ising(mean_deg=4.0, seed=1, want_samples=True)
    assert set(np.unique(X)) == {-1, 1}
    objs = [m.log_posterior()]
    for it in (1, 2):
        rec, cands = m.gcd_iteration(it, kappa=2.0, seed=3, want_candidates=True)
        objs.append(rec["objective"])
        assert rec["candidates"] == 2000 and len(cands) == 2000
    assert objs[1] > objs[0] and objs[2] >= objs[1] - 1e-6 * abs(objs[1])
    ne = len(m.get_state()[1])
    assert 500 < ne < 20000


def test_concurrent_inserts_keep_their_values(gpu):
    """set_edges on many node-disjoint pairs: the update kernel inserts them into the
    coupling hash concurrently (probe chains collide); every value must read back as
    written (regression: value stored before the slot claim could be overwritten by a
    losing inserter of another key)."""
    n, M = 20000, 64
    rng = np.random.default_rng(11)
    X = np.where(rng.random((n, M)) < 0.5, 1, -1).astype(np.int8)
    m = gpu.Model.from_samples(X, gpu.NRG_ISING, 1.0)
    for rep in range(4):
        perm = rng.permutation(n)
        ei, ej = perm[0::2].astype(np.int32), perm[1::2].astype(np.int32)
        w = rng.uniform(0.01, 0.5, len(ei)) * rng.choice([-1.0, 1.0], len(ei))
        m.reset_state()
        m.set_edges(ei, ej, w)
        _, gi, gj, gw = m.get_state()
        lo, hi = np.minimum(ei, ej), np.maximum(ei, ej)
        order = np.lexsort((hi, lo))
        np.testing.assert_array_equal(gi, lo[order])
        np.testing.assert_array_equal(gj, hi[order])
        np.testing.assert_array_equal(gw, w[order])


def test_tie_tail_rounds_match_ordered(gpu, monkeypatch):
    """apply_updates resolves the trailing block of tied (zero-gain) candidates in
    parallel rounds; three GCD iterations must give the same reconstruction as the
    purely dependency-ordered path (NRG_ORDERED_ONLY), and the rounds must be used."""
    def run(ordered):
        if ordered:
            monkeypatch.setenv("NRG_ORDERED_ONLY", "1")
        else:
            monkeypatch.delenv("NRG_ORDERED_ONLY", raising=False)
        m = gpu.Model(3000, 400, gpu.NRG_ISING, O.ising_lambda(3000, 400))
        m.generate_ising(mean_deg=4.0, seed=2)
        m.reset_counters()
        objs = [m.gcd_iteration(it, kappa=2.0, seed=5)[0]["objective"] for it in range(3)]
        return m.get_state(), objs, m.kernel_stats()["tail_rounds"]
    st_t, obj_t, rounds = run(False)
    st_o, obj_o, rounds_o = run(True)
    assert rounds > 0 and rounds_o == 0
    assert_rel(np.array(obj_t), np.array(obj_o), 1e-12, "objective per iteration")
    assert_same_couplings(st_t, st_o, tol=1e-9)
    np.testing.assert_allclose(st_t[0], st_o[0], rtol=0, atol=1e-9)


@pytest.mark.parametrize("kind", [0, 1])
def test_reconstruct_cd_vs_reference(gpu, kind):
    """reconstruct_cd (inc/reconstruct.hpp:185-207) on the device vs the compiled
    reference: all pairs in row-major order per sweep, theta pass, same trajectory."""
    rng = np.random.default_rng(8)
    n, M = 80, 120
    if kind == 0:
        X, _ = O.gen_ising(n, M, seed=6)
        lam = O.ising_lambda(n, M)
        dev = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
    else:
        A = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.05)
        X = rng.standard_normal((n, M)) + 0.5 * A @ rng.standard_normal((n, M))
        lam = 4.0
        dev = gpu.Model.from_samples(X, gpu.NRG_GAUSSIAN, lam)
    which = "ref" if O.available("ref") else "orc"
    ref = O.CpuModel(which, X, kind, lam)
    ra, ca = dev.reconstruct_cd(max_iters=5)
    rb, cb = ref.reconstruct_cd(max_iters=5)
    assert len(ra) == len(rb) and ca == cb
    np.testing.assert_array_equal(ra["candidates"], rb["candidates"])
    assert_rel(ra["objective"], rb["objective"], 1e-7, "objective per CD sweep")
    assert_rel(ra["delta"], rb["delta"], 1e-5, "delta per CD sweep")
    assert_same_couplings(dev.get_state(), ref.get_state(), tol=1e-4)


def test_packed_spin_upload_equals_int8(gpu):
    """nrg_upload_spins_packed (LSB-first rows, the Ising sample-file layout, any row
    stride >= ceil(M/8)) gives the same device samples as the int8 upload: identical
    distances and GCD iteration."""
    rng = np.random.default_rng(11)
    n, M = 300, 203
    X = np.where(rng.random((n, M)) < 0.45, -1, 1).astype(np.int8)
    lam = O.ising_lambda(n, M)
    a = gpu.Model.from_samples(X, gpu.NRG_ISING, lam)
    b = gpu.Model(n, M, gpu.NRG_ISING, lam)
    bits = np.packbits(X > 0, axis=1, bitorder="little")
    padded = np.zeros((n, bits.shape[1] + 3), np.uint8)
    padded[:, : bits.shape[1]] = bits
    padded[:, bits.shape[1] - 1] |= 0xF0  # bits past M must be ignored
    b.upload_spins_packed(padded)
    i, j = rng.integers(0, n, 3000), rng.integers(0, n, 3000)
    keep = i != j
    np.testing.assert_array_equal(a.distance(gpu.NRG_EXACT, i[keep], j[keep]),
                                  b.distance(gpu.NRG_EXACT, i[keep], j[keep]))
    ra, ca = a.gcd_iteration(0, kappa=2.0, seed=3, want_candidates=True)
    rb, cb = b.gcd_iteration(0, kappa=2.0, seed=3, want_candidates=True)
    np.testing.assert_array_equal(ca, cb)
    assert ra["objective"] == rb["objective"]


def test_device_tail_walk_equals_host_walk(gpu, monkeypatch):
    """The tie-tail round's walk on the device (tail_walk_kernel) applies exactly the pairs
    the host walk applied (NRG_HOST_TAIL_WALK=1): identical reconstructions, bitwise."""
    def run(host):
        if host:
            monkeypatch.setenv("NRG_HOST_TAIL_WALK", "1")
        else:
            monkeypatch.delenv("NRG_HOST_TAIL_WALK", raising=False)
        m = gpu.Model(3000, 400, gpu.NRG_ISING, O.ising_lambda(3000, 400))
        m.generate_ising(mean_deg=4.0, seed=7)
        m.reset_counters()
        recs = [m.gcd_iteration(it, kappa=2.0, seed=5)[0] for it in range(5)]
        return m.get_state(), [(r["delta"], r["objective"]) for r in recs], m.kernel_stats()["tail_rounds"]
    a, b = run(False), run(True)
    assert a[2] > 0 and a[2] == b[2]
    assert a[1] == b[1]
    for x, y in zip(a[0], b[0]):
        np.testing.assert_array_equal(x, y)
