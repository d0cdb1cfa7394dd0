"""The multi-GPU path (node-sharded NNDescent, key-sharded distance cache, row
all-gathers) verified on one GPU: W virtual ranks in one process (loopback
collectives, one host thread per rank) must reproduce the single-context results
bit for bit — kNN graphs, FindBest pairs, whole GCD iterations."""
from __future__ import annotations

import threading

import numpy as np
import pytest

import oracle_lib as O
from helpers import pairs_equal, row_sets

pytestmark = pytest.mark.gpu


def _run_ranks(world, fn):
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


def _models(gpu, X, lam, world):
    grp = gpu._lib.LoopbackGroup(world)
    ms = []
    for r in range(world):
        m = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
        m.comm_init_loopback(grp.h, r)
        ms.append(m)
    return grp, ms


@pytest.mark.parametrize("world", [2, 3, 5])
def test_comm_selftest_loopback(gpu, world):
    """Every collective of the interface on seeded patterns (ragged and empty
    contributions, a world x world count matrix) through the loopback backend."""
    X, _ = O.gen_ising(64, 64, seed=1)
    grp, ms = _models(gpu, X, 10.0, world)
    _run_ranks(world, lambda r: ms[r].comm_selftest())
    del ms, grp


def test_comm_selftest_nccl_one_rank(gpu):
    """The NCCL backend on this GPU: libnccl loads, a one-rank communicator starts, and
    its all-gather / all-reduce / broadcast calls return the expected data.  (Point-to-
    point exchanges need a second GPU; the driver's multi-GPU bench runs them.)"""
    X, _ = O.gen_ising(64, 64, seed=1)
    m = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, 10.0)
    m.comm_selftest()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_knn_and_find_best_match_single(gpu, world):
    X, _ = O.gen_ising(700, 300, seed=4)
    lam = O.ising_lambda(700, 300)
    nodes = np.arange(700, dtype=np.int32)
    single = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
    single.begin_generation()
    ref_knn = single.find_knn(gpu.NRG_EXACT, 8, nodes, seed=3)
    single.begin_generation()
    ref_fb = single.find_best(gpu.NRG_EXACT, 1400, nodes, seed=9)
    grp, ms = _models(gpu, X, lam, world)

    def work(r):
        m = ms[r]
        m.begin_generation()
        k = m.find_knn(gpu.NRG_EXACT, 8, nodes, seed=3)
        m.begin_generation()
        f = m.find_best(gpu.NRG_EXACT, 1400, nodes, seed=9)
        return k, f, m.counters()

    res = _run_ranks(world, work)
    for k, f, _ in res:
        assert row_sets(k[0]) == row_sets(ref_knn[0]) and k[2] == ref_knn[2]
        np.testing.assert_array_equal(k[1], ref_knn[1])
        assert pairs_equal(f[0], ref_fb[0])
        assert (f[1] == ref_fb[1]).all()
    # the key-sharded cache scores each unique pair once job-wide
    single.reset_counters()
    single.begin_generation()
    single.find_knn(gpu.NRG_EXACT, 8, nodes, seed=3)
    one = single.counters()["misses"]
    for m in ms:
        m.reset_counters()
    res = _run_ranks(world, lambda r: (ms[r].begin_generation(), ms[r].find_knn(gpu.NRG_EXACT, 8, nodes, seed=3),
                                       ms[r].counters())[2])
    assert sum(c["misses"] for c in res) == one
    grp.close()


def test_sharded_gcd_iterations_match_single(gpu):
    X, _ = O.gen_ising(600, 300, seed=6)
    lam = O.ising_lambda(600, 300)
    single = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
    ref = [single.gcd_iteration(it, kappa=2.0, seed=5, want_candidates=True) for it in (1, 2, 3)]
    ref_state = single.get_state()
    grp, ms = _models(gpu, X, lam, 2)

    def work(r):
        return [ms[r].gcd_iteration(it, kappa=2.0, seed=5, want_candidates=True) for it in (1, 2, 3)], \
            ms[r].get_state()

    for recs, st in _run_ranks(2, work):
        for (rec, cand), (rrec, rcand) in zip(recs, ref):
            assert pairs_equal(cand, rcand)
            assert rec["delta"] == rrec["delta"]
        np.testing.assert_array_equal(st[0], ref_state[0])
        assert (st[1] == ref_state[1]).all() and (st[2] == ref_state[2]).all()
        np.testing.assert_array_equal(st[3], ref_state[3])
    grp.close()


@pytest.mark.slow
def test_sharded_config4_sweeps_match_single(gpu):
    """Config 4 (Ising N=1e5, M=1000, lambda=214.6, kappa=2) at two virtual ranks: the
    first two GCD sweeps (the empty-state sweep, then a sweep with ~1.5e5 couplings) give
    bitwise the single-context candidate lists, deltas, objectives and states; the
    sharded job keeps the tensor-core dense levels (replicated per rank) and scores each
    unique pair once job-wide."""
    n, M = 100_000, 1000
    lam = O.ising_lambda(n, M)

    def make():
        m = gpu.Model(n, M, gpu.NRG_ISING, lam)
        m.generate_ising(mean_deg=5.0, seed=1, burn_in=200)
        return m

    single = make()
    single.reset_counters()
    ref = [single.gcd_iteration(it, kappa=2.0, seed=1, want_candidates=True) for it in (0, 1)]
    ref_state = single.get_state()
    ref_misses = single.counters()["misses"]
    ref_tc = single.kernel_stats()["tc_launches"]
    del single
    grp = gpu._lib.LoopbackGroup(2)
    ms = [make() for _ in range(2)]
    for r, m in enumerate(ms):
        m.comm_init_loopback(grp.h, r)
        m.reset_counters()

    def work(r):
        recs = [ms[r].gcd_iteration(it, kappa=2.0, seed=1, want_candidates=True) for it in (0, 1)]
        return recs, ms[r].get_state(), ms[r].counters()["misses"], ms[r].kernel_stats()["tc_launches"]

    res = _run_ranks(2, work)
    assert ref_tc > 0
    for recs, st, _, tc in res:
        assert tc == ref_tc, "the sharded job must keep the dense (tensor-core) levels"
        for (rec, cand), (rrec, rcand) in zip(recs, ref):
            assert pairs_equal(cand, rcand)
            assert rec["delta"] == rrec["delta"] and rec["objective"] == rrec["objective"]
        for a, b in zip(st, ref_state):
            np.testing.assert_array_equal(a, b)
    assert sum(r[2] for r in res) == ref_misses
    grp.close()
