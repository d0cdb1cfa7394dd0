"""The N>1 path over gloo, two processes (world_size 2).

* CPU: the key-sharded distance-cache exchange planned by the library itself -- keys
  routed with nrg_key_owner, the alltoallv sizes/offsets from nrg_route_plan (the
  function exchange_and_score uses, knn.cu), the exchange over gloo -- delivers every
  request to its owner exactly once and the answers back in request order; the node
  partition (nrg_shard_range) covers each level exactly.
* GPU: the product's sharded GCD (node-sharded NNDescent, key-sharded cache, replicated
  dense levels, row all-gathers) with its collectives carried by gloo through the host
  transport (nrg_comm_init_host / TorchDistTransport): two processes on one GPU, every
  exchange host-side and blocking (no kernel waits on another rank), bitwise equal to
  the single-process run."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def pair_key(a, b):
    a, b = (a, b) if a <= b else (b, a)
    return (int(a) << 32) | int(b)


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _route_worker(rank, world, port, n, queries, out):
    _init(rank, world, port)
    from paper_2401_01404_b200 import _lib as L
    lo, hi = L.shard_range(n, rank, world)
    mine = [(i, j) for (i, j) in queries if lo <= i < hi]  # this rank's node range
    keys = np.array([pair_key(i, j) for i, j in mine], np.uint64)
    dest = np.array([L.key_owner(int(k), world) for k in keys], np.int64)
    order = np.argsort(dest, kind="stable")  # requests grouped by owner, as the device sorts them
    skeys = keys[order]
    counts = np.zeros(world * world, np.uint64)
    counts[rank * world:(rank + 1) * world] = np.bincount(dest, minlength=world)
    t = torch.from_numpy(counts.astype(np.int64))
    dist.all_reduce(t)
    sb, so, rb, ro, q = L.route_plan(world, rank, t.numpy())
    tr = L.TorchDistTransport()
    recv = np.zeros(int(q) * 8, np.uint8)
    tr.alltoallv(skeys.view(np.uint8), sb.tolist(), so.tolist(), recv, rb.tolist(), ro.tolist())
    got = recv.view(np.uint64)
    # owner side: every received key is mine; answer = key * 3 (a stand-in score)
    assert all(L.key_owner(int(k), world) == rank for k in got)
    ans = (got * np.uint64(3)).view(np.uint8)
    back = np.zeros(len(skeys) * 8, np.uint8)
    tr.alltoallv(ans, rb.tolist(), ro.tolist(), back, sb.tolist(), so.tolist())
    res = np.empty(len(keys), np.uint64)
    res[order] = back.view(np.uint64)
    out.put((rank, keys.tolist(), res.tolist(), got.tolist(), (lo, hi)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_routed_key_exchange_gloo(world):
    n = 500
    rng = np.random.default_rng(world)
    q = set()
    while len(q) < 3000:
        i, j = map(int, rng.integers(0, n, 2))
        if i != j:
            q.add((i, j))
    queries = sorted(q)
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_route_worker, args=(r, world, port, n, queries, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([out.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = []
    for _, keys, answers, got, _ in res:
        assert answers == [k * 3 for k in keys]  # every answer back, in request order
        owned += got
    assert sorted(owned) == sorted(pair_key(i, j) for i, j in queries)  # each request reached its owner once
    spans = [r[4] for r in res]
    assert spans[0][0] == 0 and spans[-1][1] == n and all(spans[t][1] == spans[t + 1][0] for t in range(world - 1))


def _gcd_worker(rank, world, port, X, lam, out):
    _init(rank, world, port)
    import paper_2401_01404_b200 as P
    m = P.Model.from_samples(X, P.NRG_ISING, lam)
    m.comm_init_host(P.TorchDistTransport())
    m.comm_selftest()  # every collective of the host transport on seeded patterns first
    m.reset_counters()
    recs = [m.gcd_iteration(it, kappa=2.0, seed=5, want_candidates=True) for it in (1, 2, 3)]
    out.put((rank, [(float(r["delta"]), float(r["objective"]), c) for r, c in recs], m.get_state(),
             m.counters()["misses"]))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_gcd_over_gloo_host_transport(gpu):
    X, _ = O.gen_ising(1500, 400, seed=6)
    X = X.astype(np.int8)
    lam = O.ising_lambda(1500, 400)
    single = gpu.Model.from_samples(X, gpu.NRG_ISING, lam)
    single.reset_counters()
    ref = [single.gcd_iteration(it, kappa=2.0, seed=5, want_candidates=True) for it in (1, 2, 3)]
    ref_state, ref_misses = single.get_state(), single.counters()["misses"]
    del single
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gcd_worker, args=(r, 2, port, X, lam, out)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([out.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, recs, st, _ in res:
        for (delta, obj, cand), (rrec, rcand) in zip(recs, ref):
            np.testing.assert_array_equal(cand, rcand)
            assert delta == rrec["delta"] and obj == rrec["objective"]
        for a, b in zip(st, ref_state):
            np.testing.assert_array_equal(a, b)
    assert sum(r[3] for r in res) == ref_misses
