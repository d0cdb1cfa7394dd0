"""The N>1 host logic on CPU with two gloo processes: the library's own partition
functions (nrg_shard_range, nrg_key_owner) drive the key-sharded distance-cache
protocol of the sharded NNDescent (requests routed to the key's owner, owner dedups and
scores, answers routed back) and the per-sweep row all-gather; the C checker supplies
the pair scores.  Checks: every rank gets the checker's distance for each of its
queries, each unique pair is scored exactly once job-wide, and the gathered rows equal
the single-process result."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
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


def _worker(rank, world, port, X, lam, queries, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_01404_b200 import _lib as L
    n = X.shape[0]
    lo, hi = L.shard_range(n, rank, world)
    # this rank's candidates: queries of its own node range (as the gather kernel makes)
    mine = [(i, j) for (i, j) in queries if lo <= i < hi]
    local, remote = [], {r: [] for r in range(world)}
    for (i, j) in mine:
        k = pair_key(i, j)
        o = L.key_owner(k, world)
        (local if o == rank else remote[o]).append(k)
    # request exchange (all-to-all of keys)
    sent = [None] * world
    dist.all_gather_object(sent, {r: remote[r] for r in range(world)})
    incoming = [k for r in range(world) for k in sent[r].get(rank, [])]
    # owner: dedup in this rank's cache shard, score each new key once
    m = O.CpuModel("orc", X, 0, lam)
    m.begin_generation()
    keys = sorted(set(local) | set(incoming))
    vals = {}
    if keys:
        ki = np.array([k >> 32 for k in keys], np.int32)
        kj = np.array([k & 0xffffffff for k in keys], np.int32)
        for k, d in zip(keys, m.distance(0, ki, kj)):
            vals[k] = d
    scored = m.counters()["misses"]
    # answers back
    answers = [None] * world
    dist.all_gather_object(answers, {k: vals[k] for k in incoming})
    got = {}
    for (i, j) in mine:
        k = pair_key(i, j)
        o = L.key_owner(k, world)
        got[(i, j)] = vals[k] if o == rank else answers[o][k]
    # row all-gather: each rank contributes rows [lo, hi) of a per-node table
    rows = [None] * world
    dist.all_gather_object(rows, (lo, hi, [int(i) * 7 for i in range(lo, hi)]))
    out.put((rank, got, scored, rows, (lo, hi)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_key_sharded_cache_protocol_gloo(world):
    X, _ = O.gen_ising(120, 80, seed=3, burn_in=100, thin=3)
    lam = O.ising_lambda(120, 80)
    rng = np.random.default_rng(0)
    q = set()
    while len(q) < 900:
        i, j = map(int, rng.integers(0, 120, 2))
        if i != j:
            q.add((i, j))
            if rng.random() < 0.4:
                q.add((j, i))  # probed from both endpoints, as NNDescent does
    queries = sorted(q)
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, lam, queries, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([out.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = O.CpuModel("orc", X, 0, lam)
    ref.begin_generation()
    qi = np.array([a for a, _ in queries], np.int32)
    qj = np.array([b for _, b in queries], np.int32)
    truth = dict(zip(queries, ref.distance(0, qi, qj)))
    covered = {}
    for _, got, _, _, _ in res:
        covered.update(got)
    assert covered == truth  # every query answered with the checker's value, bitwise
    unique = len({pair_key(a, b) for a, b in queries})
    assert sum(r[2] for r in res) == unique  # each unique pair scored once job-wide
    # partition covers [0, n) exactly; the gathered table equals the single-process one
    spans = [r[4] for r in res]
    assert spans[0][0] == 0 and spans[-1][1] == 120 and all(spans[t][1] == spans[t + 1][0] for t in range(world - 1))
    for _, _, _, rows, _ in res:
        table = [v for (_, _, part) in rows for v in part]
        assert table == [i * 7 for i in range(120)]
