"""ctypes front-end for the CHECKERS under oracle/ (test infrastructure only).

Two libraries share one flat surface (see oracle/nrg_oracle.h):
  * ``orc`` — oracle/_build/libnrg_oracle.so, the plain-C restatement;
  * ``ref`` — oracle/_ref/libnetrec_ref.so, the unmodified reference headers
    (netrec) compiled behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline legs
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
LIB_PATHS = {
    "orc": ROOT / "oracle" / "_build" / "libnrg_oracle.so",
    "ref": ROOT / "oracle" / "_ref" / "libnetrec_ref.so",
}

PAIR_DT = np.dtype([("i", "<i4"), ("j", "<i4"), ("dist", "<f8")])
TRACE_DT = np.dtype([("level", "<i4"), ("k", "<i4"), ("exhaustive", "<i4"), ("knn_sweeps", "<i4"),
                     ("nodes", "<u8"), ("dedup_size", "<u8")])
ITER_DT = np.dtype([("iter", "<i4"), ("pad", "<i4"), ("delta", "<f8"), ("seconds", "<f8"),
                    ("candidates", "<u8"), ("objective", "<f8")])

_P = C.c_void_p
_I32P = np.ctypeslib.ndpointer(np.int32, flags="C")
_F64P = np.ctypeslib.ndpointer(np.float64, flags="C")
_U8P = np.ctypeslib.ndpointer(np.uint8, flags="C")
_U64P = np.ctypeslib.ndpointer(np.uint64, flags="C")
_PAIRP = np.ctypeslib.ndpointer(PAIR_DT, flags="C")
_TRP = np.ctypeslib.ndpointer(TRACE_DT, flags="C")
_ITP = np.ctypeslib.ndpointer(ITER_DT, flags="C")
_u64 = C.c_uint64
_i = C.c_int
_d = C.c_double

_SIGS = {
    "last_error": (C.c_char_p, []),
    "create": (_i, [C.POINTER(_P), _i, _i, _i, _d, _F64P, C.c_void_p]),
    "destroy": (None, [_P]),
    "set_edges": (_i, [_P, _u64, _I32P, _I32P, _F64P]),
    "set_theta": (_i, [_P, _F64P]),
    "get_state": (_i, [_P, _F64P, _u64, _I32P, _I32P, _F64P, C.POINTER(_u64)]),
    "get_sums": (_i, [_P, _F64P]),
    "log_posterior": (_i, [_P, C.POINTER(_d)]),
    "begin_generation": (None, [_P]),
    "set_table": (_i, [_P, _u64, _F64P]),
    "distance": (_i, [_P, _i, _u64, _I32P, _I32P, _F64P]),
    "optimize_edge": (_i, [_P, _u64, _I32P, _I32P, _F64P, _F64P, _U8P]),
    "edge_gradient": (_i, [_P, _u64, _I32P, _I32P, _F64P]),
    "edge_objective": (_i, [_P, C.c_int32, C.c_int32, _d, C.POINTER(_d)]),
    "optimize_theta": (_i, [_P, _F64P]),
    "find_knn": (_i, [_P, _i, _i, _I32P, _u64, _d, _u64, _i, _i, _i, _i, _i, _I32P, _F64P,
                      C.POINTER(_i), C.POINTER(_i), _F64P, _i, C.POINTER(_i)]),
    "find_best": (_i, [_P, _i, _u64, _I32P, _u64, _d, _u64, _i, _i, _PAIRP, _u64, C.POINTER(_u64),
                       _TRP, _i, C.POINTER(_i), C.POINTER(_i)]),
    "apply_updates": (_i, [_P, _u64, _PAIRP, _i, C.POINTER(_d)]),
    "theta_pass": (_i, [_P, _i]),
    "reconstruct_gcd": (_i, [_P, _d, _d, _i, _i, _d, _u64, _i, _ITP, _i, C.POINTER(_i),
                             C.POINTER(_i), C.c_void_p, _u64, C.POINTER(_u64)]),
    "reconstruct_cd": (_i, [_P, _d, _i, _i, _ITP, _i, C.POINTER(_i), C.POINTER(_i)]),
    "counters": (_i, [_P, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "recall_curve": (_i, [_u64, _PAIRP, _PAIRP, _F64P]),
    "mix64": (_u64, [_u64, _u64]),
    "rng_stream": (None, [_u64, _u64, _i, _u64, _U64P]),
}
_I8P = np.ctypeslib.ndpointer(np.int8, flags="C")
_OPTIONAL = {"gen_ising": (_i, [_i, _d, _d, _d, _i, _i, _i, _u64, C.c_void_p, _F64P, _u64, _I32P, _I32P,
                                _F64P, C.POINTER(_u64)]),
             "gen_ising_colored": (_i, [_i, _d, _d, _d, _i, _i, _i, _u64, _i, _I8P, _F64P, _u64, _I32P, _I32P,
                                        _F64P, C.POINTER(_u64)]),
             "gibbs_colored": (_i, [_i, _u64, _I32P, _I32P, _F64P, _F64P, _i, _i, _i, _u64, _i, _I8P])}

_LIBS: dict[str, C.CDLL] = {}

ERR = {22: ValueError, 34: IndexError, 75: OverflowError}


def available(which: str) -> bool:
    return LIB_PATHS[which].exists()


def lib(which: str) -> C.CDLL:
    if which not in _LIBS:
        path = LIB_PATHS[which]
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        L = C.CDLL(str(path))
        for name, (res, args) in list(_SIGS.items()) + list(_OPTIONAL.items()):
            sym = f"{which}_{name}"
            if not hasattr(L, sym):
                if name in _OPTIONAL:
                    continue
                raise AttributeError(sym)
            f = getattr(L, sym)
            f.restype = res
            f.argtypes = args
        _LIBS[which] = L
    return _LIBS[which]


def _chk(which: str, rc: int) -> None:
    if rc:
        msg = getattr(lib(which), f"{which}_last_error")().decode()
        raise ERR.get(rc, RuntimeError)(msg)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class CpuModel:
    """PseudoLikelihood + SparseWeights + DistanceCache on the CPU checker."""

    def __init__(self, which: str, X, kind: int = 0, lam: float = 0.0, theta=None):
        self.which = which
        self.L = lib(which)
        X = _f64(X)
        self.n, self.M = X.shape
        h = C.c_void_p()
        th = _f64(theta) if theta is not None else None
        rc = self._f("create")(C.byref(h), self.n, self.M, kind, float(lam), X,
                               th.ctypes.data if th is not None else None)
        _chk(which, rc)
        self.h = h
        self.kind = kind
        self.lam = lam

    def _f(self, name):
        return getattr(self.L, f"{self.which}_{name}")

    def close(self):
        if self.h:
            self._f("destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # state
    def set_edges(self, ei, ej, w):
        ei, ej, w = _i32(ei), _i32(ej), _f64(w)
        _chk(self.which, self._f("set_edges")(self.h, len(ei), ei, ej, w))

    def set_theta(self, th):
        _chk(self.which, self._f("set_theta")(self.h, _f64(th)))

    def get_state(self):
        th = np.zeros(self.n)
        ne = _u64(0)
        cap = 1 << 22
        ei = np.zeros(cap, np.int32)
        ej = np.zeros(cap, np.int32)
        w = np.zeros(cap)
        _chk(self.which, self._f("get_state")(self.h, th, cap, ei, ej, w, C.byref(ne)))
        k = ne.value
        return th, ei[:k].copy(), ej[:k].copy(), w[:k].copy()

    def get_sums(self):
        out = np.zeros((self.n, self.M))
        _chk(self.which, self._f("get_sums")(self.h, out))
        return out

    def log_posterior(self) -> float:
        v = _d()
        _chk(self.which, self._f("log_posterior")(self.h, C.byref(v)))
        return v.value

    def begin_generation(self):
        self._f("begin_generation")(self.h)

    def set_table(self, table):
        t = _f64(table)
        _chk(self.which, self._f("set_table")(self.h, t.shape[0], t))

    # pair scores
    def distance(self, mode, i, j):
        i, j = _i32(i), _i32(j)
        out = np.zeros(len(i))
        _chk(self.which, self._f("distance")(self.h, mode, len(i), i, j, out))
        return out

    def distance_parallel(self, mode, i, j, threads=None):
        """distance() under the reference's parallel_for (ref only; the C checker runs
        the same pairs serially)"""
        i, j = _i32(i), _i32(j)
        if self.which != "ref":
            return self.distance(mode, i, j)
        f = self.L.ref_distance_parallel
        f.restype = _i
        f.argtypes = [_P, _i, _u64, _I32P, _I32P, _F64P, _i]
        out = np.zeros(len(i))
        _chk(self.which, f(self.h, mode, len(i), i, j, out, int(threads or os.cpu_count() or 1)))
        return out

    def optimize_edge(self, i, j):
        i, j = _i32(i), _i32(j)
        w = np.zeros(len(i))
        g = np.zeros(len(i))
        warn = np.zeros(len(i), np.uint8)
        _chk(self.which, self._f("optimize_edge")(self.h, len(i), i, j, w, g, warn))
        return w, g, warn

    def edge_gradient(self, i, j):
        i, j = _i32(i), _i32(j)
        g = np.zeros(len(i))
        _chk(self.which, self._f("edge_gradient")(self.h, len(i), i, j, g))
        return g

    def edge_objective(self, i, j, w):
        v = _d()
        _chk(self.which, self._f("edge_objective")(self.h, int(i), int(j), float(w), C.byref(v)))
        return v.value

    def optimize_theta(self):
        out = np.zeros(self.n)
        _chk(self.which, self._f("optimize_theta")(self.h, out))
        return out

    # search
    def find_knn(self, mode, k, nodes, eps=1e-3, seed=0, max_sweeps=100, scan_floor=8,
                 width_floor=4, threads=1, exhaustive=False):
        nodes = _i32(nodes)
        n = len(nodes)
        ids = np.zeros(n * max(k, 1), np.int32)
        dists = np.zeros(n * max(k, 1))
        kk, sw, nc = _i(), _i(), _i()
        churn = np.zeros(max_sweeps + 1)
        _chk(self.which, self._f("find_knn")(self.h, mode, k, nodes, n, eps, seed, max_sweeps,
                                             scan_floor, width_floor, threads, int(exhaustive),
                                             ids, dists, C.byref(kk), C.byref(sw), churn,
                                             len(churn), C.byref(nc)))
        k2 = kk.value
        return (ids[: n * k2].reshape(n, k2), dists[: n * k2].reshape(n, k2), sw.value,
                churn[: nc.value].copy())

    def find_best(self, mode, m, nodes, knn_eps=1e-3, seed=0, threads=1, exhaustive=False):
        nodes = _i32(nodes)
        n = len(nodes)
        cap = int(min(m, n * (n - 1) // 2)) + 1
        out = np.zeros(cap, PAIR_DT)
        tr = np.zeros(64, TRACE_DT)
        nout, nl, sc = _u64(), _i(), _i()
        _chk(self.which, self._f("find_best")(self.h, mode, m, nodes, n, knn_eps, seed, threads,
                                              int(exhaustive), out, cap, C.byref(nout), tr, 64,
                                              C.byref(nl), C.byref(sc)))
        return out[: nout.value].copy(), tr[: nl.value].copy(), bool(sc.value)

    # updates
    def apply_updates(self, pairs, threads=1) -> float:
        p = np.ascontiguousarray(pairs, dtype=PAIR_DT)
        d = _d()
        _chk(self.which, self._f("apply_updates")(self.h, len(p), p, threads, C.byref(d)))
        return d.value

    def theta_pass(self, threads=1):
        _chk(self.which, self._f("theta_pass")(self.h, threads))

    def reconstruct_gcd(self, kappa=1.0, eps=-1.0, max_iters=1000, mode=0, knn_eps=1e-3, seed=0,
                        threads=1, cand_cap=0):
        recs = np.zeros(max(max_iters, 1), ITER_DT)
        ni, cv, nc = _i(), _i(), _u64()
        cand = np.zeros(max(cand_cap, 1), PAIR_DT)
        _chk(self.which, self._f("reconstruct_gcd")(self.h, kappa, eps, max_iters, mode, knn_eps,
                                                    seed, threads, recs, len(recs), C.byref(ni),
                                                    C.byref(cv),
                                                    cand.ctypes.data if cand_cap else None,
                                                    cand_cap, C.byref(nc)))
        return recs[: ni.value].copy(), bool(cv.value), cand[: nc.value].copy()

    def reconstruct_cd(self, eps=-1.0, max_iters=1000, threads=1):
        recs = np.zeros(max(max_iters, 1), ITER_DT)
        ni, cv = _i(), _i()
        _chk(self.which, self._f("reconstruct_cd")(self.h, eps, max_iters, threads, recs, len(recs), C.byref(ni),
                                                   C.byref(cv)))
        return recs[: ni.value].copy(), bool(cv.value)

    def counters(self):
        v = [_u64() for _ in range(4)]
        _chk(self.which, self._f("counters")(self.h, *[C.byref(x) for x in v]))
        return dict(misses=v[0].value, hits=v[1].value, evals=v[2].value, warnings=v[3].value)


def recall_curve(which, exact, approx):
    e = np.ascontiguousarray(exact, dtype=PAIR_DT)
    a = np.ascontiguousarray(approx, dtype=PAIR_DT)
    out = np.zeros(len(e))
    _chk(which, getattr(lib(which), f"{which}_recall_curve")(len(e), e, a, out))
    return out


def mix64(a, b, which="orc"):
    return int(getattr(lib(which), f"{which}_mix64")(a, b))


def rng_stream(seed, split, n, bound=0, which="orc"):
    out = np.zeros(n, np.uint64)
    getattr(lib(which), f"{which}_rng_stream")(seed, split, n, bound, out)
    return out


def gen_ising(n, M, seed, mean_deg=4.0, w_sigma=0.3, th_sigma=0.1, burn_in=1000, thin=10):
    """Seeded Ising instance (truth + Gibbs samples) from the C checker."""
    L = lib("orc")
    X = np.zeros((n, M))
    th = np.zeros(n)
    cap = int(n * mean_deg) + 1024
    ei = np.zeros(cap, np.int32)
    ej = np.zeros(cap, np.int32)
    w = np.zeros(cap)
    ne = _u64()
    _chk("orc", L.orc_gen_ising(n, mean_deg, w_sigma, th_sigma, M, burn_in, thin, seed, X.ctypes.data, th, cap,
                                ei, ej, w, C.byref(ne)))
    k = ne.value
    return X, dict(theta=th, i=ei[:k].copy(), j=ej[:k].copy(), w=w[:k].copy())


def gen_ising_colored(n, M, seed, mean_deg=4.0, w_sigma=0.3, th_sigma=0.1, burn_in=1000, thin=10, threads=None):
    """The device data pipeline's chain (gen.cu generate_ising) restated in C: the same
    truth as gen_ising and the coloured Gibbs chain, int8 samples [n][M]."""
    L = lib("orc")
    X = np.zeros((n, M), np.int8)
    th = np.zeros(n)
    cap = int(n * mean_deg * 1.5) + 1024
    ei = np.zeros(cap, np.int32)
    ej = np.zeros(cap, np.int32)
    w = np.zeros(cap)
    ne = _u64()
    _chk("orc", L.orc_gen_ising_colored(n, mean_deg, w_sigma, th_sigma, M, burn_in, thin, seed,
                                        int(threads or os.cpu_count() or 1), X, th, cap, ei, ej, w, C.byref(ne)))
    k = ne.value
    return X, dict(theta=th, i=ei[:k].copy(), j=ej[:k].copy(), w=w[:k].copy())


def gibbs_colored(ei, ej, w, theta, M, seed, burn_in=1000, thin=10, threads=None):
    """Coloured Gibbs samples of a given truth (gen.cu generate_ising_graph)."""
    L = lib("orc")
    n = len(theta)
    lo, hi = np.minimum(ei, ej).astype(np.int32), np.maximum(ei, ej).astype(np.int32)
    X = np.zeros((n, M), np.int8)
    _chk("orc", L.orc_gibbs_colored(n, len(lo), lo, hi, _f64(w), _f64(theta), M, burn_in, thin, seed,
                                    int(threads or os.cpu_count() or 1), X))
    return X


def ising_lambda(n: int, M: int) -> float:
    """Pinned L1 strength lambda = 2 sqrt(M ln N)."""
    return float(2.0 * np.sqrt(M * np.log(n)))


if os.environ.get("NRG_ORACLE_DEBUG"):
    print({k: available(k) for k in LIB_PATHS})
