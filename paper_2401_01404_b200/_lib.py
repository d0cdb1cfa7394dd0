"""ctypes binding of libnetrec_b200.so (include/netrec_b200.h).

There is no CPU fallback: importing the binding fails loudly when the CUDA library
is missing, and every call runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

# NRG_LIB: another build of the same library (A/B timing of two builds on one box)
LIB_PATH = Path(os.environ.get("NRG_LIB") or Path(__file__).resolve().parent / "libnetrec_b200.so")

NRG_ISING, NRG_GAUSSIAN = 0, 1
NRG_EXACT, NRG_GRADIENT, NRG_TABLE, NRG_LINE = 0, 1, 2, 3

PAIR_DT = np.dtype([("i", "<i4"), ("j", "<i4"), ("dist", "<f8")])
TRACE_DT = np.dtype([("level", "<i4"), ("k", "<i4"), ("exhaustive", "<i4"), ("knn_sweeps", "<i4"),
                     ("nodes", "<u8"), ("dedup_size", "<u8")])
ITER_DT = np.dtype([("iter", "<i4"), ("pad", "<i4"), ("delta", "<f8"), ("seconds", "<f8"),
                    ("candidates", "<u8"), ("objective", "<f8")])


class KnnParams(C.Structure):
    """nrg_knn_params == KnnParams (inc/knn.hpp:92-104)."""
    _fields_ = [("eps", C.c_double), ("seed", C.c_uint64), ("max_sweeps", C.c_int32),
                ("scan_floor", C.c_int32), ("width_floor", C.c_int32), ("threads", C.c_int32),
                ("reverse", C.c_int32), ("pad", C.c_int32)]


class FbParams(C.Structure):
    """nrg_fb_params == FindBestParams (inc/find_best.hpp:45-49)."""
    _fields_ = [("knn_eps", C.c_double), ("seed", C.c_uint64), ("threads", C.c_int32),
                ("reverse", C.c_int32)]


class GcdCfg(C.Structure):
    """nrg_gcd_cfg == ReconstructionConfig (inc/reconstruct.hpp:45-55)."""
    _fields_ = [("kappa", C.c_double), ("eps", C.c_double), ("max_iters", C.c_int32),
                ("mode", C.c_int32), ("knn_eps", C.c_double), ("seed", C.c_uint64),
                ("threads", C.c_int32), ("reverse", C.c_int32)]


_P = C.c_void_p
_I32P = np.ctypeslib.ndpointer(np.int32, flags="C")
_F64P = np.ctypeslib.ndpointer(np.float64, flags="C")
_U8P = np.ctypeslib.ndpointer(np.uint8, flags="C")
_I8P = np.ctypeslib.ndpointer(np.int8, flags="C")
_PAIRP = np.ctypeslib.ndpointer(PAIR_DT, flags="C")
_TRP = np.ctypeslib.ndpointer(TRACE_DT, flags="C")
_ITP = np.ctypeslib.ndpointer(ITER_DT, flags="C")
_u64, _i32, _d = C.c_uint64, C.c_int32, C.c_double
_VP = C.c_void_p

SIGNATURES = {
    "nrg_last_error": (C.c_char_p, []),
    "nrg_version": (C.c_int, []),
    "nrg_create": (C.c_int, [C.POINTER(_P), _i32, _i32, _i32, _d, _i32]),
    "nrg_destroy": (C.c_int, [_P]),
    "nrg_upload_samples": (C.c_int, [_P, _F64P]),
    "nrg_upload_spins_i8": (C.c_int, [_P, _I8P]),
    "nrg_upload_spins_packed": (C.c_int, [_P, C.c_void_p, C.c_uint64]),
    "nrg_reset_state": (C.c_int, [_P]),
    "nrg_set_theta": (C.c_int, [_P, _F64P]),
    "nrg_set_edges": (C.c_int, [_P, _u64, _I32P, _I32P, _F64P]),
    "nrg_get_state": (C.c_int, [_P, _F64P, _u64, _I32P, _I32P, _F64P, C.POINTER(_u64)]),
    "nrg_get_sums": (C.c_int, [_P, _F64P]),
    "nrg_begin_generation": (C.c_int, [_P]),
    "nrg_log_posterior": (C.c_int, [_P, C.POINTER(_d)]),
    "nrg_distance": (C.c_int, [_P, _i32, _u64, _I32P, _I32P, _F64P]),
    "nrg_optimize_edge": (C.c_int, [_P, _u64, _I32P, _I32P, _VP, _VP, _VP]),
    "nrg_edge_gradient": (C.c_int, [_P, _u64, _I32P, _I32P, _F64P]),
    "nrg_optimize_theta": (C.c_int, [_P, _F64P]),
    "nrg_set_table": (C.c_int, [_P, _u64, _F64P]),
    "nrg_set_line": (C.c_int, [_P, _u64, _F64P]),
    "nrg_find_knn": (C.c_int, [_P, _i32, _i32, _I32P, _u64, C.POINTER(KnnParams), _i32, _I32P, _F64P,
                               C.POINTER(_i32), C.POINTER(_i32), _F64P, _i32, C.POINTER(_i32)]),
    "nrg_find_best": (C.c_int, [_P, _i32, _u64, _I32P, _u64, C.POINTER(FbParams), _i32, _PAIRP, _u64,
                                C.POINTER(_u64), _TRP, _i32, C.POINTER(_i32), C.POINTER(_i32)]),
    "nrg_apply_updates": (C.c_int, [_P, _PAIRP, _u64, C.POINTER(_d)]),
    "nrg_theta_pass": (C.c_int, [_P]),
    "nrg_gcd_iteration": (C.c_int, [_P, C.POINTER(GcdCfg), _i32, _ITP, _VP, _u64, C.POINTER(_u64)]),
    "nrg_reconstruct_gcd": (C.c_int, [_P, C.POINTER(GcdCfg), _ITP, _i32, C.POINTER(_i32), C.POINTER(_i32)]),
    "nrg_reconstruct_cd": (C.c_int, [_P, _d, _i32, _i32, _ITP, _i32, C.POINTER(_i32), C.POINTER(_i32)]),
    "nrg_counters": (C.c_int, [_P, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "nrg_reset_counters": (C.c_int, [_P]),
    "nrg_recall_curve": (C.c_int, [_u64, _PAIRP, _PAIRP, _F64P]),
    "nrg_phase_times": (C.c_int, [_P, _F64P, _i32]),
    "nrg_timer": (C.c_int, [_P, _i32, C.POINTER(_d)]),
    "nrg_kernel_stats": (C.c_int, [_P, _F64P, _i32]),
    "nrg_sample_scored_pairs": (C.c_int, [_P, _u64, _u64, _I32P, _I32P, C.POINTER(_u64)]),
    "nrg_generate_ising": (C.c_int, [_P, _d, _d, _d, _i32, _i32, _u64, _VP]),
    "nrg_generated_truth": (C.c_int, [_P, _u64, _VP, _VP, _VP, _VP, C.POINTER(_u64)]),
    "nrg_generate_ising_powerlaw": (C.c_int, [_P, _d, _i32, _d, _d, _i32, _i32, _u64, _VP]),
    "nrg_generate_ising_graph": (C.c_int, [_P, _u64, _I32P, _I32P, _F64P, _F64P, _i32, _i32, _u64, _VP]),
    "nrg_generate_gaussian": (C.c_int, [_P, _i32, _d, _i32, _i32, _u64, _VP]),
    "nrg_generate_gaussian_graph": (C.c_int, [_P, _u64, _I32P, _I32P, _F64P, _F64P, _i32, _i32, _u64, _VP]),
    "nrg_write_samples_file": (C.c_int, [C.c_char_p, _i32, _i32, _i32, _F64P]),
    "nrg_read_samples_info": (C.c_int, [C.c_char_p, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "nrg_read_samples_file": (C.c_int, [C.c_char_p, _F64P]),
    "nrg_load_samples_file": (C.c_int, [_P, C.c_char_p]),
    "nrg_save_samples_file": (C.c_int, [_P, C.c_char_p]),
    "nrg_write_state_file": (C.c_int, [C.c_char_p, _i32, _F64P, _u64, _I32P, _I32P, _F64P]),
    "nrg_read_state_info": (C.c_int, [C.c_char_p, C.POINTER(_i32), C.POINTER(_u64)]),
    "nrg_read_state_file": (C.c_int, [C.c_char_p, _F64P, _I32P, _I32P, _F64P]),
    "nrg_load_state_file": (C.c_int, [_P, C.c_char_p]),
    "nrg_save_state_file": (C.c_int, [_P, C.c_char_p]),
    "nrg_comm_unique_id": (C.c_int, [C.c_char_p]),
    "nrg_comm_init": (C.c_int, [_P, C.c_char_p, _i32, _i32]),
    "nrg_loopback_create": (C.c_int, [_i32, C.POINTER(_VP)]),
    "nrg_loopback_destroy": (C.c_int, [_VP]),
    "nrg_comm_init_loopback": (C.c_int, [_P, _VP, _i32]),
    "nrg_comm_selftest": (C.c_int, [_P]),
    "nrg_comm_init_host": (C.c_int, [_P, C.c_void_p, _i32, _i32]),
    "nrg_route_plan": (C.c_int, [_i32, _i32, np.ctypeslib.ndpointer(np.uint64, flags="C"),
                                 np.ctypeslib.ndpointer(np.uint64, flags="C"), np.ctypeslib.ndpointer(np.uint64, flags="C"),
                                 np.ctypeslib.ndpointer(np.uint64, flags="C"), np.ctypeslib.ndpointer(np.uint64, flags="C"),
                                 C.POINTER(_u64)]),
    "nrg_shard_range": (C.c_int, [_u64, _i32, _i32, C.POINTER(_u64), C.POINTER(_u64)]),
    "nrg_key_owner": (_i32, [_u64, _i32]),
}

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load the CUDA library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2401_01404_b200.build`")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


ERRORS = {22: ValueError, 34: IndexError, 75: OverflowError}


def check(rc: int) -> None:
    if rc:
        msg = load().nrg_last_error().decode()
        raise ERRORS.get(rc, RuntimeError)(msg)


def _i32a(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64a(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def write_samples_file(path, X, kind=0):
    """Binary sample file (bit-packed +-1 for kind 0, f64 for kind 1)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    check(load().nrg_write_samples_file(str(path).encode(), X.shape[0], X.shape[1], kind, X))


def read_samples_file(path):
    n, m, k = _i32(), _i32(), _i32()
    check(load().nrg_read_samples_info(str(path).encode(), C.byref(n), C.byref(m), C.byref(k)))
    X = np.zeros((n.value, m.value))
    check(load().nrg_read_samples_file(str(path).encode(), X))
    return X, k.value


def write_state_file(path, theta, ei, ej, w):
    theta, ei, ej, w = _f64a(theta), _i32a(ei), _i32a(ej), _f64a(w)
    check(load().nrg_write_state_file(str(path).encode(), len(theta), theta, len(ei), ei, ej, w))


def read_state_file(path):
    n, ne = _i32(), _u64()
    check(load().nrg_read_state_info(str(path).encode(), C.byref(n), C.byref(ne)))
    th = np.zeros(n.value)
    k = ne.value
    ei, ej, w = np.zeros(max(k, 1), np.int32), np.zeros(max(k, 1), np.int32), np.zeros(max(k, 1))
    check(load().nrg_read_state_file(str(path).encode(), th, ei, ej, w))
    return th, ei[:k], ej[:k], w[:k]


class Model:
    """One device-resident GCD problem: PseudoLikelihood + SparseWeights + SampleMatrix +
    DistanceCache (inc/model.hpp:107-124) on one B200."""

    def __init__(self, n: int, M: int, kind: int = NRG_ISING, lam: float = 0.0, device: int = 0):
        self.L = load()
        h = C.c_void_p()
        check(self.L.nrg_create(C.byref(h), n, M, kind, float(lam), device))
        self.h = h
        self.n, self.M, self.kind, self.lam = n, M, kind, lam

    @classmethod
    def from_samples(cls, X, kind=NRG_ISING, lam=0.0, theta=None, device=0):
        X = np.asarray(X)
        m = cls(X.shape[0], X.shape[1], kind, lam, device)
        if X.dtype == np.int8:
            m.upload_spins_i8(X)
        else:
            m.upload_samples(X)
        if theta is not None:
            m.set_theta(theta)
        return m

    def close(self):
        if getattr(self, "h", None):
            self.L.nrg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- samples / state
    def upload_samples(self, X):
        check(self.L.nrg_upload_samples(self.h, _f64a(X)))

    def upload_spins_i8(self, X):
        check(self.L.nrg_upload_spins_i8(self.h, np.ascontiguousarray(X, dtype=np.int8)))

    def upload_spins_packed(self, bits):
        """bits: uint8 [N][row_bytes], LSB-first (numpy.packbits(X > 0, axis=1, bitorder='little'))"""
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        check(self.L.nrg_upload_spins_packed(self.h, bits.ctypes.data, bits.shape[1]))

    def generate_ising(self, mean_deg=4.0, w_sigma=0.3, th_sigma=0.1, burn_in=1000, thin=10, seed=0,
                       want_samples=False):
        out = np.zeros((self.n, self.M), np.int8) if want_samples else None
        check(self.L.nrg_generate_ising(self.h, mean_deg, w_sigma, th_sigma, burn_in, thin, seed,
                                        out.ctypes.data if out is not None else None))
        return out

    def generate_ising_powerlaw(self, gamma=2.5, dmin=2, w_sigma=0.2, th_sigma=0.1, burn_in=1000, thin=10, seed=0,
                                want_samples=False):
        out = np.zeros((self.n, self.M), np.int8) if want_samples else None
        check(self.L.nrg_generate_ising_powerlaw(self.h, gamma, dmin, w_sigma, th_sigma, burn_in, thin, seed,
                                                 out.ctypes.data if out is not None else None))
        return out

    def generate_ising_graph(self, ei, ej, w, theta, burn_in=1000, thin=10, seed=0, want_samples=False):
        ei, ej, w, theta = _i32a(ei), _i32a(ej), _f64a(w), _f64a(theta)
        out = np.zeros((self.n, self.M), np.int8) if want_samples else None
        check(self.L.nrg_generate_ising_graph(self.h, len(ei), ei, ej, w, theta, burn_in, thin, seed,
                                              out.ctypes.data if out is not None else None))
        return out

    def generate_gaussian_graph(self, ei, ej, kij, kdiag, burn_in=1000, thin=10, seed=0, want_samples=False):
        ei, ej, kij, kdiag = _i32a(ei), _i32a(ej), _f64a(kij), _f64a(kdiag)
        out = np.zeros((self.n, self.M)) if want_samples else None
        check(self.L.nrg_generate_gaussian_graph(self.h, len(ei), ei, ej, kij, kdiag, burn_in, thin, seed,
                                                 out.ctypes.data if out is not None else None))
        return out

    def generate_gaussian(self, degree=4, amp=0.2, burn_in=1000, thin=10, seed=0, want_samples=False):
        out = np.zeros((self.n, self.M)) if want_samples else None
        check(self.L.nrg_generate_gaussian(self.h, degree, amp, burn_in, thin, seed,
                                           out.ctypes.data if out is not None else None))
        return out

    def generated_truth(self):
        """(ei, ej, w, node) of the last generate_* call: couplings and fields (Ising) or
        precision off-diagonals and diagonal (Gaussian)."""
        ne = _u64()
        check(self.L.nrg_generated_truth(self.h, 0, None, None, None, None, C.byref(ne)))
        k = ne.value
        ei, ej, w, node = np.zeros(max(k, 1), np.int32), np.zeros(max(k, 1), np.int32), np.zeros(max(k, 1)), \
            np.zeros(self.n)
        check(self.L.nrg_generated_truth(self.h, k, ei.ctypes.data, ej.ctypes.data, w.ctypes.data, node.ctypes.data,
                                         C.byref(ne)))
        return ei[:k], ej[:k], w[:k], node

    def load_samples_file(self, path):
        check(self.L.nrg_load_samples_file(self.h, str(path).encode()))

    def save_samples_file(self, path):
        check(self.L.nrg_save_samples_file(self.h, str(path).encode()))

    def load_state_file(self, path):
        check(self.L.nrg_load_state_file(self.h, str(path).encode()))

    def save_state_file(self, path):
        check(self.L.nrg_save_state_file(self.h, str(path).encode()))

    def reset_state(self):
        check(self.L.nrg_reset_state(self.h))

    def set_theta(self, th):
        check(self.L.nrg_set_theta(self.h, _f64a(th)))

    def set_edges(self, ei, ej, w):
        ei, ej, w = _i32a(ei), _i32a(ej), _f64a(w)
        check(self.L.nrg_set_edges(self.h, len(ei), ei, ej, w))

    def get_state(self):
        th = np.zeros(self.n)
        ne = _u64(0)
        check(self.L.nrg_get_state(self.h, th, 0, np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1),
                                   C.byref(ne)))
        k = ne.value
        ei = np.zeros(max(k, 1), np.int32)
        ej = np.zeros(max(k, 1), np.int32)
        w = np.zeros(max(k, 1))
        check(self.L.nrg_get_state(self.h, th, k, ei, ej, w, C.byref(ne)))
        if ne.value != k:
            raise RuntimeError(f"get_state: {ne.value} couplings, {k} counted")
        return th, ei[:k], ej[:k], w[:k]

    def get_sums(self):
        out = np.zeros((self.n, self.M))
        check(self.L.nrg_get_sums(self.h, out))
        return out

    def begin_generation(self):
        check(self.L.nrg_begin_generation(self.h))

    def log_posterior(self) -> float:
        v = _d()
        check(self.L.nrg_log_posterior(self.h, C.byref(v)))
        return v.value

    def set_table(self, table):
        t = _f64a(table)
        check(self.L.nrg_set_table(self.h, t.shape[0], t))

    def set_line(self, pos):
        p = _f64a(pos)
        check(self.L.nrg_set_line(self.h, len(p), p))

    # ---- pair scores
    def distance(self, mode, i, j):
        i, j = _i32a(i), _i32a(j)
        out = np.zeros(len(i))
        check(self.L.nrg_distance(self.h, mode, len(i), i, j, out))
        return out

    def optimize_edge(self, i, j):
        i, j = _i32a(i), _i32a(j)
        w, g, warn = np.zeros(len(i)), np.zeros(len(i)), np.zeros(len(i), np.uint8)
        check(self.L.nrg_optimize_edge(self.h, len(i), i, j, w.ctypes.data, g.ctypes.data, warn.ctypes.data))
        return w, g, warn

    def edge_gradient(self, i, j):
        i, j = _i32a(i), _i32a(j)
        g = np.zeros(len(i))
        check(self.L.nrg_edge_gradient(self.h, len(i), i, j, g))
        return g

    def optimize_theta(self):
        out = np.zeros(self.n)
        check(self.L.nrg_optimize_theta(self.h, out))
        return out

    # ---- search
    def find_knn(self, mode, k, nodes, eps=1e-3, seed=0, max_sweeps=100, scan_floor=8, width_floor=4,
                 threads=1, exhaustive=False, reverse=False):
        nodes = _i32a(nodes)
        n = len(nodes)
        p = KnnParams(eps, seed, max_sweeps, scan_floor, width_floor, threads, int(reverse), 0)
        ids = np.zeros(n * max(k, 1), np.int32)
        dists = np.zeros(n * max(k, 1))
        kk, sw, nc = _i32(), _i32(), _i32()
        churn = np.zeros(max_sweeps + 1)
        check(self.L.nrg_find_knn(self.h, mode, k, nodes, n, C.byref(p), int(exhaustive), ids, dists,
                                  C.byref(kk), C.byref(sw), churn, len(churn), C.byref(nc)))
        k2 = kk.value
        return ids[: n * k2].reshape(n, k2), dists[: n * k2].reshape(n, k2), sw.value, churn[: nc.value].copy()

    def find_best(self, mode, m, nodes, knn_eps=1e-3, seed=0, threads=1, exhaustive=False, reverse=False):
        nodes = _i32a(nodes)
        n = len(nodes)
        cap = int(min(m, n * (n - 1) // 2)) + 1
        out = np.zeros(cap, PAIR_DT)
        tr = np.zeros(64, TRACE_DT)
        p = FbParams(knn_eps, seed, threads, int(reverse))
        nout, nl, sc = _u64(), _i32(), _i32()
        check(self.L.nrg_find_best(self.h, mode, m, nodes, n, C.byref(p), int(exhaustive), out, cap,
                                   C.byref(nout), tr, 64, C.byref(nl), C.byref(sc)))
        return out[: nout.value].copy(), tr[: nl.value].copy(), bool(sc.value)

    # ---- updates / driver
    def apply_updates(self, pairs) -> float:
        p = np.ascontiguousarray(pairs, dtype=PAIR_DT)
        d = _d()
        check(self.L.nrg_apply_updates(self.h, p, len(p), C.byref(d)))
        return d.value

    def theta_pass(self):
        check(self.L.nrg_theta_pass(self.h))

    def gcd_iteration(self, it, kappa=1.0, eps=-1.0, mode=NRG_EXACT, knn_eps=1e-3, seed=0, reverse=False,
                      want_candidates=False):
        cfg = GcdCfg(kappa, eps, 1, mode, knn_eps, seed, 1, int(reverse))
        rec = np.zeros(1, ITER_DT)
        cap = int(max(1, round(kappa * self.n))) + 1 if want_candidates else 0
        cand = np.empty(max(cap, 1), PAIR_DT)  # filled by the call (a fresh array: no copy on return)
        nc = _u64()
        check(self.L.nrg_gcd_iteration(self.h, C.byref(cfg), it, rec, cand.ctypes.data if cap else None, cap,
                                       C.byref(nc)))
        return rec[0], (cand[: min(nc.value, cap)] if cap else None)

    def reconstruct_gcd(self, kappa=1.0, eps=-1.0, max_iters=1000, mode=NRG_EXACT, knn_eps=1e-3, seed=0,
                        reverse=False):
        cfg = GcdCfg(kappa, eps, max_iters, mode, knn_eps, seed, 1, int(reverse))
        recs = np.zeros(max(max_iters, 1), ITER_DT)
        ni, cv = _i32(), _i32()
        check(self.L.nrg_reconstruct_gcd(self.h, C.byref(cfg), recs, len(recs), C.byref(ni), C.byref(cv)))
        return recs[: ni.value].copy(), bool(cv.value)

    def reconstruct_cd(self, eps=-1.0, max_iters=1000, threads=1):
        recs = np.zeros(max(max_iters, 1), ITER_DT)
        ni, cv = _i32(), _i32()
        check(self.L.nrg_reconstruct_cd(self.h, eps, max_iters, threads, recs, len(recs), C.byref(ni), C.byref(cv)))
        return recs[: ni.value].copy(), bool(cv.value)

    def counters(self):
        v = [_u64() for _ in range(4)]
        check(self.L.nrg_counters(self.h, *[C.byref(x) for x in v]))
        return dict(misses=v[0].value, hits=v[1].value, evals=v[2].value, warnings=v[3].value)

    def reset_counters(self):
        check(self.L.nrg_reset_counters(self.h))

    def timer_start(self):
        check(self.L.nrg_timer(self.h, 0, None))

    def timer_stop(self) -> float:
        v = _d()
        check(self.L.nrg_timer(self.h, 1, C.byref(v)))
        return v.value

    def kernel_stats(self):
        out = np.zeros(11)
        check(self.L.nrg_kernel_stats(self.h, out, 11))
        keys = ["k1_ms", "k1_launches", "k1_pairs", "k2_ms", "k2_launches", "k2_pairs", "launches", "tail_rounds",
                "tc_launches", "tc_pairs", "cache_flushes"]
        return dict(zip(keys, out.tolist()))

    def sample_scored_pairs(self, cap, seed=0):
        i = np.zeros(max(cap, 1), np.int32)
        j = np.zeros(max(cap, 1), np.int32)
        n = _u64()
        check(self.L.nrg_sample_scored_pairs(self.h, cap, seed, i, j, C.byref(n)))
        return i[: n.value].copy(), j[: n.value].copy()

    def comm_init(self, uid: bytes, rank: int, world: int):
        """Join an NCCL job (uid from comm_unique_id() on rank 0)."""
        check(self.L.nrg_comm_init(self.h, uid, rank, world))

    def comm_selftest(self):
        """Run every collective of the installed communicator on seeded patterns (all
        ranks call it); on a single-GPU context, on a one-rank NCCL communicator."""
        check(self.L.nrg_comm_selftest(self.h))

    def comm_init_host(self, transport: "HostTransport"):
        """Join a sharded job whose collectives run over a host transport (e.g.
        TorchDistTransport: any torch.distributed backend, gloo included)."""
        check(self.L.nrg_comm_init_host(self.h, C.byref(transport.struct), transport.rank, transport.world))
        self._transport = transport  # the callbacks must outlive the context's use of them

    def comm_init_loopback(self, group, rank: int):
        check(self.L.nrg_comm_init_loopback(self.h, group, rank))

    def phase_times(self):
        out = np.zeros(7)
        check(self.L.nrg_phase_times(self.h, out, 7))
        names = ["score", "knn", "select", "update", "theta", "logpost", "snapshot"]
        return dict(zip(names, out.tolist()))


_AGV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, _u64, C.c_void_p, C.POINTER(_u64))
_A2A = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(_u64), C.POINTER(_u64), C.c_void_p, C.POINTER(_u64),
                   C.POINTER(_u64))
_ARU = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(_u64), _i32, _i32)
_BCF = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), _i32)


class _HostTransportStruct(C.Structure):
    """nrg_host_transport (include/netrec_b200.h)"""
    _fields_ = [("user", C.c_void_p), ("allgatherv", _AGV), ("alltoallv", _A2A), ("allreduce_u64", _ARU),
                ("bcast_f64", _BCF)]


class HostTransport:
    """Base of a host transport: subclasses implement the four collectives on numpy
    views of the host buffers the library hands over."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world
        self._cbs = (_AGV(self._agv), _A2A(self._a2a), _ARU(self._aru), _BCF(self._bcf))
        self.struct = _HostTransportStruct(None, *self._cbs)

    @staticmethod
    def _view(ptr, n):
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(max(int(n), 1),))[: int(n)] \
            if n else np.zeros(0, np.uint8)

    def _agv(self, _u, send, sbytes, recv, rbytes):
        try:
            rb = [int(rbytes[r]) for r in range(self.world)]
            self.allgatherv(self._view(send, sbytes), self._view(recv, sum(rb)), rb)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    def _a2a(self, _u, send, sb, so, recv, rb, ro):
        try:
            w = self.world
            sb_, so_, rb_, ro_ = ([int(a[r]) for r in range(w)] for a in (sb, so, rb, ro))
            st = max((o + b for o, b in zip(so_, sb_)), default=0)
            rt = max((o + b for o, b in zip(ro_, rb_)), default=0)
            self.alltoallv(self._view(send, st), sb_, so_, self._view(recv, rt), rb_, ro_)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def _aru(self, _u, v, n, is_max):
        try:
            a = np.ctypeslib.as_array(v, shape=(int(n),))
            a[:] = self.allreduce_u64(a.copy(), bool(is_max))
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def _bcf(self, _u, v, n):
        try:
            a = np.ctypeslib.as_array(v, shape=(int(n),))
            a[:] = self.bcast_f64(a.copy())
            return 0
        except Exception:  # noqa: BLE001
            return 1


class TorchDistTransport(HostTransport):
    """The sharded path's collectives over torch.distributed on CPU tensors (gloo, or
    any backend with CPU send/recv): a multi-process / multi-node job without NCCL."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        super().__init__(dist.get_rank(group), dist.get_world_size(group))

    def allgatherv(self, send, recv, rbytes):
        import torch
        mx = max(rbytes)
        buf = torch.zeros(max(mx, 1), dtype=torch.uint8)
        buf[: len(send)] = torch.from_numpy(send.copy())
        parts = [torch.zeros_like(buf) for _ in range(self.world)]
        self.dist.all_gather(parts, buf, group=self.group)
        off = 0
        for r, b in enumerate(rbytes):
            recv[off:off + b] = parts[r][:b].numpy()
            off += b

    def alltoallv(self, send, sb, so, recv, rb, ro):
        import torch
        reqs, bufs = [], []
        for r in range(self.world):
            if r == self.rank:
                recv[ro[r]:ro[r] + rb[r]] = send[so[r]:so[r] + sb[r]]
                continue
            if sb[r]:
                reqs.append(self.dist.isend(torch.from_numpy(send[so[r]:so[r] + sb[r]].copy()), r, group=self.group))
            if rb[r]:
                t = torch.zeros(rb[r], dtype=torch.uint8)
                bufs.append((r, t))
                reqs.append(self.dist.irecv(t, r, group=self.group))
        for q in reqs:
            q.wait()
        for r, t in bufs:
            recv[ro[r]:ro[r] + rb[r]] = t.numpy()

    def allreduce_u64(self, v, is_max):
        import torch
        t = torch.from_numpy(v.astype(np.int64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if is_max else self.dist.ReduceOp.SUM, group=self.group)
        return t.numpy().astype(np.uint64)

    def bcast_f64(self, v):
        import torch
        t = torch.from_numpy(v.copy())
        self.dist.broadcast(t, 0, group=self.group)
        return t.numpy()


def route_plan(world: int, rank: int, counts):
    """alltoallv plan of one key exchange (nrg_route_plan): (send_bytes, send_off,
    recv_bytes, recv_off, n_recv) for `rank` from the world x world count matrix."""
    cnt = np.ascontiguousarray(counts, dtype=np.uint64).reshape(-1)
    out = [np.zeros(world, np.uint64) for _ in range(4)]
    q = _u64()
    check(load().nrg_route_plan(world, rank, cnt, *out, C.byref(q)))
    return (*out, q.value)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    lo, hi = _u64(), _u64()
    check(load().nrg_shard_range(n, rank, world, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def key_owner(key: int, world: int) -> int:
    return int(load().nrg_key_owner(key, world))


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(load().nrg_comm_unique_id(buf))
    return buf.raw


class LoopbackGroup:
    """In-process group of virtual ranks (one host thread per rank)."""

    def __init__(self, world: int):
        self.L = load()
        h = C.c_void_p()
        check(self.L.nrg_loopback_create(world, C.byref(h)))
        self.h = h
        self.world = world

    def close(self):
        if self.h:
            self.L.nrg_loopback_destroy(self.h)
            self.h = None


def recall_curve(exact, approx):
    e = np.ascontiguousarray(exact, dtype=PAIR_DT)
    a = np.ascontiguousarray(approx, dtype=PAIR_DT)
    out = np.zeros(len(e))
    check(load().nrg_recall_curve(len(e), e, a, out))
    return out
