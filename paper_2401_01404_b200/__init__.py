"""paper_2401_01404_b200 — B200-native GCD hot path of arXiv 2401.01404 (netrec).

The product is libnetrec_b200.so (CUDA, sm_100a) behind the C-ABI in
include/netrec_b200.h; this package holds its sources (csrc/), the build script and a
thin ctypes binding used by the tests and the benchmark.
"""
from ._lib import (  # noqa: F401
    NRG_EXACT,
    NRG_GAUSSIAN,
    NRG_GRADIENT,
    NRG_ISING,
    NRG_LINE,
    NRG_TABLE,
    PAIR_DT,
    HostTransport,
    Model,
    TorchDistTransport,
    load,
    recall_curve,
    route_plan,
)

__all__ = ["Model", "HostTransport", "TorchDistTransport", "route_plan", "load", "recall_curve", "PAIR_DT", "NRG_ISING", "NRG_GAUSSIAN", "NRG_EXACT",
           "NRG_GRADIENT", "NRG_TABLE", "NRG_LINE"]
