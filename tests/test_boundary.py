"""The drop-in boundary: libnetrec_b200.so loads, exports every symbol
include/netrec_b200.h declares, the ctypes binding covers them all, and without a GPU
the library fails loudly (no CPU fallback).  CPU only."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "netrec_b200.h"
LIB = ROOT / "paper_2401_01404_b200" / "libnetrec_b200.so"


def declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"\b(nrg_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        from paper_2401_01404_b200 import build
        build.build_lib()
    return C.CDLL(str(LIB))


def test_header_declares_the_path():
    names = declared()
    for must in ["nrg_create", "nrg_distance", "nrg_find_knn", "nrg_find_best", "nrg_apply_updates",
                 "nrg_theta_pass", "nrg_gcd_iteration", "nrg_reconstruct_gcd", "nrg_log_posterior"]:
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (nrg_[a-z0-9_]+)", out))
    assert set(declared()) <= exported


def test_binding_covers_header():
    from paper_2401_01404_b200._lib import SIGNATURES
    assert set(declared()) == set(SIGNATURES)


def test_kernels_are_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2401_01404_b200 import _lib
    with pytest.raises(RuntimeError, match="CUDA"):
        _lib.Model(10, 10, 0, 1.0)


def test_error_codes_map_to_reference_exceptions():
    from paper_2401_01404_b200._lib import ERRORS
    assert ERRORS[22] is ValueError and ERRORS[34] is IndexError and ERRORS[75] is OverflowError


@pytest.mark.skipif(not Path("/root/reference/proj/include/netrec/io.hpp").exists(),
                    reason="reference headers not present")
def test_reference_io_compiles_on_dropin_types(tmp_path):
    """the reference's own text I/O header compiles unchanged on the
    drop-in types (and round-trips a state through them)."""
    src = tmp_path / "io_dropin.cpp"
    src.write_text("""
#include "netrec_b200/netrec.hpp"
#include "netrec/io.hpp"
int main() {
    netrec::SampleMatrix x(3, 2);
    for (int i = 0; i < 3; ++i) for (int m = 0; m < 2; ++m) x.set(i, m, (i + m) % 2 ? 1.0 : -1.0);
    netrec::SparseWeights w(3, 2);
    w.set_edge(0, 2, 0.25, x);
    w.set_theta(1, -0.5);
    const std::string t = netrec::weights_to_text(w);
    return t.find("0.25") == std::string::npos;
}
""")
    out = tmp_path / "io_dropin"
    r = subprocess.run(["g++", "-std=c++20", f"-I{ROOT / 'include'}", "-I/root/reference/proj/include", str(src),
                        "-o", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert subprocess.run([str(out)]).returncode == 0
