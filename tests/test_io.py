"""Binary sample / state files: host-side round trips (CPU) and the
context load/save path (GPU).  The drop-in library must load for the CPU tests."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2401_01404_b200 import _lib as L


def test_sample_file_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    Xi = np.where(rng.random((37, 203)) < 0.5, -1.0, 1.0)
    L.write_samples_file(tmp_path / "a.bin", Xi, kind=0)
    Y, k = L.read_samples_file(tmp_path / "a.bin")
    assert k == 0
    np.testing.assert_array_equal(Y, Xi)
    assert (tmp_path / "a.bin").stat().st_size == 32 + 37 * 26  # bit-packed rows
    Xg = rng.standard_normal((11, 17))
    L.write_samples_file(tmp_path / "g.bin", Xg, kind=1)
    Y, k = L.read_samples_file(tmp_path / "g.bin")
    assert k == 1
    np.testing.assert_array_equal(Y, Xg)


def test_state_file_round_trip(tmp_path):
    th = np.linspace(-1, 1, 9)
    ei, ej, w = np.array([0, 2, 5], np.int32), np.array([3, 7, 8], np.int32), np.array([0.5, -0.25, 1e-3])
    L.write_state_file(tmp_path / "s.bin", th, ei, ej, w)
    a, b, c, d = L.read_state_file(tmp_path / "s.bin")
    np.testing.assert_array_equal(a, th)
    np.testing.assert_array_equal(b, ei)
    np.testing.assert_array_equal(c, ej)
    np.testing.assert_array_equal(d, w)


def test_io_errors(tmp_path):
    with pytest.raises(ValueError):
        L.write_samples_file(tmp_path / "x.bin", np.array([[0.5, 1.0]]), kind=0)  # not +-1
    (tmp_path / "junk.bin").write_bytes(b"not a netrec file at all")
    with pytest.raises(ValueError):
        L.read_samples_file(tmp_path / "junk.bin")
    with pytest.raises(RuntimeError):
        L.read_samples_file(tmp_path / "missing.bin")


@pytest.mark.gpu
def test_context_load_save(gpu, tmp_path):
    import oracle_lib as O
    X, _ = O.gen_ising(300, 150, seed=2)
    lam = O.ising_lambda(300, 150)
    L.write_samples_file(tmp_path / "x.bin", X, kind=0)
    a = gpu.Model(300, 150, gpu.NRG_ISING, lam)
    a.load_samples_file(tmp_path / "x.bin")
    b = gpu.Model.from_samples(X.astype(np.int8), gpu.NRG_ISING, lam)
    a.gcd_iteration(0, kappa=2.0, seed=1)
    b.gcd_iteration(0, kappa=2.0, seed=1)
    a.save_state_file(tmp_path / "s.bin")
    a.save_samples_file(tmp_path / "x2.bin")
    np.testing.assert_array_equal(L.read_samples_file(tmp_path / "x2.bin")[0], X)
    c = gpu.Model(300, 150, gpu.NRG_ISING, lam)
    c.load_samples_file(tmp_path / "x2.bin")
    c.load_state_file(tmp_path / "s.bin")
    for s_a, s_b, s_c in zip(a.get_state(), b.get_state(), c.get_state()):
        np.testing.assert_array_equal(s_a, s_b)
        np.testing.assert_array_equal(s_a, s_c)
    assert abs(a.log_posterior() - c.log_posterior()) <= 1e-9 * abs(a.log_posterior())


def test_failed_write_keeps_previous_file(tmp_path):
    """Writes are atomic (the reference's atomic_write, inc/io.hpp): an invalid input is
    rejected before the target is touched, and no temporary is left behind."""
    rng = np.random.default_rng(1)
    Xi = np.where(rng.random((5, 9)) < 0.5, -1.0, 1.0)
    L.write_samples_file(tmp_path / "a.bin", Xi, kind=0)
    before = (tmp_path / "a.bin").read_bytes()
    bad = Xi.copy()
    bad[4, 8] = 0.5  # the last value is invalid: nothing may be written
    with pytest.raises(ValueError):
        L.write_samples_file(tmp_path / "a.bin", bad, kind=0)
    assert (tmp_path / "a.bin").read_bytes() == before
    assert not (tmp_path / "a.bin.tmp").exists()
    with pytest.raises(RuntimeError):  # unwritable directory: the error surfaces, nothing created
        L.write_state_file(tmp_path / "no" / "dir" / "s.bin", np.zeros(3), [], [], [])


def test_corrupt_headers_rejected_before_allocation(tmp_path):
    """A state / sample header whose counts disagree with the file length is rejected
    (no multi-GB allocation from a corrupt n_edges)."""
    th = np.zeros(4)
    L.write_state_file(tmp_path / "s.bin", th, np.array([0], np.int32), np.array([1], np.int32), np.array([0.5]))
    raw = bytearray((tmp_path / "s.bin").read_bytes())
    raw[16:24] = (1 << 36).to_bytes(8, "little")  # n_edges
    (tmp_path / "bad.bin").write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        L.read_state_file(tmp_path / "bad.bin")
    (tmp_path / "short.bin").write_bytes((tmp_path / "s.bin").read_bytes()[:-3])
    with pytest.raises(ValueError):
        L.read_state_file(tmp_path / "short.bin")
    L.write_samples_file(tmp_path / "x.bin", np.ones((3, 10)), kind=0)
    (tmp_path / "x2.bin").write_bytes((tmp_path / "x.bin").read_bytes() + b"\0")
    with pytest.raises(ValueError):
        L.read_samples_file(tmp_path / "x2.bin")
