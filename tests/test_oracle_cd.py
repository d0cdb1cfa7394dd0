"""reconstruct_cd (inc/reconstruct.hpp:185-207): the C restatement against the compiled
reference on seeded Ising and Gaussian data — same trajectory (delta, objective per
sweep) and same final couplings.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O


@pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind", [0, 1])
def test_cd_oracle_matches_reference(kind):
    rng = np.random.default_rng(3)
    n, M = 50, 80
    if kind == 0:
        X, _ = O.gen_ising(n, M, seed=5)
        lam = O.ising_lambda(n, M)
    else:
        A = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.05)
        X = rng.standard_normal((n, M)) + 0.5 * A @ rng.standard_normal((n, M))
        lam = 4.0
    a = O.CpuModel("orc", X, kind, lam)
    b = O.CpuModel("ref", X, kind, lam)
    ra, ca = a.reconstruct_cd(max_iters=6)
    rb, cb = b.reconstruct_cd(max_iters=6)
    assert ca == cb and len(ra) == len(rb)
    np.testing.assert_array_equal(ra["candidates"], rb["candidates"])
    np.testing.assert_allclose(ra["delta"], rb["delta"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(ra["objective"], rb["objective"], rtol=1e-12)
    sa, sb = a.get_state(), b.get_state()
    np.testing.assert_array_equal(sa[1], sb[1])
    np.testing.assert_array_equal(sa[2], sb[2])
    np.testing.assert_allclose(sa[3], sb[3], rtol=0, atol=1e-9)
