"""The screen's A/B switches leave the distances unchanged (M = 1000: the pipelined K1):
  * the 4-bit first pass (default) vs the int8-only screen (NRG_K1_NO4=1): bitwise — a
    pair the 4-bit bound prunes is a proven kink pair, every other pair takes the
    unchanged int8 path;
  * the CTA-per-survivor K2 (default) vs the warp-per-survivor K2 (NRG_K2_WARP=1): the
    same fp64 arithmetic in another reduction order, so equal to rounding (1e-12 rel).
Each variant runs in its own process (the switches are read once per process)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent


def _run(tmp_path, name, env_extra):
    out = tmp_path / f"{name}.npz"
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, str(HERE / "k1_passes_script.py"), str(out)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return dict(np.load(out))


def test_k1_four_bit_pass_and_k2_cta_match(tmp_path):
    base = _run(tmp_path, "default", {})
    no4 = _run(tmp_path, "no4", {"NRG_K1_NO4": "1"})
    warp = _run(tmp_path, "warp", {"NRG_K2_WARP": "1"})
    assert (base["i"] == no4["i"]).all() and (base["j"] == warp["j"]).all()
    assert int(base["edges"]) > 0
    d = base["d"]
    unpruned = d != d.max()
    assert unpruned.sum() > 100, "the list must exercise K2"
    np.testing.assert_array_equal(d, no4["d"])
    np.testing.assert_allclose(warp["d"], d, rtol=1e-12, atol=0)
