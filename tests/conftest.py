"""Shared fixtures.  `-m gpu` tests need a B200 and the built CUDA library; everything
else runs on the CPU (oracle vs golden vectors, boundary/symbol checks, host logic,
gloo multi-process tests)."""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and libnetrec_b200.so")
    config.addinivalue_line("markers", "slow: larger GPU parity cases")


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    """Build the C checker if missing (gcc only; never the product)."""
    so = ROOT / "oracle" / "_build" / "libnrg_oracle.so"
    if not so.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle"], check=True, capture_output=True)
    yield


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return dict(np.load(GOLDEN / f"{name}.npz"))
    return load


@pytest.fixture(scope="session")
def gpu():
    """The product library on cuda:0 (fails loudly if it cannot run)."""
    import paper_2401_01404_b200 as P
    P.load()
    return P
