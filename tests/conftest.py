"""Shared pytest configuration.

``-m gpu`` tests need a CUDA device and the in-tree C-ABI library; everything
else runs on the CPU (oracle pinning, host logic, ABI symbol checks, gloo).
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def golden_forwards():
    return dict(np.load(GOLDEN / "forwards.npz"))


@pytest.fixture(scope="session")
def golden_streams():
    return json.loads((GOLDEN / "streams.json").read_text())


@pytest.fixture(scope="session")
def golden_topk():
    return dict(np.load(GOLDEN / "topk_kat.npz"))


@pytest.fixture(scope="session")
def golden_budgets():
    return json.loads((GOLDEN / "budget_kat.json").read_text())


@pytest.fixture(scope="session")
def golden_weight_sigs():
    return json.loads((GOLDEN / "weights_sig.json").read_text())
