import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs on the GPU box")
    config.addinivalue_line("markers", "slow: long-running (full config sizes)")


@pytest.fixture(scope="session")
def G():
    """The product module (C++ drop-in API over the sm_100a kernels)."""
    from paper_2412_13269_b200 import tetris
    return tetris


@pytest.fixture(scope="session")
def R():
    """The compiled, unmodified reference (oracle/_ref); skip if not built."""
    from common import load_ref
    mod = load_ref()
    if mod is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return mod


@pytest.fixture(scope="session")
def gpu_available(G):
    if G.device_count() < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    return True
