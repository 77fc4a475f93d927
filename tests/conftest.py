import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and librkb200.so")
    config.addinivalue_line("markers", "slow: multi-second GPU property tests at full size")


@pytest.fixture(scope="session")
def golden():
    from tests import _golden

    return _golden


@pytest.fixture(scope="session")
def gpu():
    """Fails (never skips) when the CUDA path is unavailable: a GPU test that silently
    passed on a fallback would hide a missing native build."""
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_1810_01051_b200 import _lib

    lib = _lib.lib()
    assert lib.rk_device_count() > 0
    return _lib.context(0)
