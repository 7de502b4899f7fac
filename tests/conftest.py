import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT in sys.path:
    sys.path.remove(ROOT)
sys.path.insert(0, ROOT)  # the repo's own `tests`/`oracle` packages win over site-packages


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long CPU test")


def gpu_count() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle
