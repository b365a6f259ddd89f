import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels through the C-ABI)")
    config.addinivalue_line("markers", "slow: CPU test that takes tens of seconds")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Compile the native libraries in-tree if they are missing or stale."""
    from paper_2201_12050_b200 import build

    build.build_host()
    build.build_oracle()
    build.build_cuda()


def rel(a, b):
    import numpy as np

    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))
