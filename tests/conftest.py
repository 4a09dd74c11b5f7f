import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def api():
    from paper_2107_11650_b200 import api as A
    return A


@pytest.fixture(scope="session")
def gpu(api):
    if api.device_count() < 1:
        pytest.fail("GPU test collected on a host without a CUDA device")
    return api
