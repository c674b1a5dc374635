import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long CPU case")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Both the oracle port and the product library must be built before any test."""
    import oracle
    if not os.path.exists(oracle.PORT_SO):
        oracle.build(ref=False)
    yield
