import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built libcoexb200.so")


_BACKENDS = {}


@pytest.fixture(scope="session")
def b200_factory():
    """Session-wide B200 backends keyed by precision (one CUDA context each)."""
    from paper_2201_09210_b200.b200 import B200Backend

    def make(precision="f64", fresh=False):
        if fresh:
            return B200Backend(precision=precision, timeout_s=60.0)
        if precision not in _BACKENDS:
            _BACKENDS[precision] = B200Backend(precision=precision, timeout_s=60.0)
        return _BACKENDS[precision]

    return make
