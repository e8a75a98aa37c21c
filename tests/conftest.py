import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def native():
    """The sm_100a extension, built in-tree if stale; fails loudly without CUDA."""
    from paper_2205_11226_b200 import _native

    _native.build()
    _native.require_cuda()
    return _native.lib()
