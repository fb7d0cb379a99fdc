import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def gpu():
    """The product library on a visible B200; fails (never skips) under -m gpu."""
    from paper_2006_16423_b200 import solver
    lib = solver.load_library()
    assert lib.dsg_device_count() > 0, "no CUDA device visible to libdsg_b200.so"
    return lib
