import os
import sys

# CUDA lazy loading can make a kernel's first launch wait for the context to go idle, which deadlocks the
# single-GPU multi-rank tests (several ranks of one process whose streams wait on each other's device-side
# flags); load every kernel at context creation instead
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def ora():
    import oracle
    return oracle.Oracle()
