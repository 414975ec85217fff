import os
import sys

import pytest

# In-process rank groups (tests/test_gpu_inproc.py) run up to 8 handles' streams concurrently on one
# GPU, each spinning on the others' exchange words: every stream needs its own hardware work queue
# (the default of 8 lets two ranks' streams share one, and a kernel queued behind another rank's
# spinning kernel never starts).  Set before any CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
