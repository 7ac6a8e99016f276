import os
import sys

import pytest

# the GPU tests run several slot streams at once, like bench.py: give every stream its own
# hardware work queue (must be set before CUDA is initialised; bench.py sets the same)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (4K tiles)")


@pytest.fixture(scope="session")
def tile512():
    from synth.hne import make_config_tile
    return make_config_tile(1)
