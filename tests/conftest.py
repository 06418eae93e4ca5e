import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libflexlink.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    oracle.build()
    return oracle

# Loopback worlds put 3 streams per emulated rank on one device; give every
# stream its own hardware queue (must be set before CUDA initialises).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# Peer waits give up after FLX_TIMEOUT_S (product default 600 s, PyTorch's NCCL
# timeout); the suite fails fast instead if a protocol ever stalls.
os.environ.setdefault("FLX_TIMEOUT_S", "30")
os.environ.setdefault("FLX_BOOT_TIMEOUT", "120")
