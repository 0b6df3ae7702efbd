import os
import sys

import pytest

# the emulated-rank exchange tests (test_gpu_exchange_emulated.py) run up to
# 16 streams of one process whose kernels wait on each other (bounded waits):
# give every stream its own hardware queue so none is falsely serialised
# behind another's waiting kernel (must be set before CUDA initialises)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libsagips.so")
    config.addinivalue_line("markers", "slow: long CPU test")
