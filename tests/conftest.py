import os
import sys

import pytest

# Ranks emulated in one process (tests/test_gpu_remap_emulated.py) wait on each
# other through flags CUDA cannot see: give every stream its own hardware queue
# (set before the first CUDA call of the test process).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU and the built libzp_b200.so")
    config.addinivalue_line("markers", "reference: needs /root/reference (container only)")
