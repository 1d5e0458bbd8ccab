import os
import sys

# Ranks simulated by threads (tests/test_gpu_ep.py, test_gpu_stack.py) each launch on their own
# stream, and a rank's device flag barrier spins until every peer arrives: with the default 8
# hardware work queues two ranks' streams can share one queue, so a peer's kernels wait behind a
# spinning barrier (a false dependency that ends in the barrier's timeout).  One queue per stream.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libdymoe.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)

