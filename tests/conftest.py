import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        # Long full-size / multi-process runs (bench under torchrun, the
        # reference's 220-plan acceptance corpus, full-size partition
        # invariance) need PLANC_B200_SLOW_TESTS=1; their logs are committed
        # under profiles/ (the default GPU suite stays within minutes).
        if os.environ.get("PLANC_B200_SLOW_TESTS") != "1":
            skip_slow = pytest.mark.skip(reason="slow: set PLANC_B200_SLOW_TESTS=1")
            for it in items:
                if "slow" in it.keywords:
                    it.add_marker(skip_slow)
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
