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
        # Long full-size / multi-process runs (bench under torchrun, full-size
        # partition invariance; ~3 min together on a B200) can be skipped with
        # PLANC_B200_SKIP_SLOW=1.
        if os.environ.get("PLANC_B200_SKIP_SLOW") == "1":
            skip_slow = pytest.mark.skip(reason="slow: PLANC_B200_SKIP_SLOW=1")
            for it in items:
                if "slow" in it.keywords:
                    it.add_marker(skip_slow)
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
