import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running GPU parity case")


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # GPU tests must FAIL (not skip) when selected with -m gpu on a box without a GPU would be
    # misleading; we only skip them when no GPU exists AND they were not explicitly requested.
    markexpr = config.getoption("-m") or ""
    if "gpu" in markexpr and "not gpu" not in markexpr:
        return
    if not _cuda_available():
        skip = pytest.mark.skip(reason="no CUDA device (GPU tests run with -m gpu on a B200)")
        for it in items:
            if "gpu" in it.keywords:
                it.add_marker(skip)
