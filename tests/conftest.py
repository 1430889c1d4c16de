import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libbdlora.so")
    config.addinivalue_line("markers", "slow: long-running (full-size sampled parity)")


def pytest_collection_modifyitems(config, items):
    # GPU tests are skipped (not failed) on a box without CUDA only when not explicitly selected.
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    sel = config.getoption("-m") or ""
    if "gpu" in sel and "not gpu" not in sel:
        return  # explicitly asked for gpu tests on a non-GPU box: let them fail loudly
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
