import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def cases(z):
    return [int(k) for k in z["cases"]]


def rel_err(f, g, f_ref, g_ref):
    """||delta||_inf / max(||f||_inf, ||g||_inf)."""
    scale = max(np.abs(f_ref).max(), np.abs(g_ref).max(), 1e-300)
    return max(np.abs(f - f_ref).max(), np.abs(g - g_ref).max()) / scale


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
