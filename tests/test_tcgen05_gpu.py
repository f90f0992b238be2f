"""tcgen05 mechanics (TMEM A operand, canonical shared-memory B, kind::tf32)."""

import ctypes

import numpy as np
import pytest

from paper_2201_00730_b200 import _device as D
from paper_2201_00730_b200 import _lib

pytestmark = pytest.mark.gpu


def _tf32(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32)
    b = (b + 0x1000) & 0xFFFFE000  # round-to-nearest on the 13 dropped bits
    return b.view(np.float32)


@pytest.mark.parametrize("K", [8, 64, 200])
def test_tc_selftest_tile(K):
    import torch

    lib = _lib.load()
    rng = np.random.default_rng(K)
    A = _tf32(rng.standard_normal((128, K)))
    B = _tf32(rng.standard_normal((128, K)))
    a = torch.as_tensor(A, device="cuda")
    b = torch.as_tensor(B, device="cuda")
    d = torch.zeros((128, 128), dtype=torch.float32, device="cuda")
    _lib.check(lib.uot_tc_selftest(_lib.ptr(a), _lib.ptr(b), K, _lib.ptr(d), _lib.stream_handle()))
    got = D.to_np(d)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    np.testing.assert_allclose(got, ref, rtol=0, atol=2e-5 * np.sqrt(K))


@pytest.mark.parametrize("K", [8, 64, 144])
def test_tc_selftest_pair(K):
    """cta_group::2: A rows split across the pair's TMEM, B rows across its smem."""
    import torch

    lib = _lib.load()
    rng = np.random.default_rng(100 + K)
    A = _tf32(rng.standard_normal((256, K)))
    B = _tf32(rng.standard_normal((128, K)))
    a = torch.as_tensor(A, device="cuda")
    b = torch.as_tensor(B, device="cuda")
    d = torch.zeros((256, 128), dtype=torch.float32, device="cuda")
    _lib.check(lib.uot_tc_selftest2(_lib.ptr(a), _lib.ptr(b), K, _lib.ptr(d),
                                    _lib.stream_handle()))
    got = D.to_np(d)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    np.testing.assert_allclose(got, ref, rtol=0, atol=2e-5 * np.sqrt(K))
