"""Host <-> device helpers shared by the API mirror (torch is the allocator /
stream provider only; all arithmetic happens in the CUDA kernels)."""

from __future__ import annotations

import numpy as np


def torch():
    import torch as _t

    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        from .exceptions import UotError

        raise UotError("no CUDA device: the B200 kernels cannot run (no CPU fallback)")
    return t.device("cuda", t.cuda.current_device())


def to_dev(a, dtype):
    """numpy / torch -> contiguous CUDA tensor of ``dtype``."""
    t = torch()
    if isinstance(a, t.Tensor):
        return a.to(device=device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    if not arr.flags.writeable:  # read-only API arrays: torch wants a writable buffer
        arr = arr.copy()
    return t.as_tensor(arr, dtype=dtype, device=device()).contiguous()


def to_np(t, readonly=True):
    arr = t.detach().cpu().numpy()
    arr = np.ascontiguousarray(arr, dtype=arr.dtype)
    if readonly:
        arr.flags.writeable = False
    return arr


def empty(shape, dtype):
    return torch().empty(shape, dtype=dtype, device=device())


def workspace(nbytes):
    t = torch()
    return t.empty(max(int(nbytes), 1), dtype=t.uint8, device=device())
