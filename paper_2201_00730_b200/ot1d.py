"""Exact balanced 1-D OT (Algorithm 1) on the B200 (mirror of src/ot1d.py).

``solve_ot_1d(a, b, cost)`` keeps the reference signature and returns
``(SparsePlan, DualPair)``; the oracle runs in ``csrc/fw1d.cu`` (merge of
cumulative masses + prefix sums of cost differences, one CTA per problem).
``solve_ot_1d_batched`` takes device tensors for many problems at once.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .duality import DualPair
from .exceptions import MassBalanceError
from .measures import ExplicitMatrix, PowerDistance, check_submodular

MASS_TOL = 1e-9  # src/ot1d.py:27


@dataclass(frozen=True)
class SparsePlan:
    """Monotone plan as (i, j, mass) triplets (src/ot1d.py:34-89)."""

    source_idx: np.ndarray
    target_idx: np.ndarray
    mass: np.ndarray

    def __post_init__(self):
        si = np.ascontiguousarray(np.asarray(self.source_idx, dtype=np.int64))
        ti = np.ascontiguousarray(np.asarray(self.target_idx, dtype=np.int64))
        ms = np.ascontiguousarray(np.asarray(self.mass, dtype=np.float64))
        if si.ndim != 1 or not (si.shape == ti.shape == ms.shape):
            raise ValueError("plan columns must be equally sized vectors")
        if (ms <= 0).any():
            raise ValueError("plan masses must be positive")
        if (si < 0).any() or (ti < 0).any():
            raise ValueError("plan indices must be nonnegative")
        if si.size > 1:
            di, dj = np.diff(si), np.diff(ti)
            if (di < 0).any() or (dj < 0).any() or ((di == 0) & (dj == 0)).any():
                raise ValueError("plan support must be monotone without repeats")
        for arr in (si, ti, ms):
            arr.flags.writeable = False
        object.__setattr__(self, "source_idx", si)
        object.__setattr__(self, "target_idx", ti)
        object.__setattr__(self, "mass", ms)

    def __len__(self):
        return int(self.mass.size)

    @property
    def total_mass(self):
        return float(self.mass.sum())

    def row_sums(self, n):
        return np.bincount(self.source_idx, weights=self.mass, minlength=n).astype(np.float64)

    def col_sums(self, m):
        return np.bincount(self.target_idx, weights=self.mass, minlength=m).astype(np.float64)

    def to_dense(self, n, m):
        out = np.zeros((n, m))
        out[self.source_idx, self.target_idx] = self.mass
        return out

    def cost_value(self, C):
        return float(np.dot(self.mass, np.asarray(C)[self.source_idx, self.target_idx]))


def solve_ot_1d_batched(x, y, a, b, p=2.0, stream=None, C=None):
    """Device batch: x, a [B, N], y, b [B, M] (sorted supports).  Returns
    (f, g, ei, ej, em, count, status) device tensors; entries of problem k
    are ei[k, :count[k]] etc. in sweep order.  ``C`` [B, N, M] (optional)
    is an explicit Monge cost used instead of |x - y|^p."""
    t = D.torch()
    lib = _lib.load()
    x, y, a, b = (D.to_dev(v, t.float64) for v in (x, y, a, b))
    if x.ndim == 1:
        x, y, a, b = (v.unsqueeze(0) for v in (x, y, a, b))
    B, n = x.shape
    m = y.shape[1]
    f = D.empty((B, n), t.float64)
    g = D.empty((B, m), t.float64)
    ei = D.empty((B, n + m - 1), t.int32)
    ej = D.empty((B, n + m - 1), t.int32)
    em = D.empty((B, n + m - 1), t.float64)
    count = D.empty((B,), t.int32)
    status = D.empty((B,), t.int32)
    if C is not None:
        C = D.to_dev(C, t.float64).reshape(B, n, m).contiguous()
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_ot1d_workspace_size(B, n, m, ctypes.byref(size)))
    ws = D.workspace(size.value)
    _lib.check(lib.uot_ot1d_batched(
        B, n, m, _lib.ptr(x), _lib.ptr(y), _lib.ptr(a), _lib.ptr(b),
        _lib.COST_POWER if C is None else _lib.COST_EXPLICIT, ctypes.c_double(p),
        None if C is None else _lib.ptr(C), _lib.ptr(f), _lib.ptr(g), _lib.ptr(ei), _lib.ptr(ej),
        _lib.ptr(em), _lib.ptr(count), _lib.ptr(status), _lib.ptr(ws),
        ctypes.c_size_t(size.value), _lib.stream_handle(stream)), "uot_ot1d_batched")
    return f, g, ei, ej, em, count, status


def solve_ot_1d(a, b, cost=PowerDistance(2.0)):
    """Balanced 1-D OT between sorted measures of equal mass (src/ot1d.py:112-172).

    Returns ``(plan, duals)``; raises MassBalanceError when the masses differ
    by more than 1e-9 relative."""
    ma, mb = a.mass, b.mass
    if abs(ma - mb) > MASS_TOL * max(ma, mb):
        raise MassBalanceError(f"balanced solver needs equal masses, got {ma:.12g} and {mb:.12g}")
    if isinstance(cost, ExplicitMatrix):
        if cost.matrix.shape != (len(a), len(b)):
            raise ValueError(f"explicit cost shape {cost.matrix.shape} does not match supports "
                             f"({len(a)}, {len(b)})")
        check_submodular(cost.matrix)
        f, g, ei, ej, em, count, status = solve_ot_1d_batched(
            a.points, b.points, a.weights, b.weights, C=cost.matrix)
    elif isinstance(cost, PowerDistance):
        f, g, ei, ej, em, count, status = solve_ot_1d_batched(a.points, b.points, a.weights,
                                                              b.weights, cost.p)
    else:
        raise TypeError(f"unknown cost specification {cost!r}")
    if int(status[0].item()) != 0:
        raise MassBalanceError("balanced solver needs equal masses")
    k = int(count[0].item())
    plan = SparsePlan(D.to_np(ei[0, :k]), D.to_np(ej[0, :k]), D.to_np(em[0, :k]))
    return plan, DualPair(D.to_np(f[0]), D.to_np(g[0]))


def check_complementary_slackness(plan, d, C, tol=1e-9):
    """f_i + g_j = C_ij on the support and f + g <= C (src/ot1d.py:175-185);
    host-side validation helper."""
    C = np.asarray(C, dtype=np.float64)
    spread = d.f[:, None] + d.g[None, :] - C
    if float(spread.max()) > tol:
        return False
    on = spread[plan.source_idx, plan.target_idx]
    return bool(np.abs(on).max(initial=0.0) <= tol)


# File formats (paper_2201_00730_b200/formats.py), re-exported where the reference defines them.


def write_plan_csv(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.write_plan_csv`."""
    from . import formats as _F

    return _F.write_plan_csv(*args, **kwargs)


def read_plan_csv(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.read_plan_csv`."""
    from . import formats as _F

    return _F.read_plan_csv(*args, **kwargs)
