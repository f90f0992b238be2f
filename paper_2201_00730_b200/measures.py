"""Measures and ground costs (src/measures.py:38-145), plus point clouds.

``DiscreteMeasure`` keeps the reference contract: atoms sorted by position
(stable), exact duplicate positions merged by summing weights, nonnegative
weights with a positive finite total, read-only storage.  ``SqEuclideanPoints``
is new: a squared-Euclidean cost between d-dimensional point clouds that the
kernels evaluate on the fly (BASELINE configs 3 and 4 need it; the reference
can only express them through a dense ExplicitMatrix).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def _finite_vector(values, label):
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError(f"{label} must be one-dimensional")
    if arr.size == 0:
        raise ValueError(f"{label} must hold at least one entry")
    if not np.isfinite(arr).all():
        raise ValueError(f"{label} must be finite")
    return arr


def _frozen(arr):
    arr = np.ascontiguousarray(arr)
    arr.flags.writeable = False
    return arr


class DiscreteMeasure:
    """Weighted atoms on the real line with strictly increasing positions."""

    __slots__ = ("points", "weights")

    def __init__(self, points, weights):
        x = _finite_vector(points, "points")
        w = _finite_vector(weights, "weights")
        if x.shape != w.shape:
            raise ValueError("points and weights must have equal length")
        if (w < 0).any():
            raise ValueError("weights must be nonnegative")
        perm = np.argsort(x, kind="stable")
        x, w = x[perm], w[perm]
        if x.size > 1 and (np.diff(x) == 0.0).any():
            x, inv = np.unique(x, return_inverse=True)
            w = np.bincount(inv, weights=w, minlength=x.size)
        mass = float(w.sum())
        if not (math.isfinite(mass) and mass > 0):
            raise ValueError("total mass must be positive and finite")
        self.points = _frozen(x)
        self.weights = _frozen(w)

    def __len__(self):
        return int(self.points.size)

    def __repr__(self):
        return f"DiscreteMeasure(n={len(self)}, mass={self.mass:.6g})"

    @property
    def mass(self):
        return float(self.weights.sum())

    def prune_zeros(self):
        keep = self.weights > 0
        return DiscreteMeasure(self.points[keep], self.weights[keep])


@dataclass(frozen=True)
class PowerDistance:
    """c(x, y) = |x - y|**p, p >= 1 (submodular on sorted supports)."""

    p: float = 2.0

    def __post_init__(self):
        if not (math.isfinite(self.p) and self.p >= 1):
            raise ValueError("exponent p must satisfy p >= 1")


@dataclass(frozen=True)
class ExplicitMatrix:
    """Dense user-supplied cost with finite entries."""

    matrix: np.ndarray

    def __post_init__(self):
        m = np.asarray(self.matrix, dtype=np.float64)
        if m.ndim != 2:
            raise ValueError("explicit cost must be a 2-D matrix")
        if not np.isfinite(m).all():
            raise ValueError("cost entries must be finite")
        object.__setattr__(self, "matrix", _frozen(m))


@dataclass(frozen=True)
class SqEuclideanPoints:
    """C_ij = |X_i - Y_j|^2 between point clouds X (N x d), Y (M x d), never
    materialised: the kernels evaluate it tile by tile."""

    X: np.ndarray
    Y: np.ndarray

    def __post_init__(self):
        X = np.asarray(self.X, dtype=np.float64)
        Y = np.asarray(self.Y, dtype=np.float64)
        X = X.reshape(len(X), -1) if X.ndim == 1 else X
        Y = Y.reshape(len(Y), -1) if Y.ndim == 1 else Y
        if X.ndim != 2 or Y.ndim != 2 or X.shape[1] != Y.shape[1]:
            raise ValueError("point clouds must be (N, d) and (M, d) with equal d")
        if not (np.isfinite(X).all() and np.isfinite(Y).all()):
            raise ValueError("point coordinates must be finite")
        object.__setattr__(self, "X", _frozen(X))
        object.__setattr__(self, "Y", _frozen(Y))

    @property
    def d(self):
        return int(self.X.shape[1])


def check_submodular(C, tol=None):
    """Adjacent Monge check (src/measures.py:148-165); host-side validation."""
    from .exceptions import SubmodularityError

    C = np.asarray(C, dtype=np.float64)
    if C.shape[0] < 2 or C.shape[1] < 2:
        return
    if tol is None:
        tol = 1e-12 * max(1.0, float(np.abs(C).max()))
    worst = float((C[:-1, 1:] + C[1:, :-1] - C[:-1, :-1] - C[1:, 1:]).min())
    if worst < -tol:
        raise SubmodularityError(f"cost matrix is not submodular (worst adjacent minor {worst:.3e})")


def build_cost_matrix(a, b, cost):
    """Dense C[i, j] = c(x_i, y_j) (src/measures.py:125-145): computed on the
    device for PowerDistance (uot_cost_matrix); ExplicitMatrix returns the
    stored matrix after the shape check.  Returns a read-only numpy array."""
    if isinstance(cost, PowerDistance):
        from . import _device as D
        from . import _lib

        t = D.torch()
        lib = _lib.load()
        x = D.to_dev(a.points, t.float64)
        y = D.to_dev(b.points, t.float64)
        C = D.empty((len(a), len(b)), t.float64)
        _lib.check(lib.uot_cost_matrix(len(a), len(b), _lib.ptr(x), _lib.ptr(y), float(cost.p),
                                       _lib.ptr(C), _lib.stream_handle()), "uot_cost_matrix")
        return D.to_np(C)
    if isinstance(cost, ExplicitMatrix):
        if cost.matrix.shape != (len(a), len(b)):
            raise ValueError(f"explicit cost shape {cost.matrix.shape} does not match supports "
                             f"({len(a)}, {len(b)})")
        return cost.matrix
    raise TypeError(f"unknown cost specification {cost!r}")


def cost_quadruple_diameter(C):
    """max over index quadruples of C[j,k] + C[i,l] - C[j,l] - C[i,k]
    (src/measures.py:168-184): per column pair the range of the
    column-difference vector, O(N M^2) on the device."""
    from . import _device as D
    from . import _lib

    t = D.torch()
    if isinstance(C, t.Tensor):
        Cd = C.to(device=D.device(), dtype=t.float64).contiguous()
    else:
        Cn = np.asarray(C, dtype=np.float64)
        if Cn.ndim != 2:
            raise ValueError("cost must be a 2-D matrix")
        if not np.all(np.isfinite(Cn)):
            raise ValueError("cost entries must be finite")
        Cd = D.to_dev(Cn, t.float64)
    if Cd.ndim != 2:
        raise ValueError("cost must be a 2-D matrix")
    lib = _lib.load()
    out = D.empty((1,), t.float64)
    _lib.check(lib.uot_cost_quadruple_diameter(Cd.shape[0], Cd.shape[1], _lib.ptr(Cd), _lib.ptr(out),
                                               _lib.stream_handle()), "uot_cost_quadruple_diameter")
    return float(out.item())


# File formats (paper_2201_00730_b200/formats.py), re-exported where the reference defines them.


def read_measure_csv(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.read_measure_csv`."""
    from . import formats as _F

    return _F.read_measure_csv(*args, **kwargs)


def write_measure_csv(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.write_measure_csv`."""
    from . import formats as _F

    return _F.write_measure_csv(*args, **kwargs)


def read_measure_json(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.read_measure_json`."""
    from . import formats as _F

    return _F.read_measure_json(*args, **kwargs)


def write_measure_json(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.write_measure_json`."""
    from . import formats as _F

    return _F.write_measure_json(*args, **kwargs)


def measure_to_csv_text(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.measure_to_csv_text`."""
    from . import formats as _F

    return _F.measure_to_csv_text(*args, **kwargs)
