"""Marginal penalties and the entropy-family functions (src/entropies.py).

KL(rho), Berg(rho) and Balanced keep the reference's types and validation.
logdotexp, softmin, conj, conj_grad, conj_hess, aprox and divergence run on
the device (uot_logdotexp / uot_entropy_map / uot_divergence); they accept
scalars or arrays like the reference and return floats for scalars.  The
Sinkhorn kernels run all three penalties; the FW solvers run KL.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


def _check_rho(rho):
    if not (isinstance(rho, (int, float)) and math.isfinite(rho) and rho > 0):
        raise ValueError("rho must be positive and finite")


@dataclass(frozen=True)
class KL:
    """KL marginal penalty rho * KL(. | nu), rho > 0."""

    rho: float = 1.0

    def __post_init__(self):
        _check_rho(self.rho)


@dataclass(frozen=True)
class Berg:
    """Berg marginal penalty rho * (sum log(nu/mu) ...): F and G Sinkhorn steps
    run it on the device (aprox by per-element Newton, lambda* by Newton)."""

    rho: float = 1.0

    def __post_init__(self):
        _check_rho(self.rho)


@dataclass(frozen=True)
class Balanced:
    """Hard marginal constraint (aprox = identity): F Sinkhorn steps only."""


def ent_code(spec):
    """UOT_ENT_* code of an entropy spec (include/uot_b200.h)."""
    from .exceptions import UnsupportedEntropyError

    if isinstance(spec, KL):
        return 0
    if isinstance(spec, Berg):
        return 1
    if isinstance(spec, Balanced):
        return 2
    raise UnsupportedEntropyError(f"unknown entropy {spec!r}")


def ent_rho(spec):
    return float(getattr(spec, "rho", 1.0))


def require_kl(*specs, what="this solver"):
    from .exceptions import UnsupportedEntropyError

    for s in specs:
        if not isinstance(s, KL):
            raise UnsupportedEntropyError(f"{what} runs KL penalties on the B200 path, got {s!r}")


# ---------------------------------------------------------------------------
# Device-backed entropy functions (src/entropies.py:67-263).

_BALANCED_EQ_TOL = 1e-9


def _dev():
    from . import _device as D
    from . import _lib

    return D, _lib, _lib.load()


def logdotexp(values, weights, axis=None):
    """Stabilised log(sum_i w_i exp(v_i)) with zero-weight entries masked
    before the max shift; with ``axis`` the weights run along that axis and
    the reduction is vectorised over the others.  -inf when every weight is
    zero (src/entropies.py:67-92)."""
    import numpy as np

    D, L, lib = _dev()
    t = D.torch()
    v = np.asarray(values, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64).reshape(-1)
    if axis is None:
        vv = v.reshape(-1)
        if vv.size != w.size:
            raise ValueError("values and weights must have equal length")
        outer, k, inner = 1, w.size, 1
    else:
        ax = axis % v.ndim
        if v.shape[ax] != w.size:
            raise ValueError("weights must run along the reduced axis")
        outer = int(np.prod(v.shape[:ax], dtype=np.int64))
        k = v.shape[ax]
        inner = int(np.prod(v.shape[ax + 1:], dtype=np.int64))
        vv = np.ascontiguousarray(v)
    if k == 0:
        res = np.full((outer * inner,), -np.inf)
    else:
        dv, dw = D.to_dev(vv, t.float64), D.to_dev(w, t.float64)
        out = D.empty((outer * inner,), t.float64)
        L.check(lib.uot_logdotexp(outer, k, inner, L.ptr(dv), L.ptr(dw), 1.0, L.ptr(out),
                                  L.stream_handle()), "uot_logdotexp")
        res = D.to_np(out, readonly=False)
    if axis is None:
        return float(res[0])
    return res.reshape(v.shape[:ax] + v.shape[ax + 1:])


def softmin(a, eps, f):
    """-eps log <a, e^(-f/eps)> over the measure's weights (src/entropies.py:187-200)."""
    import numpy as np

    if eps <= 0:
        raise ValueError("eps must be positive")
    f = np.asarray(f, dtype=np.float64)
    if f.shape != a.weights.shape:
        raise ValueError("potential length must match the measure")
    if not np.all(np.isfinite(f)):
        raise ValueError("potential must be finite")
    D, L, lib = _dev()
    t = D.torch()
    dv, dw = D.to_dev(f, t.float64), D.to_dev(a.weights, t.float64)
    out = D.empty((1,), t.float64)
    L.check(lib.uot_logdotexp(1, f.size, 1, L.ptr(dv), L.ptr(dw), -1.0 / eps, L.ptr(out),
                              L.stream_handle()), "uot_logdotexp")
    return -eps * float(out.item())


def _emap(op, spec, x, eps=0.0):
    import numpy as np

    from .exceptions import UnsupportedEntropyError

    if not isinstance(spec, (KL, Berg, Balanced)):
        raise UnsupportedEntropyError(f"unknown entropy {spec!r}")
    x = np.asarray(x, dtype=np.float64)
    D, L, lib = _dev()
    t = D.torch()
    flat = np.ascontiguousarray(x.reshape(-1))
    dx = D.to_dev(flat, t.float64)
    out = D.empty((flat.size,), t.float64)
    bad = t.zeros((1,), dtype=t.int32, device=out.device)
    L.check(lib.uot_entropy_map(op, ent_code(spec), ent_rho(spec), float(eps), flat.size,
                                L.ptr(dx), L.ptr(out), L.ptr(bad), L.stream_handle()),
            "uot_entropy_map")
    if int(bad.item()) != 0:
        raise ValueError("Berg conjugate requires x < rho")
    res = D.to_np(out, readonly=False).reshape(x.shape)
    return float(res) if res.ndim == 0 else res


def conj(spec, x):
    """Legendre transform phi*(x) (src/entropies.py:142-156)."""
    return _emap(0, spec, x)


def conj_grad(spec, x):
    """Derivative of the conjugate, the marginals' reweighting factor (:157-171)."""
    return _emap(1, spec, x)


def conj_hess(spec, x):
    """Second derivative of the conjugate (:172-184)."""
    return _emap(2, spec, x)


def aprox(spec, eps, x):
    """argmin_y eps e^((x-y)/eps) + phi*(y): KL scales by rho/(eps+rho),
    Balanced is the identity, Berg is the per-element safeguarded Newton
    (src/entropies.py:203-263)."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    return _emap(3, spec, x, eps)


def phi_prime_inf(spec):
    """Recession slope of phi: inf for KL and Balanced, rho for Berg (:95-101)."""
    from .exceptions import UnsupportedEntropyError

    if isinstance(spec, (KL, Balanced)):
        return math.inf
    if isinstance(spec, Berg):
        return spec.rho
    raise UnsupportedEntropyError(f"unknown entropy {spec!r}")


def divergence(spec, mu, nu):
    """Csiszar divergence sum_{nu>0} phi(mu/nu) nu + phi'_inf sum_{nu=0} mu,
    +inf where the reference returns +inf (src/entropies.py:104-140)."""
    import numpy as np

    from .exceptions import UnsupportedEntropyError

    mu = np.asarray(mu, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    if mu.shape != nu.shape:
        raise ValueError("mu and nu must have equal length")
    if np.any(mu < 0) or np.any(nu < 0):
        raise ValueError("weights must be nonnegative")
    if not isinstance(spec, (KL, Berg, Balanced)):
        raise UnsupportedEntropyError(f"unknown entropy {spec!r}")
    D, L, lib = _dev()
    t = D.torch()
    n = int(mu.size)
    dm = D.to_dev(mu.reshape(-1), t.float64) if n else None
    dn = D.to_dev(nu.reshape(-1), t.float64) if n else None
    out = D.empty((1,), t.float64)
    L.check(lib.uot_divergence(ent_code(spec), ent_rho(spec), n, L.ptr(dm), L.ptr(dn), L.ptr(out),
                               L.stream_handle()), "uot_divergence")
    return float(out.item())
