"""Dual-pair / problem value types, the closed-form KL translation and the
dual objectives (src/duality.py:42-91, :117-178, :250-303).  The reductions
run in the ``uot_kl_scalars`` / ``uot_sinkhorn_verify`` kernels (no N x M
cost matrix is formed)."""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from functools import cached_property

import numpy as np

from . import _device as D
from . import _lib
from .entropies import KL, Balanced, Berg, ent_code, ent_rho, require_kl
from .exceptions import NewtonError, UnsupportedEntropyError
from .measures import DiscreteMeasure


@dataclass(frozen=True)
class DualPair:
    """Potentials (f, g) attached to the two marginals; read-only fp64."""

    f: np.ndarray
    g: np.ndarray

    def __post_init__(self):
        f = np.array(self.f, dtype=np.float64, copy=True)
        g = np.array(self.g, dtype=np.float64, copy=True)
        if f.ndim != 1 or g.ndim != 1:
            raise ValueError("potentials must be vectors")
        if not (np.isfinite(f).all() and np.isfinite(g).all()):
            raise ValueError("potentials must be finite")
        f.flags.writeable = False
        g.flags.writeable = False
        object.__setattr__(self, "f", f)
        object.__setattr__(self, "g", g)

    @staticmethod
    def zeros(n, m):
        return DualPair(np.zeros(n), np.zeros(m))


@dataclass(frozen=True)
class UotProblem:
    """One unbalanced transport instance (alpha, beta, cost, ent1, ent2, eps)."""

    alpha: DiscreteMeasure
    beta: DiscreteMeasure
    cost: object
    ent1: object
    ent2: object
    eps: float = 0.0

    def __post_init__(self):
        if not (math.isfinite(self.eps) and self.eps >= 0):
            raise ValueError("eps must be nonnegative and finite")

    @cached_property
    def cost_matrix(self):
        """Dense C (src/duality.py:85-87), built on the device on first use and
        cached; the solvers never need it (costs are formed on the fly)."""
        from .measures import build_cost_matrix

        return build_cost_matrix(self.alpha, self.beta, self.cost)

    def check_pair(self, d):
        if d.f.size != len(self.alpha) or d.g.size != len(self.beta):
            raise ValueError("potential lengths do not match the marginals")


def kl_scalars(a, b, f, g, rho1, rho2):
    """Batched (lambda*, H_0, Smin_a^{rho1}(f)) on device tensors [B, N]/[B, M]."""
    t = D.torch()
    lib = _lib.load()
    a, b, f, g = (D.to_dev(v, t.float64) for v in (a, b, f, g))
    if a.ndim == 1:
        a, b, f, g = (v.unsqueeze(0) for v in (a, b, f, g))
    out = D.empty((a.shape[0], 3), t.float64)
    st = lib.uot_kl_scalars(a.shape[0], a.shape[1], b.shape[1], _lib.ptr(a), _lib.ptr(b),
                            _lib.ptr(f), _lib.ptr(g), ctypes.c_double(rho1),
                            ctypes.c_double(rho2), _lib.ptr(out), _lib.stream_handle())
    _lib.check(st, "uot_kl_scalars")
    return out


def _strictly_convex(spec):
    return isinstance(spec, (KL, Berg))


_NEWTON_MSG = {1: "empty translation domain for Berg conjugates",
               2: "failed to bracket the optimal translation",
               3: "translation Newton did not reach the residual target"}


def translation(prob, f, g, solve=True, lam0=0.0, marginals=False, value=False, tol=1e-11,
                max_iters=100):
    """One ``uot_translation`` launch: the bracketed-Newton translation of
    (f, g) (src/duality.py:182-247) from ``lam0`` (or lam0 itself with
    ``solve=False``), optionally the updated marginals (:293-303) and the
    value <a, -phi1*(-(f + lam))> + <b, -phi2*(-(g - lam))> (:102-114).
    Returns (lam, ta, tb, h) with device tensors / None; raises NewtonError
    like the reference."""
    t = D.torch()
    lib = _lib.load()
    n, m = len(prob.alpha), len(prob.beta)
    a, b, fd, gd = (D.to_dev(v, t.float64) for v in (prob.alpha.weights, prob.beta.weights, f, g))
    lam = D.empty((1,), t.float64)
    st = D.empty((1,), t.int32)
    ta = D.empty((n,), t.float64) if marginals else None
    tb = D.empty((m,), t.float64) if marginals else None
    h = D.empty((1,), t.float64) if value else None
    _lib.check(lib.uot_translation(1, n, m, _lib.ptr(a), _lib.ptr(b), _lib.ptr(fd), _lib.ptr(gd),
                                   ent_code(prob.ent1), ent_code(prob.ent2), ent_rho(prob.ent1),
                                   ent_rho(prob.ent2), 1 if solve else 0, float(lam0),
                                   float(tol), int(max_iters), _lib.ptr(lam), _lib.ptr(ta), _lib.ptr(tb), _lib.ptr(h),
                                   _lib.ptr(st), _lib.stream_handle()), "uot_translation")
    code = int(st[0].item())
    if code:
        raise NewtonError(_NEWTON_MSG[code])
    return float(lam[0].item()), ta, tb, h


def _both_kl(prob):
    return isinstance(prob.ent1, KL) and isinstance(prob.ent2, KL)


def lambda_star(prob, d, tol=1e-11, max_iters=100, initial=0.0):
    """Optimal translation t* maximising G(f + t, g - t) (src/duality.py:160-179).

    KL/KL has the closed form rho1 rho2/(rho1+rho2) (LSE_a(-f/rho1) -
    LSE_b(-g/rho2)), evaluated on the GPU; KL/Berg mixes and Berg/Berg run the
    reference's bracketed Newton (:182-247) in ``uot_translation`` with the
    given ``tol`` / ``max_iters`` / ``initial``.  Balanced is rejected like
    the reference."""
    prob.check_pair(d)
    if not (_strictly_convex(prob.ent1) and _strictly_convex(prob.ent2)):
        raise UnsupportedEntropyError(
            "optimal translation needs strictly convex conjugates (KL or Berg)")
    if not _both_kl(prob):
        return translation(prob, d.f, d.g, True, initial, tol=tol, max_iters=max_iters)[0]
    out = kl_scalars(prob.alpha.weights, prob.beta.weights, d.f, d.g, prob.ent1.rho, prob.ent2.rho)
    return float(out[0, 0].item())


def translate(prob, d):
    """(f + t*, g - t*) (src/duality.py:250-253)."""
    lam = lambda_star(prob, d)
    return DualPair(d.f + lam, d.g - lam)


DUAL_FEAS_TOL = 1e-9  # src/duality.py:39


def _kl_parts(prob, sf, sg):
    """From the softmins S = Smin^rho_w(pot): <w, rho(1 - e^(-pot/rho))> per side
    and the coupled closed form of _eval_h_kl (duality.py:279-290)."""
    r1, r2 = prob.ent1.rho, prob.ent2.rho
    ma, mb = float(np.sum(prob.alpha.weights)), float(np.sum(prob.beta.weights))
    la, lb = -sf / r1, -sg / r2  # LSE_a(-f/r1), LSE_b(-g/r2)
    f_part = r1 * (ma - math.exp(la)) + r2 * (mb - math.exp(lb))
    h_part = r1 * ma + r2 * mb - (r1 + r2) * math.exp((r1 * la + r2 * lb) / (r1 + r2))
    return f_part, h_part, ma, mb


def dual_feasibility_violation(prob, d):
    """max(0, max_ij f_i + g_j - C_ij) (duality.py:117-121) on the device
    (1-D |x - y|^p costs and explicit matrices)."""
    from .fw import feasibility_violation
    from .measures import ExplicitMatrix, PowerDistance

    prob.check_pair(d)
    if isinstance(prob.cost, ExplicitMatrix):
        return float(feasibility_violation(prob.alpha.points, prob.beta.points, d.f, d.g,
                                           C=prob.cost.matrix)[0].item())
    if not isinstance(prob.cost, PowerDistance):
        raise UnsupportedEntropyError("the device feasibility check runs 1-D |x - y|^p costs")
    return float(feasibility_violation(prob.alpha.points, prob.beta.points, d.f, d.g,
                                       prob.cost.p)[0].item())


def _eps_term(prob, d):
    """eps (<a x b, e^((f+g-C)/eps)> - m_a m_b) (duality.py:124-132)."""
    from .sinkhorn import _step_inputs, _verify_prob, verify_batched

    if _both_kl(prob):
        v = _verify_prob(prob, d)
    else:  # the log-partition column does not depend on the penalties
        costname, p, x, y, C = _step_inputs(prob)
        v = D.to_np(verify_batched(x, y, prob.alpha.weights, prob.beta.weights, d.f, d.g,
                                   prob.eps, 1.0, 1.0, cost=costname, p=p, c=C)[0],
                    readonly=False)
    ma, mb = float(np.sum(prob.alpha.weights)), float(np.sum(prob.beta.weights))
    return prob.eps * (math.exp(v[1]) - ma * mb), v


def _check_feasible(prob, d):
    if prob.eps == 0:
        from .exceptions import InfeasibleDualError

        viol = dual_feasibility_violation(prob, d)
        if viol > DUAL_FEAS_TOL:
            raise InfeasibleDualError(f"dual constraint violated by {viol:.3e} at eps = 0")


def _eval_f_generic(prob, d):
    """<a, -phi1*(-f)> + <b, -phi2*(-g)> (- the eps term) for any penalties
    (duality.py:135-152), the sums in uot_translation at lam = 0."""
    _check_feasible(prob, d)
    h = translation(prob, d.f, d.g, solve=False, lam0=0.0, value=True)[3]
    total = float(h[0].item())
    if prob.eps > 0:
        total -= _eps_term(prob, d)[0]
    return total


def eval_F(prob, d):
    """Plain dual objective (duality.py:135-152); KL/KL through the LSE
    kernels, other penalties through the uot_translation sums."""
    prob.check_pair(d)
    if not _both_kl(prob):
        return _eval_f_generic(prob, d)
    if prob.eps == 0:
        from .exceptions import InfeasibleDualError

        viol = dual_feasibility_violation(prob, d)
        if viol > DUAL_FEAS_TOL:
            raise InfeasibleDualError(f"dual constraint violated by {viol:.3e} at eps = 0")
        out = kl_scalars(prob.alpha.weights, prob.beta.weights, d.f, d.g, prob.ent1.rho,
                         prob.ent2.rho)
        sf = float(out[0, 2].item())
        sg = _smin(prob.beta.weights, prob.ent2.rho, d.g)
        return _kl_parts(prob, sf, sg)[0]
    et, v = _eps_term(prob, d)
    return _kl_parts(prob, float(v[5]), float(v[6]))[0] - et


def eval_G(prob, d, lam):
    """Overparameterised dual: eval_F at (f + lam, g - lam) (duality.py:155-157)."""
    return eval_F(prob, DualPair(d.f + lam, d.g - lam))


def eval_H(prob, d):
    """Translation-invariant dual (duality.py:256-276): KL closed form,
    eval_F for Balanced/Balanced, else eval_G at the Newton translation."""
    prob.check_pair(d)
    if isinstance(prob.ent1, Balanced) and isinstance(prob.ent2, Balanced):
        return eval_F(prob, d)  # every translation gives the same value (:264-265)
    if not _both_kl(prob):
        return eval_G(prob, d, lambda_star(prob, d))  # :275-276
    if prob.eps == 0:
        from .exceptions import InfeasibleDualError

        viol = dual_feasibility_violation(prob, d)
        if viol > DUAL_FEAS_TOL:
            raise InfeasibleDualError(f"dual constraint violated by {viol:.3e} at eps = 0")
        out = kl_scalars(prob.alpha.weights, prob.beta.weights, d.f, d.g, prob.ent1.rho,
                         prob.ent2.rho)
        return float(out[0, 1].item())
    et, v = _eps_term(prob, d)
    return _kl_parts(prob, float(v[5]), float(v[6]))[1] - et


def _smin(w, rho, pot):
    """Smin^rho_w(pot) = -rho LSE_w(-pot/rho) via the kl_scalars kernel."""
    w = np.asarray(w, dtype=np.float64)
    pot = np.asarray(pot, dtype=np.float64)
    out = kl_scalars(w, w, pot, pot, rho, rho)
    return float(out[0, 2].item())


def updated_marginals(prob, d):
    """Reweighted marginals at the optimal translation (src/duality.py:293-303):
    (a exp((-f - t*)/rho1), b exp((-g + t*)/rho2)) for KL/KL, on the device."""
    prob.check_pair(d)
    if not _both_kl(prob):
        if not (_strictly_convex(prob.ent1) and _strictly_convex(prob.ent2)):
            raise UnsupportedEntropyError(
                "optimal translation needs strictly convex conjugates (KL or Berg)")
        _, ta, tb, _ = translation(prob, d.f, d.g, marginals=True)
        return D.to_np(ta, readonly=False), D.to_np(tb, readonly=False)
    t = D.torch()
    lib = _lib.load()
    n, m = len(prob.alpha), len(prob.beta)
    a, b, f, g = (D.to_dev(v, t.float64) for v in (prob.alpha.weights, prob.beta.weights, d.f, d.g))
    lam = float(kl_scalars(a, b, f, g, prob.ent1.rho, prob.ent2.rho)[0, 0].item())
    ta, tb = D.empty((n,), t.float64), D.empty((m,), t.float64)
    _lib.check(lib.uot_updated_marginals(n, m, _lib.ptr(a), _lib.ptr(b), _lib.ptr(f), _lib.ptr(g),
                                         float(prob.ent1.rho), float(prob.ent2.rho), lam,
                                         _lib.ptr(ta), _lib.ptr(tb), _lib.stream_handle()),
               "uot_updated_marginals")
    return D.to_np(ta, readonly=False), D.to_np(tb, readonly=False)


def eval_primal(prob, plan):
    """Primal objective of a transport plan (src/duality.py:320-344):
    <plan, C> + eps KL(plan | alpha x beta) + D1(plan_1 | alpha) +
    D2(plan_2 | beta), +inf where the reference gives +inf.  ``plan`` is a
    SparsePlan-like object or a dense (N, M) array; evaluated on the device
    (KL and Balanced divergences)."""
    from .entropies import Balanced
    from .measures import ExplicitMatrix, PowerDistance

    n, m = len(prob.alpha), len(prob.beta)
    if hasattr(plan, "source_idx"):
        ii, jj, mass = plan.source_idx, plan.target_idx, plan.mass
    else:
        dense = np.asarray(plan, dtype=np.float64)
        if dense.shape != (n, m):
            raise ValueError(f"dense plan must have shape ({n}, {m})")
        if np.any(dense < 0):
            raise ValueError("plan mass must be nonnegative")
        ii, jj = np.nonzero(dense)
        mass = dense[ii, jj]
    mass = np.asarray(mass, dtype=np.float64)
    if np.any(mass < 0):
        raise ValueError("plan mass must be nonnegative")
    codes = []
    for spec in (prob.ent1, prob.ent2):
        if isinstance(spec, KL):
            codes.append((_lib.ENT_KL, float(spec.rho)))
        elif isinstance(spec, Balanced):
            codes.append((_lib.ENT_BALANCED, 0.0))
        elif isinstance(spec, Berg):
            codes.append((_lib.ENT_BERG, float(spec.rho)))
        else:
            raise UnsupportedEntropyError(f"unknown entropy {spec!r}")
    t = D.torch()
    lib = _lib.load()
    x = y = C = None
    p = 2.0
    if isinstance(prob.cost, PowerDistance):
        x = D.to_dev(prob.alpha.points, t.float64)
        y = D.to_dev(prob.beta.points, t.float64)
        p = float(prob.cost.p)
    elif isinstance(prob.cost, ExplicitMatrix):
        C = D.to_dev(prob.cost.matrix, t.float64)
    else:
        raise TypeError(f"unknown cost specification {prob.cost!r}")
    a = D.to_dev(prob.alpha.weights, t.float64)
    b = D.to_dev(prob.beta.weights, t.float64)
    E = int(mass.size)
    di = D.to_dev(np.asarray(ii, dtype=np.int64), t.int64) if E else None
    dj = D.to_dev(np.asarray(jj, dtype=np.int64), t.int64) if E else None
    dm = D.to_dev(mass, t.float64) if E else None
    out = D.empty((1,), t.float64)
    _lib.check(lib.uot_eval_primal(n, m, _lib.ptr(x), _lib.ptr(y), p, _lib.ptr(C), _lib.ptr(a),
                                   _lib.ptr(b), E, _lib.ptr(di), _lib.ptr(dj), _lib.ptr(dm),
                                   codes[0][0], codes[1][0], codes[0][1], codes[1][1],
                                   float(prob.eps), _lib.ptr(out), _lib.stream_handle()),
               "uot_eval_primal")
    return float(out.item())
