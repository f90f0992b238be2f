"""CPU oracle: an fp64 restatement of the reference (uotkit) hot paths.

TEST INFRASTRUCTURE ONLY.  This package is the *checker*: it may be imported
by ``tests/``, by ``__graft_entry__.smoke()`` and by ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs, and by nothing else.  The
product package ``paper_2201_00730_b200`` never imports it and has no CPU
fallback.

Pinning: every function here is checked against golden vectors produced by
the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/uotkit`` in the build container and commits the
fixtures; ``tests/test_oracle_golden.py`` replays them).

Each function cites the reference lines it restates, relative to
``/root/reference/pkg/src/uotkit/``.  The sequential sweeps and the dense
softmin reduction live in ``oracle/csrc/oracle.c`` (built by
``oracle/Makefile`` into ``oracle/_oracle.so``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

COST_SQEUCLID, COST_POWER1D, COST_EXPLICIT = 0, 1, 2

MASS_TOL = 1e-9  # ot1d.py:27, barycenter.py:43
LMO_MASS_TOL = 1e-9  # fw.py:49


def build():
    """Compile oracle/csrc/oracle.c into oracle/_oracle.so (gcc -O2 -pthread)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_oracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        L.oracle_smin.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, ctypes.c_double,
            dp, ctypes.c_long, ctypes.c_long, dp, dp, ctypes.c_double, dp,
        ]
        L.oracle_smin.restype = None
        L.oracle_ot1d.argtypes = [
            ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, ctypes.c_int, ctypes.c_double, dp,
            ip, ip, dp, dp, dp,
        ]
        L.oracle_ot1d.restype = ctypes.c_long
        L.oracle_mot1d.argtypes = [
            ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_long), dp, dp,
            dp, ip, dp, dp,
        ]
        L.oracle_mot1d.restype = ctypes.c_long
        _LIB = L
    return _LIB


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------------------
# entropies.py


def logdotexp(values, weights, axis=None):
    """entropies.py:67-92: stabilised log sum_i w_i exp(v_i), zero weights masked."""
    v = np.asarray(values, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64)
    if axis is None:
        keep = w > 0
        if not keep.any():
            return -np.inf
        vk = v[keep]
        top = vk.max()
        return float(top + np.log(np.dot(w[keep], np.exp(vk - top))))
    shape = [1] * v.ndim
    shape[axis] = w.size
    wb = w.reshape(shape)
    masked = np.where(wb > 0, v, -np.inf)
    top = masked.max(axis=axis, keepdims=True)
    top = np.where(np.isfinite(top), top, 0.0)
    with np.errstate(divide="ignore"):
        s = np.log(np.sum(wb * np.exp(masked - top), axis=axis))
    return s + np.squeeze(top, axis=axis)


def softmin(weights, eps, f):
    """entropies.py:187-200: -eps log <w, exp(-f/eps)>."""
    return -eps * logdotexp(-np.asarray(f) / eps, weights)


def kl_divergence(rho, mu, nu):
    """entropies.py:123-131 (KL branch of divergence)."""
    mu = np.asarray(mu, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    pos = nu > 0
    if float(mu[~pos].sum()) > 0:
        return np.inf
    m, n = mu[pos], nu[pos]
    with np.errstate(divide="ignore", invalid="ignore"):
        terms = np.where(m > 0, m * np.log(np.where(m > 0, m / n, 1.0)), 0.0)
    return float(rho * (terms.sum() - m.sum() + n.sum()))


# ---------------------------------------------------------------------------
# duality.py


def lambda_star_kl(aw, bw, f, g, r1, r2):
    """duality.py:175-178: closed-form optimal translation for KL/KL."""
    la = logdotexp(-np.asarray(f) / r1, aw)
    lb = logdotexp(-np.asarray(g) / r2, bw)
    return (r1 * r2 / (r1 + r2)) * (la - lb)


def eval_h_kl(aw, bw, f, g, r1, r2, eps=0.0, smin_fn=None):
    """duality.py:279-290 (+ _eps_term :124-132 when eps > 0).

    ``smin_fn(pot_f, eps)`` must return smin over the source index of
    (f - C)/eps for every column (the column reduction of the eps term)."""
    la = logdotexp(-np.asarray(f) / r1, aw)
    lb = logdotexp(-np.asarray(g) / r2, bw)
    t1, t2 = r1 / (r1 + r2), r2 / (r1 + r2)
    out = r1 * float(np.sum(aw)) + r2 * float(np.sum(bw)) - (r1 + r2) * np.exp(t1 * la + t2 * lb)
    if eps > 0:
        # eps <a x b, e^((f+g-C)/eps) - 1>: LSE over i of (f_i - C_ij)/eps, then
        # over j of g_j/eps + that, duality.py:127-132.
        col = -smin_fn(f, eps) / eps  # log sum_i a_i exp((f_i - C_ij)/eps)
        total_log = logdotexp(col + np.asarray(g) / eps, bw)
        out -= eps * (np.exp(total_log) - float(np.sum(aw)) * float(np.sum(bw)))
    return float(out)


# ---------------------------------------------------------------------------
# Plan-support hash of the device trace mode (include/uot_b200.h, "plan-support
# hash"): entry (i_0 .. i_{K-1}) -> mix64(sum_q mix64(((q+1) << 40) | i_q)),
# plan -> wrapping sum over its entries.  numpy uint64 arithmetic wraps mod 2^64.


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def plan_hash(idx):
    """idx: (E, K) entry index tuples (a SparsePlan as columns (i, j), or a
    MultiPlan's indices).  Returns (hash as int64 bit pattern, entry count)."""
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size == 0:
        return np.int64(0), 0
    key = np.zeros(idx.shape[0], dtype=np.uint64)
    with np.errstate(over="ignore"):
        for q in range(idx.shape[1]):
            key = key + _mix64((np.uint64(q + 1) << np.uint64(40)) | idx[:, q].astype(np.uint64))
        tot = _mix64(key).sum(dtype=np.uint64)  # integer reductions wrap mod 2^64
    return np.array([tot], dtype=np.uint64).view(np.int64)[0], int(idx.shape[0])


# ---------------------------------------------------------------------------
# sinkhorn.py


class DenseCost:
    """Dense C (N x M) evaluated by the C oracle (sinkhorn.py:93-100)."""

    def __init__(self, C):
        self.C = _c64(C)
        self.n, self.m = self.C.shape

    def smin_cols(self, f, eps, aw):
        out = np.empty(self.m)
        lib().oracle_smin(COST_EXPLICIT, self.n, self.m, 0, None, None, 0.0, _dp(self.C),
                          self.m, 1, _dp(_c64(f)), _dp(_c64(aw)), eps, _dp(out))
        return out

    def smin_rows(self, g, eps, bw):
        out = np.empty(self.n)
        lib().oracle_smin(COST_EXPLICIT, self.m, self.n, 0, None, None, 0.0, _dp(self.C),
                          1, self.m, _dp(_c64(g)), _dp(_c64(bw)), eps, _dp(out))
        return out


class PointCost:
    """On-the-fly cost: squared Euclidean between point clouds (d >= 1) or
    |x - y|^p for 1-D points; never materialises C (needed for cfg3)."""

    def __init__(self, x, y, p=2.0, power1d=False):
        self.x = _c64(x)
        self.y = _c64(y)
        self.power1d = power1d
        self.p = float(p)
        if power1d:
            self.n, self.m, self.d = self.x.size, self.y.size, 1
        else:
            self.x = self.x.reshape(len(self.x), -1)
            self.y = self.y.reshape(len(self.y), -1)
            self.n, self.d = self.x.shape
            self.m = self.y.shape[0]

    def _run(self, xr, xo, nred, nout, pot, w, eps):
        out = np.empty(nout)
        kind = COST_POWER1D if self.power1d else COST_SQEUCLID
        lib().oracle_smin(kind, nred, nout, self.d, _dp(xr), _dp(xo), self.p, None, 0, 0,
                          _dp(_c64(pot)), _dp(_c64(w)), eps, _dp(out))
        return out

    def smin_cols(self, f, eps, aw):
        return self._run(self.x, self.y, self.n, self.m, f, aw, eps)

    def smin_rows(self, g, eps, bw):
        return self._run(self.y, self.x, self.m, self.n, g, bw, eps)


def f_sinkhorn_step(cost, aw, bw, f, g, eps, r1, r2):
    """sinkhorn.py:103-114 with KL aprox (entropies.py:213-214)."""
    g_new = (r2 / (eps + r2)) * cost.smin_cols(f, eps, aw)
    f_new = (r1 / (eps + r1)) * cost.smin_rows(g_new, eps, bw)
    return f_new, g_new


def h_sinkhorn_step(cost, aw, bw, f, g, eps, r1, r2):
    """sinkhorn.py:137-163: translation-invariant step, g first then f."""
    g_hat = (r2 / (r2 + eps)) * cost.smin_cols(f, eps, aw)
    g_hat = g_hat - (eps / (eps + r2)) * (r2 / (r1 + r2)) * softmin(aw, r1, f)
    k2 = (eps / (eps + r2)) * (r1 / (r1 + r2))
    g_new = g_hat + (k2 / (1.0 - k2)) * softmin(bw, r2, g_hat)
    f_hat = (r1 / (r1 + eps)) * cost.smin_rows(g_new, eps, bw)
    f_hat = f_hat - (eps / (eps + r1)) * (r1 / (r1 + r2)) * softmin(bw, r2, g_new)
    k1 = (eps / (eps + r1)) * (r2 / (r1 + r2))
    f_new = f_hat + (k1 / (1.0 - k1)) * softmin(aw, r1, f_hat)
    return f_new, g_new


def berg_aprox(rho, eps, x, tol=1e-12, max_iters=100):
    """entropies.py:224-263: root of y + eps log(rho/(rho - y)) = x, bracketed
    safeguarded Newton (vectorised)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))

    def h(y):
        return y + eps * np.log(rho / (rho - y)) - x

    lo = np.minimum(x, rho - 1.0)
    step = np.maximum(1.0, eps)
    for _ in range(200):
        bad = h(lo) > 0
        if not bad.any():
            break
        lo = np.where(bad, lo - step, lo)
        step = step * 2
    top = np.nextafter(rho, -np.inf)
    gap = rho - np.minimum(x, rho - 1.0)
    hi = np.minimum(rho - gap, top)
    for _ in range(200):
        bad = h(hi) < 0
        if not (bad & (hi < top)).any():
            break
        gap = np.where(bad, gap / 4, gap)
        hi = np.minimum(rho - gap, top)
    y = np.clip(np.minimum(x, rho - gap), lo, hi)
    em = np.finfo(np.float64).eps
    for _ in range(max_iters):
        res = h(y)
        resolved = (hi - lo) <= 4 * em * (1.0 + np.abs(y))
        if np.all((np.abs(res) < tol) | resolved):
            return y
        lo = np.where(res < 0, y, lo)
        hi = np.where(res > 0, y, hi)
        newton = y - res / (1.0 + eps / (rho - y))
        inside = (newton > lo) & (newton < hi)
        y = np.where(inside, newton, 0.5 * (lo + hi))
    raise ValueError("Berg aprox Newton did not converge")


def aprox(ent, rho, eps, x):
    """entropies.py:203-221 for ent in {"kl", "berg", "balanced"}."""
    if ent == "kl":
        return (rho / (eps + rho)) * np.asarray(x, dtype=np.float64)
    if ent == "balanced":
        return np.asarray(x, dtype=np.float64) + 0.0
    return berg_aprox(rho, eps, x)


def _cgrad(ent, rho, x):
    return np.exp(x / rho) if ent == "kl" else rho / (rho - x)


def _chess(ent, rho, x):
    return np.exp(x / rho) / rho if ent == "kl" else rho / (rho - x) ** 2


def lambda_star_any(aw, bw, f, g, ents, r1, r2, initial=0.0, tol=1e-11, max_iters=100):
    """duality.py:170-247: closed form for KL/KL, else the bracketed Newton."""
    e1, e2 = ents
    if e1 == "kl" and e2 == "kl":
        return lambda_star_kl(aw, bw, f, g, r1, r2)
    lo_dom = -np.inf if e1 != "berg" else -r1 - float(f.min())
    hi_dom = np.inf if e2 != "berg" else r2 + float(g.min())

    def residual(lam):
        with np.errstate(over="ignore"):
            return float(np.dot(aw, _cgrad(e1, r1, -f - lam))) - float(
                np.dot(bw, _cgrad(e2, r2, -g + lam)))

    def slope(lam):
        with np.errstate(over="ignore"):
            return -float(np.dot(aw, _chess(e1, r1, -f - lam))) - float(
                np.dot(bw, _chess(e2, r2, -g + lam)))

    def clamp(x):
        if np.isfinite(lo_dom):
            x = max(x, lo_dom + 1e-12 * max(1.0, abs(lo_dom)))
        if np.isfinite(hi_dom):
            x = min(x, hi_dom - 1e-12 * max(1.0, abs(hi_dom)))
        return x

    lam = clamp(initial)
    r0 = residual(lam)
    if abs(r0) < tol:
        return lam
    step = 1.0
    lo, hi = lam, lam
    if r0 > 0:
        for _ in range(200):
            hi = clamp(lam + step)
            if residual(hi) <= 0:
                break
            step *= 2
    else:
        for _ in range(200):
            lo = clamp(lam - step)
            if residual(lo) >= 0:
                break
            step *= 2
    x = 0.5 * (lo + hi)
    for _ in range(max_iters):
        r = residual(x)
        if abs(r) < tol:
            return x
        if r > 0:
            lo = x
        else:
            hi = x
        ds = slope(x)
        newton = x - r / ds if ds < 0 and np.isfinite(ds) else None
        x = newton if newton is not None and lo < newton < hi else 0.5 * (lo + hi)
    raise ValueError("translation Newton did not converge")


def f_sinkhorn_step_any(cost, aw, bw, f, g, eps, r1, r2, ents):
    """sinkhorn.py:103-114 with any aprox."""
    g_new = -aprox(ents[1], r2, eps, -cost.smin_cols(f, eps, aw))
    f_new = -aprox(ents[0], r1, eps, -cost.smin_rows(g_new, eps, bw))
    return f_new, g_new


def g_sinkhorn_step_any(cost, aw, bw, f, g, eps, r1, r2, lam, ents):
    """sinkhorn.py:117-134 with any aprox and lambda_star(initial=lam)."""
    smin_a = cost.smin_cols(f + lam, eps, aw)
    g_new = lam - aprox(ents[1], r2, eps, -smin_a)
    smin_b = cost.smin_rows(g_new - lam, eps, bw)
    f_new = -lam - aprox(ents[0], r1, eps, -smin_b)
    return f_new, g_new, lambda_star_any(aw, bw, f_new, g_new, ents, r1, r2, initial=lam)


def g_sinkhorn_step(cost, aw, bw, f, g, eps, r1, r2, lam):
    """sinkhorn.py:117-134 with KL aprox: both half-updates at the incoming
    translation lam, then lambda* of the new pair (duality.py:175-178).
    Returns (f', g', lambda')."""
    smin_a = cost.smin_cols(f + lam, eps, aw)
    g_new = lam + (r2 / (eps + r2)) * smin_a
    smin_b = cost.smin_rows(g_new - lam, eps, bw)
    f_new = -lam + (r1 / (eps + r1)) * smin_b
    return f_new, g_new, lambda_star_kl(aw, bw, f_new, g_new, r1, r2)


def sinkhorn_fixed(cost, aw, bw, eps, r1, r2, variant, iters, f0=None, g0=None,
                   ents=("kl", "kl")):
    """sinkhorn.py:246-315 (run) with the early exit removed (:304-306):
    exactly ``iters`` steps; returns (f, g, delta_f trace).  Variant "g"
    starts from lambda*(f0, g0) (:263-265) and carries lambda (:270-271)."""
    f = np.zeros(cost.n) if f0 is None else _c64(f0).copy()
    g = np.zeros(cost.m) if g0 is None else _c64(g0).copy()
    deltas = np.empty(iters)
    if variant == "g":
        lam = lambda_star_any(aw, bw, f, g, ents, r1, r2)
        for t in range(iters):
            fn, gn, lam = g_sinkhorn_step_any(cost, aw, bw, f, g, eps, r1, r2, lam, ents)
            deltas[t] = float(np.abs(fn - f).max())
            f, g = fn, gn
        return f, g, deltas
    if tuple(ents) != ("kl", "kl"):
        for t in range(iters):
            fn, gn = f_sinkhorn_step_any(cost, aw, bw, f, g, eps, r1, r2, ents)
            deltas[t] = float(np.abs(fn - f).max())
            f, g = fn, gn
        return f, g, deltas
    step = h_sinkhorn_step if variant == "h" else f_sinkhorn_step
    for t in range(iters):
        fn, gn = step(cost, aw, bw, f, g, eps, r1, r2)
        deltas[t] = float(np.abs(fn - f).max())
        f, g = fn, gn
    return f, g, deltas


def anderson_weights(U, r):
    """sinkhorn.py:197-212: the window weights c with (U'U + r I) c
    proportional to the ones vector and sum(c) = 1.  The k x k system is
    solved by Gaussian elimination with partial pivoting (the device's
    algorithm; LAPACK dgesv in the reference); an exactly zero pivot or a
    zero / non-finite normaliser raises LinAlgError like the reference."""
    U = np.asarray(U, dtype=np.float64)
    if U.ndim != 2 or U.shape[1] < 1:
        raise ValueError("U must be a matrix with at least one column")
    k = U.shape[1]
    A = np.empty((k, k))
    for i in range(k):
        for j in range(k):
            A[i, j] = float(np.dot(U[:, i], U[:, j]))
        A[i, i] += r
    sol = _solve_pivoted(A, np.ones(k))
    den = float(sol.sum())
    if not np.isfinite(den) or den == 0.0:
        raise np.linalg.LinAlgError("degenerate weight normalization")
    return sol / den


def _solve_pivoted(A, rhs):
    A = A.copy()
    x = rhs.astype(np.float64).copy()
    k = A.shape[0]
    for col in range(k):
        piv = col + int(np.argmax(np.abs(A[col:, col])))
        if A[piv, col] == 0.0:
            raise np.linalg.LinAlgError("Singular matrix")
        if piv != col:
            A[[col, piv]] = A[[piv, col]]
            x[[col, piv]] = x[[piv, col]]
        for row in range(col + 1, k):
            fac = A[row, col] / A[col, col]
            A[row, col:] -= fac * A[col, col:]
            x[row] -= fac * x[col]
    for row in range(k - 1, -1, -1):
        x[row] = (x[row] - float(np.dot(A[row, row + 1:], x[row + 1:]))) / A[row, row]
    return x


class AndersonState:
    """sinkhorn.py:215-243: window of (T z, T z - z); restart when the new
    residual's sup norm exceeds the previous one's, keep the last ``depth``."""

    def __init__(self, depth, reg):
        self.depth, self.reg = depth, reg
        self.maps, self.res, self.sizes = [], [], []

    def push_extrapolate(self, z, tz):
        r = tz - z
        size = float(np.abs(r).max())
        if self.sizes and size > self.sizes[-1]:
            self.maps, self.res, self.sizes = [], [], []
        self.maps.append(tz)
        self.res.append(r)
        self.sizes.append(size)
        if len(self.maps) > self.depth:
            self.maps, self.res, self.sizes = self.maps[1:], self.res[1:], self.sizes[1:]
        if len(self.maps) == 1:
            return self.maps[0]
        c = anderson_weights(np.stack(self.res, axis=1), self.reg)
        zn = np.zeros(len(z))
        for ck, mk in zip(c, self.maps):
            zn = zn + ck * mk
        return zn


def sinkhorn_anderson(cost, aw, bw, eps, r1, r2, variant, iters, depth, reg, f0=None,
                      g0=None, ents=("kl", "kl")):
    """sinkhorn.py:246-315 with ``config.anderson`` set (window state
    :215-243): every iteration maps z = (f, g) through one step, pushes
    (T z, T z - z) -- the window restarts when the new residual's sup norm
    exceeds the previous one's, and keeps the last ``depth`` entries -- and
    moves to the extrapolation sum_k c_k (T z)_k.  Variant "g" carries the
    step's lambda (:270-271).  Exactly ``iters`` iterations (no early
    exit); returns (f, g, delta_f trace)."""
    n, m = cost.n, cost.m
    f = np.zeros(n) if f0 is None else _c64(f0).copy()
    g = np.zeros(m) if g0 is None else _c64(g0).copy()
    lam = lambda_star_any(aw, bw, f, g, ents, r1, r2) if variant == "g" else 0.0
    win = AndersonState(depth, reg)
    deltas = np.empty(iters)
    for t in range(iters):
        if variant == "g":
            fn, gn, lam = g_sinkhorn_step_any(cost, aw, bw, f, g, eps, r1, r2, lam, ents)
        elif variant == "h":
            fn, gn = h_sinkhorn_step(cost, aw, bw, f, g, eps, r1, r2)
        else:
            fn, gn = f_sinkhorn_step_any(cost, aw, bw, f, g, eps, r1, r2, ents)
        zn = win.push_extrapolate(np.concatenate([f, g]), np.concatenate([fn, gn]))
        deltas[t] = float(np.abs(zn[:n] - f).max())
        f, g = zn[:n].copy(), zn[n:].copy()
    return f, g, deltas


def h_optimality_residual(cost, aw, bw, f, g, eps, r1, r2, side="f"):
    """sinkhorn.py:166-189."""
    lam = lambda_star_kl(aw, bw, f, g, r1, r2)
    if side == "f":
        res = f - (r1 / (r1 + eps)) * cost.smin_rows(g, eps, bw) + (eps / (eps + r1)) * lam
    else:
        res = g - (r2 / (r2 + eps)) * cost.smin_cols(f, eps, aw) - (eps / (eps + r2)) * lam
    return float(np.abs(res).max())


# ---------------------------------------------------------------------------
# ot1d.py


def solve_ot_1d(x, y, wa, wb, p=2.0, explicit=None):
    """ot1d.py:112-172; returns (i, j, mass, f, g).  Raises ValueError on a
    mass mismatch beyond 1e-9 relative (ot1d.py:133-136)."""
    wa = _c64(wa)
    wb = _c64(wb)
    ma, mb = float(wa.sum()), float(wb.sum())
    if abs(ma - mb) > MASS_TOL * max(ma, mb):
        raise ValueError(f"balanced solver needs equal masses, got {ma:.12g} and {mb:.12g}")
    n, m = wa.size, wb.size
    ei = np.empty(n + m, dtype=np.int64)
    ej = np.empty(n + m, dtype=np.int64)
    em = np.empty(n + m)
    f = np.empty(n)
    g = np.empty(m)
    x = _c64(x) if x is not None else np.zeros(n)
    y = _c64(y) if y is not None else np.zeros(m)
    kind = COST_EXPLICIT if explicit is not None else COST_POWER1D
    cm = _c64(explicit) if explicit is not None else None
    ip = ctypes.POINTER(ctypes.c_int64)
    e = lib().oracle_ot1d(n, m, _dp(x), _dp(y), _dp(wa), _dp(wb), kind, float(p),
                          _dp(cm) if cm is not None else None, ei.ctypes.data_as(ip),
                          ej.ctypes.data_as(ip), _dp(em), _dp(f), _dp(g))
    return ei[:e].copy(), ej[:e].copy(), em[:e].copy(), f, g


def power_cost_at(x, y, i, j, p):
    d = np.abs(x[i] - y[j])
    if p == 1.0:
        return d
    if p == 2.0:
        return d * d
    return d**p


# ---------------------------------------------------------------------------
# fw.py


def h0_kl(aw, bw, f, g, r1, r2):
    """fw.py:106-115 -> duality.py:279-290 with skip_eps_term."""
    return eval_h_kl(aw, bw, f, g, r1, r2)


def ternary_max(fn, lo=0.0, hi=1.0, iters=60):
    """fw.py:118-128."""
    a, b = float(lo), float(hi)
    for _ in range(iters):
        m1 = a + (b - a) / 3.0
        m2 = b - (b - a) / 3.0
        if fn(m1) < fn(m2):
            a = m1
        else:
            b = m2
    return 0.5 * (a + b)


def line_search_h0(aw, bw, f, g, r, s, r1, r2):
    """fw.py:131-148: ternary search then best of {gamma, 0, 1}."""

    def value(gam):
        return h0_kl(aw, bw, (1.0 - gam) * f + gam * r, (1.0 - gam) * g + gam * s, r1, r2)

    gam = ternary_max(value, 0.0, 1.0, iters=60)
    best = max(((value(c), c) for c in (gam, 0.0, 1.0)), key=lambda t: t[0])
    return best[1]


def eval_primal_1d(x, y, aw, bw, ii, jj, mass, p, r1, r2):
    """duality.py:320-344 at eps = 0 with KL divergences (entropies.py:123-131)."""
    cost = float(np.dot(mass, power_cost_at(x, y, ii, jj, p)))
    m1 = np.zeros(aw.size)
    m2 = np.zeros(bw.size)
    np.add.at(m1, ii, mass)
    np.add.at(m2, jj, mass)
    return cost + kl_divergence(r1, m1, aw) + kl_divergence(r2, m2, bw)


def fw_fixed(x, y, aw, bw, r1, r2, iters, step="linesearch", p=2.0, f0=None, g0=None,
             gap_tol=None, gammas=None):
    """fw.py:176-232 (fw_solve) + _lmo :159-173 + _finalize :235-252.

    With ``gap_tol=None`` the early exit (:220-222) is removed so exactly
    ``iters`` iterations run (BASELINE fixed-iteration configs); otherwise
    the reference's exit rule applies.  ``gammas`` replays given step sizes.
    Returns a dict with the final translated pair, the untranslated iterate,
    traces (incl. gamma and each iteration's plan_hash / entry count) and the
    last plan."""
    x, y, aw, bw = _c64(x), _c64(y), _c64(aw), _c64(bw)
    f = np.zeros(aw.size) if f0 is None else _c64(f0).copy()
    g = np.zeros(bw.size) if g0 is None else _c64(g0).copy()
    tr = {k: [] for k in ("h0", "fw_gap", "pd_gap", "gamma", "supp_hash", "nnz")}
    plan = None
    converged = False
    for t in range(iters):
        lam = lambda_star_kl(aw, bw, f, g, r1, r2)
        with np.errstate(over="ignore"):
            ta = aw * np.exp((-f - lam) / r1)
            tb = bw * np.exp((-g + lam) / r2)
        ma, mb = float(ta.sum()), float(tb.sum())
        if abs(ma - mb) > LMO_MASS_TOL * max(ma, mb):
            raise ValueError("reweighted marginal masses disagree")
        ii, jj, mm, r, s = solve_ot_1d(x, y, ta, tb, p)
        plan = (ii, jj, mm)
        hh, cc = plan_hash(np.stack([ii, jj], axis=1))
        tr["supp_hash"].append(hh)
        tr["nnz"].append(cc)
        fw_gap = float(np.dot(ta, r - f) + np.dot(tb, s - g))
        dual = h0_kl(aw, bw, f, g, r1, r2)
        primal = eval_primal_1d(x, y, aw, bw, ii, jj, mm, p, r1, r2)
        tr["h0"].append(dual)
        tr["fw_gap"].append(fw_gap)
        tr["pd_gap"].append(primal - dual)
        if gap_tol is not None and primal - dual < gap_tol:
            converged = True
            break
        if gammas is not None:
            gam = float(gammas[t])
        elif step == "harmonic":
            gam = 2.0 / (2.0 + t)
        else:
            gam = line_search_h0(aw, bw, f, g, r, s, r1, r2)
        tr["gamma"].append(gam)
        f = (1.0 - gam) * f + gam * r
        g = (1.0 - gam) * g + gam * s
    lam = lambda_star_kl(aw, bw, f, g, r1, r2)
    return {
        "f": f + lam,
        "g": g - lam,
        "f_raw": f,
        "g_raw": g,
        "plan": plan,
        "converged": converged,
        **{k: np.asarray(v) for k, v in tr.items()},
    }


ATOM_DEDUP_TOL = 1e-12


def pfw_fixed(x, y, aw, bw, r1, r2, iters, p=2.0, gap_tol=None):
    """Pairwise FW, fw.py:255-357 (_active_scores :255-257, _merge_atom
    :260-272, _pfw_iteration :275-310, _pfw_solve :326-357) on the same LMO.

    The atom store holds dual-pair atoms with convex weights; the iterate is
    the weighted atom.  Each iteration: LMO at the iterate, away atom =
    argmin over active atoms of <r_a, ta> + <s_a, tb> (lowest index on
    ties), ternary line search of H0 along (new - away) on [0, w_away],
    weight transfer, merge of the new atom into an existing one closer than
    1e-12 (sup norm), drop of zero-weight atoms.  ``gap_tol=None`` removes
    the early exit (:351-353).  Returns the dict of ``fw_fixed`` plus the
    step sizes and atom counts."""
    x, y, aw, bw = _c64(x), _c64(y), _c64(aw), _c64(bw)
    R = np.zeros((1, aw.size))
    Sg = np.zeros((1, bw.size))
    W = np.array([1.0])
    tr = {k: [] for k in ("h0", "fw_gap", "pd_gap", "gamma", "natoms", "supp_hash", "nnz")}
    plan = None
    converged = False
    for t in range(iters):
        f, g = W @ R, W @ Sg
        lam = lambda_star_kl(aw, bw, f, g, r1, r2)
        with np.errstate(over="ignore"):
            ta = aw * np.exp((-f - lam) / r1)
            tb = bw * np.exp((-g + lam) / r2)
        ma, mb = float(ta.sum()), float(tb.sum())
        if abs(ma - mb) > LMO_MASS_TOL * max(ma, mb):
            raise ValueError("reweighted marginal masses disagree")
        ii, jj, mm, r, s = solve_ot_1d(x, y, ta, tb, p)
        plan = (ii, jj, mm)
        hh, cc = plan_hash(np.stack([ii, jj], axis=1))
        tr["supp_hash"].append(hh)
        tr["nnz"].append(cc)
        fw_gap = float(np.dot(ta, r - f) + np.dot(tb, s - g))
        dual = h0_kl(aw, bw, f, g, r1, r2)
        primal = eval_primal_1d(x, y, aw, bw, ii, jj, mm, p, r1, r2)
        tr["h0"].append(dual)
        tr["fw_gap"].append(fw_gap)
        tr["pd_gap"].append(primal - dual)
        scores = np.where(W > 0, R @ ta + Sg @ tb, np.inf)
        away = int(np.argmin(scores))
        max_step = float(W[away])
        dr, ds = r - R[away], s - Sg[away]
        gam = 0.0
        if not (max_step <= 0.0 or (np.abs(dr).max() < ATOM_DEDUP_TOL
                                     and np.abs(ds).max() < ATOM_DEDUP_TOL)):
            def value(gg):
                return h0_kl(aw, bw, f + gg * dr, g + gg * ds, r1, r2)

            gam = ternary_max(value, 0.0, max_step, iters=60)
            gam = max(((value(c), c) for c in (gam, 0.0, max_step)), key=lambda q: q[0])[1]
            if gam > 0.0:
                W = W.copy()
                W[away] = max(W[away] - gam, 0.0)
                dist = np.maximum(np.abs(R - r).max(axis=1), np.abs(Sg - s).max(axis=1))
                hit = np.nonzero(dist < ATOM_DEDUP_TOL)[0]
                if hit.size:
                    W[hit[0]] += gam
                else:
                    R, Sg, W = np.vstack([R, r]), np.vstack([Sg, s]), np.concatenate([W, [gam]])
                keep = W > 0
                R, Sg, W = R[keep], Sg[keep], W[keep]
        tr["gamma"].append(gam)
        tr["natoms"].append(W.size)
        if gap_tol is not None and primal - dual < gap_tol:
            converged = True
            break
    f, g = W @ R, W @ Sg
    lam = lambda_star_kl(aw, bw, f, g, r1, r2)
    return {
        "f": f + lam, "g": g - lam, "f_raw": f, "g_raw": g, "plan": plan,
        "converged": converged, **{k: np.asarray(v) for k, v in tr.items()},
    }


# ---------------------------------------------------------------------------
# barycenter.py


def multimarginal_cost(pts, w):
    """barycenter.py:148-156."""
    pts = np.asarray(pts, dtype=np.float64)
    b = float(np.dot(w, pts))
    return float(np.dot(w, (pts - b) ** 2)), b


def solve_mot_1d(xs, ws, w):
    """barycenter.py:169-233 (Algorithm 3).  xs/ws: lists of K 1-D arrays.
    Returns (indices (E, K) int64, mass (E,), potentials list)."""
    k = len(xs)
    masses = np.array([float(np.sum(a)) for a in ws])
    if float(masses.max() - masses.min()) > MASS_TOL * float(masses.max()):
        raise ValueError(f"multimarginal sweep needs equal masses, got {masses.tolist()}")
    lens = np.array([len(a) for a in xs], dtype=np.int32)
    off = np.zeros(k, dtype=np.int64)
    off[1:] = np.cumsum(lens)[:-1]
    X = _c64(np.concatenate(xs))
    W = _c64(np.concatenate(ws))
    total = int(lens.sum())
    cap = total - k + 1
    idx = np.empty((cap, k), dtype=np.int64)
    mass = np.empty(cap)
    pots = np.empty(total)
    e = lib().oracle_mot1d(
        k, lens.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
        off.ctypes.data_as(ctypes.POINTER(ctypes.c_long)), _dp(X), _dp(W), _dp(_c64(w)),
        idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(mass), _dp(pots))
    return idx[:e].copy(), mass[:e].copy(), [pots[off[q]:off[q] + lens[q]].copy() for q in range(k)]


def solve_mot_1d_custom(xs, ws, costfn):
    """barycenter.py:169-233 with a caller costfn (pure-Python restatement of
    the sweep loop :209-229; small cases only).  Returns (indices, mass,
    potentials list)."""
    k = len(xs)
    last = np.array([len(a) - 1 for a in xs], dtype=np.int64)
    idx = np.zeros(k, dtype=np.int64)
    rem = np.array([float(w[0]) for w in ws])
    pots = [np.zeros(len(a)) for a in xs]
    cur = np.array([float(x[0]) for x in xs])
    pots[0][0] = costfn(cur)
    pot_sum = pots[0][0]
    ent_i, ent_m = [], []
    while True:
        can = idx < last
        if not can.any():
            step = float(rem.min())
            if step > 0:
                ent_i.append(idx.copy())
                ent_m.append(step)
            break
        p = int(np.argmin(np.where(can, rem, np.inf)))
        step = float(rem[p])
        if step > 0:
            ent_i.append(idx.copy())
            ent_m.append(step)
        rem = np.maximum(rem - step, 0.0)
        idx[p] += 1
        cur[p] = xs[p][idx[p]]
        old = pots[p][idx[p] - 1]
        new = costfn(cur) - (pot_sum - old)
        pots[p][idx[p]] = new
        pot_sum += new - old
        rem[p] = ws[p][idx[p]]
    return np.array(ent_i, dtype=np.int64).reshape(-1, k), np.array(ent_m), pots


def large_ot_inputs(n, m, seed):
    """Seeded balanced 1-D OT inputs for the large-size goldens (test
    fixture generator): sorted uniform supports with a run of duplicated
    points, Exp(1) weights with ~10% exact zeros, both scaled to mass 1.3."""
    rng = np.random.default_rng(seed)
    x = np.sort(rng.uniform(0.0, 1.0, n))
    y = np.sort(rng.uniform(0.0, 1.0, m))
    x[n // 3:n // 3 + 5] = x[n // 3]  # coincident atoms
    wa = rng.exponential(1.0, n) * (rng.random(n) > 0.1)
    wb = rng.exponential(1.0, m) * (rng.random(m) > 0.1)
    wa[0] = wb[0] = 1.0
    wa *= 1.3 / wa.sum()
    wb *= 1.3 / wb.sum()
    return x, y, wa, wb


def mot_mismatch_report(idx_a, mass_a, idx_b, mass_b, cums):
    """Compare two K-marginal plans (tuples + masses) entry by entry.  Returns
    the entry counts, the number of entries present in only one plan, the
    mass those entries carry (mass_moved = max over the two plans), and, at
    every place where the two sweeps take a different step, the gap between
    the cumulative breakpoints that decided it (cums[q][i] = sum_{s<=i} w_q[s],
    barycenter.py:209-229): max_gap (absolute) and max_gap_rel (relative to
    the total mass)."""
    ta = {tuple(r): m for r, m in zip(np.asarray(idx_a).tolist(), mass_a)}
    tb = {tuple(r): m for r, m in zip(np.asarray(idx_b).tolist(), mass_b)}
    only_a = set(ta) - set(tb)
    only_b = set(tb) - set(ta)
    total = float(np.sum(mass_b))
    gaps = []
    ia, ib = np.asarray(idx_a), np.asarray(idx_b)
    e = 0
    n = min(len(ia), len(ib))
    while e < n:
        if np.array_equal(ia[e], ib[e]):
            e += 1
            continue
        prev = ia[e - 1] if e > 0 else np.zeros(ia.shape[1], dtype=np.int64)
        qs = sorted(set(np.nonzero(ia[e] != prev)[0]) | set(np.nonzero(ib[e] != prev)[0]))
        vals = [float(cums[q][prev[q]]) for q in qs]
        gaps.append(max(vals) - min(vals) if vals else 0.0)
        # resynchronise on the next common tuple
        rest_b = {tuple(r): k for k, r in enumerate(ib[e:].tolist())}
        k = e
        while k < len(ia) and tuple(ia[k].tolist()) not in rest_b:
            k += 1
        if k >= len(ia):
            break
        shift = rest_b[tuple(ia[k].tolist())] + e - k
        ia_k, ib_k = ia[k:], ib[k + shift:]
        ia, ib = ia_k, ib_k
        n = min(len(ia), len(ib))
        e = 0
    return {"entries": (len(idx_a), len(idx_b)), "differing": (len(only_a), len(only_b)),
            "mass_moved": max(sum(ta[t] for t in only_a), sum(tb[t] for t in only_b), 0.0),
            "mismatch_sites": len(gaps), "max_gap": max(gaps) if gaps else 0.0,
            "max_gap_rel": (max(gaps) / total) if gaps else 0.0}


def multimarginal_lambda(pots, ws, w, rho):
    """barycenter.py:298-317."""
    rhos = np.asarray(w, dtype=np.float64) * float(rho)
    q = np.array([logdotexp(-f / rk, a) for f, a, rk in zip(pots, ws, rhos)])
    rho_tot = float(rhos.sum())
    return rhos * q - (rhos / rho_tot) * float(np.dot(rhos, q))


def h_value(ws, rhos, pots):
    """barycenter.py:320-327."""
    q = np.array([logdotexp(-f / rk, a) for f, a, rk in zip(pots, ws, rhos)])
    rho_tot = float(rhos.sum())
    masses = np.array([float(np.sum(a)) for a in ws])
    return float(np.dot(rhos, masses) - rho_tot * np.exp(float(np.dot(rhos, q)) / rho_tot))


def plan_cost(idx, mass, xs, w):
    """barycenter.py:236-240 with the barycentric cost (vectorised over entries)."""
    pts = np.stack([xs[k][idx[:, k]] for k in range(idx.shape[1])], axis=1)
    b = pts @ w
    return float(np.dot(mass, ((pts - b[:, None]) ** 2) @ w))


def fw_barycenter_fixed(xs, ws, w, rho, iters, step="linesearch", pots0=None, gap_tol=None,
                        gammas=None):
    """barycenter.py:330-430 loop body (:361-411) without the exhaustive
    feasibility check of _finalize (:416-418, overflows at cfg5 scale,
    SURVEY.md §0 finding 3).  ``gap_tol=None`` removes the early exit;
    ``gammas`` replays given step sizes.  Traces include gamma and each
    iteration's plan_hash / entry count."""
    w = _c64(w)
    rhos = w * float(rho)
    k = len(xs)
    pots = [np.zeros(len(a)) for a in xs] if pots0 is None else [_c64(p).copy() for p in pots0]
    tr = {k_: [] for k_ in ("h0", "fw_gap", "pd_gap", "gamma", "supp_hash", "nnz")}
    plan = None
    converged = False
    for t in range(iters):
        lam = multimarginal_lambda(pots, ws, w, rho)
        tilted = [a * np.exp(-(f + lk) / rk) for a, f, lk, rk in zip(ws, pots, lam, rhos)]
        masses = np.array([float(tw.sum()) for tw in tilted])
        if float(masses.max() - masses.min()) > MASS_TOL * float(masses.max()):
            raise ValueError("translated masses disagree; translation broken")
        idx, mass, atoms = solve_mot_1d(xs, tilted, w)
        plan = (idx, mass)
        hh, cc = plan_hash(idx)
        tr["supp_hash"].append(hh)
        tr["nnz"].append(cc)
        fw_gap = float(sum(np.dot(tw, r - f) for tw, r, f in zip(tilted, atoms, pots)))
        dual = h_value(ws, rhos, pots)
        marg = []
        for q in range(k):
            mq = np.zeros(len(xs[q]))
            np.add.at(mq, idx[:, q], mass)
            marg.append(mq)
        primal = plan_cost(idx, mass, xs, w) + float(
            sum(kl_divergence(rhos[q], marg[q], ws[q]) for q in range(k)))
        tr["h0"].append(dual)
        tr["fw_gap"].append(fw_gap)
        tr["pd_gap"].append(primal - dual)
        if gap_tol is not None and primal - dual < gap_tol:
            converged = True
            break
        if gammas is not None:
            gam = float(gammas[t])
        elif step == "harmonic":
            gam = 2.0 / (2.0 + t)
        else:

            def value(gg):
                return h_value(ws, rhos, [(1.0 - gg) * f + gg * r for f, r in zip(pots, atoms)])

            gam = ternary_max(value, 0.0, 1.0, iters=60)
            gam = max(((value(c), c) for c in (gam, 0.0, 1.0)), key=lambda z: z[0])[1]
        tr["gamma"].append(gam)
        pots = [(1.0 - gam) * f + gam * r for f, r in zip(pots, atoms)]
    lam = multimarginal_lambda(pots, ws, w, rho)
    return {
        "pots": [f + lk for f, lk in zip(pots, lam)],
        "pots_raw": pots,
        "plan": plan,
        "converged": converged,
        **{k_: np.asarray(v) for k_, v in tr.items()},
    }


def extract_barycenter(idx, mass, xs, w):
    """barycenter.py:433-443 (DiscreteMeasure merge of coincident atoms, measures.py:51-74)."""
    pts = np.stack([xs[k][idx[:, k]] for k in range(idx.shape[1])], axis=1) @ _c64(w)
    order = np.argsort(pts, kind="stable")
    pts, wts = pts[order], mass[order]
    if pts.size > 1 and np.any(np.diff(pts) == 0.0):
        uniq, inv = np.unique(pts, return_inverse=True)
        merged = np.zeros_like(uniq)
        np.add.at(merged, inv, wts)
        pts, wts = uniq, merged
    return pts, wts
