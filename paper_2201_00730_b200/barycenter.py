"""Multimarginal 1-D transport and KL barycenters on the B200
(mirror of src/barycenter.py).

``solve_mot_1d`` and ``fw_barycenter`` keep the reference signatures; the
K-marginal sweep and the Frank-Wolfe iterations run in ``csrc/mot1d.cu``
(cluster of K CTAs per problem + sample-sorted event buckets).
``fw_barycenter_batched`` is the batched entry point of BASELINE config 5.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .certify import assemble_certificate
from .exceptions import MassBalanceError
from .fw import FwConfig
from .measures import DiscreteMeasure
from .sinkhorn import SolverReport

EXHAUSTIVE_LIMIT = 10**5  # src/barycenter.py:44
MASS_TOL = 1e-9  # src/barycenter.py:43


@dataclass(frozen=True)
class BarycenterProblem:
    """K input measures, barycentric weights omega, KL strength rho
    (rho_k = omega_k rho); rho=None is the balanced problem."""

    inputs: tuple
    omega: np.ndarray
    rho: float | None = None

    def __post_init__(self):
        inputs = tuple(self.inputs)
        if len(inputs) < 2:
            raise ValueError("need at least two input measures")
        om = np.asarray(self.omega, dtype=np.float64)
        if om.shape != (len(inputs),):
            raise ValueError("omega must hold one weight per input")
        if (om <= 0).any() or abs(float(om.sum()) - 1.0) > 1e-12:
            raise ValueError("omega must be positive and sum to one")
        if self.rho is not None and not (np.isfinite(self.rho) and self.rho > 0):
            raise ValueError("rho must be positive (or None for balanced)")
        om = np.ascontiguousarray(om)
        om.flags.writeable = False
        object.__setattr__(self, "inputs", inputs)
        object.__setattr__(self, "omega", om)

    @property
    def k(self):
        return len(self.inputs)

    def rhos(self):
        if self.rho is None:
            raise ValueError("balanced problem has no KL strengths")
        return self.omega * self.rho


@dataclass(frozen=True)
class MultiPlan:
    """Plan entries: one index tuple (row of ``indices``) and a positive mass each."""

    indices: np.ndarray
    mass: np.ndarray

    def __post_init__(self):
        idx = np.ascontiguousarray(np.asarray(self.indices, dtype=np.int64))
        ms = np.ascontiguousarray(np.asarray(self.mass, dtype=np.float64))
        if idx.ndim != 2 or ms.ndim != 1 or idx.shape[0] != ms.size or ms.size == 0:
            raise ValueError("plan needs matching index rows and masses")
        if (ms <= 0).any():
            raise ValueError("plan masses must be positive")
        if idx.shape[0] > 1 and (np.diff(idx, axis=0) < 0).any():
            raise ValueError("plan support must be monotone in every coordinate")
        idx.flags.writeable = False
        ms.flags.writeable = False
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "mass", ms)

    def __len__(self):
        return int(self.mass.size)

    @property
    def k(self):
        return int(self.indices.shape[1])

    @property
    def total_mass(self):
        return float(self.mass.sum())

    def marginal(self, k, size):
        return np.bincount(self.indices[:, k], weights=self.mass, minlength=size).astype(float)


@dataclass(frozen=True)
class MultiDual:
    """One potential vector per marginal."""

    potentials: tuple

    def __post_init__(self):
        pots = []
        for f in self.potentials:
            arr = np.array(f, dtype=np.float64, copy=True)
            if arr.ndim != 1 or not np.isfinite(arr).all():
                raise ValueError("potentials must be finite vectors")
            arr.flags.writeable = False
            pots.append(arr)
        object.__setattr__(self, "potentials", tuple(pots))

    def __iter__(self):
        return iter(self.potentials)

    def __len__(self):
        return len(self.potentials)


def multimarginal_cost(points, w):
    """(sum_k w_k (x_k - B)^2, B) with B = <w, x> (src/barycenter.py:148-156)."""
    pts = np.asarray(points, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    b = float(np.dot(w, pts))
    return float(np.dot(w, (pts - b) ** 2)), b


def _pack(inputs, extra=None):
    """Ragged list of measures -> padded (x, a, [extra]) [1, K, n] + lens."""
    k = len(inputs)
    lens = np.array([len(m) for m in inputs], dtype=np.int32)
    n = int(lens.max())
    x = np.zeros((1, k, n))
    a = np.zeros((1, k, n))
    f = np.zeros((1, k, n))
    for q, m in enumerate(inputs):
        x[0, q, :lens[q]] = m.points
        x[0, q, lens[q]:] = m.points[-1]
        a[0, q, :lens[q]] = m.weights
        if extra is not None:
            f[0, q, :lens[q]] = extra[q]
    return x, a, f, lens


def _plan_from(idx, mass, count):
    c = int(count)
    return MultiPlan(D.to_np(idx[:c]).astype(np.int64), D.to_np(mass[:c]))


def solve_mot_1d_batched(x, a, omega, lens=None, stream=None):
    """Balanced K-marginal sweep on device: x, a [B, K, n].  Returns
    (duals [B, K, n], idx [B, E, K], mass [B, E], count [B], status [B])."""
    t = D.torch()
    lib = _lib.load()
    x = D.to_dev(x, t.float64)
    a = D.to_dev(a, t.float64)
    B, K, n = x.shape
    cap = K * (n - 1) + 1
    f = D.empty((B, K, n), t.float64)
    idx = D.empty((B, cap, K), t.int32)
    mass = D.empty((B, cap), t.float64)
    count = D.empty((B,), t.int32)
    status = D.empty((B,), t.int32)
    om = np.ascontiguousarray(np.asarray(omega, dtype=np.float64))
    ln = None if lens is None else np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_mot1d_workspace_size(B, K, n, ctypes.byref(size)))
    ws = D.workspace(size.value)
    _lib.check(lib.uot_mot1d_batched(
        B, K, n, ln.ctypes.data_as(ctypes.c_void_p) if ln is not None else None, _lib.ptr(x),
        _lib.ptr(a), om.ctypes.data_as(ctypes.c_void_p), _lib.ptr(f), _lib.ptr(idx),
        _lib.ptr(mass), _lib.ptr(count), _lib.ptr(status), _lib.ptr(ws),
        ctypes.c_size_t(size.value), _lib.stream_handle(stream)), "uot_mot1d_batched")
    D.torch().cuda.current_stream().synchronize()
    return f, idx, mass, count, status


def mot_states_batched(a, lens=None, stream=None):
    """Every state of the balanced sweep (zero-mass ones included), in sweep
    order: (idx [B, E, K], mass [B, E], count [B], status [B]) on the device
    (uot_mot1d_states; src/barycenter.py:209-229 visits them in this order)."""
    t = D.torch()
    lib = _lib.load()
    a = D.to_dev(a, t.float64)
    B, K, n = a.shape
    cap = K * (n - 1) + 1
    idx = D.empty((B, cap, K), t.int32)
    mass = D.empty((B, cap), t.float64)
    count = D.empty((B,), t.int32)
    status = D.empty((B,), t.int32)
    ln = None if lens is None else np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_mot1d_workspace_size(B, K, n, ctypes.byref(size)))
    ws = D.workspace(size.value)
    _lib.check(lib.uot_mot1d_states(
        B, K, n, ln.ctypes.data_as(ctypes.c_void_p) if ln is not None else None, _lib.ptr(a),
        _lib.ptr(idx), _lib.ptr(mass), _lib.ptr(count), _lib.ptr(status), _lib.ptr(ws),
        ctypes.c_size_t(size.value), _lib.stream_handle(stream)), "uot_mot1d_states")
    return idx, mass, count, status


def mot_cost_duals_batched(idx, count, cost, k, n, lens=None, stream=None):
    """Duals of the sweep from caller-evaluated state costs cost [B, E]
    (uot_mot1d_cost_duals; src/barycenter.py:224-228).  Returns f [B, K, n]."""
    t = D.torch()
    lib = _lib.load()
    idx = D.to_dev(idx, t.int32)
    count = D.to_dev(count, t.int32)
    cost = D.to_dev(cost, t.float64)
    B = idx.shape[0]
    f = t.zeros((B, k, n), dtype=t.float64, device=idx.device)
    ln = None if lens is None else np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_mot1d_workspace_size(B, k, n, ctypes.byref(size)))
    ws = D.workspace(size.value)
    _lib.check(lib.uot_mot1d_cost_duals(
        B, k, n, ln.ctypes.data_as(ctypes.c_void_p) if ln is not None else None, _lib.ptr(idx),
        _lib.ptr(count), _lib.ptr(cost), _lib.ptr(f), _lib.ptr(ws), ctypes.c_size_t(size.value),
        _lib.stream_handle(stream)), "uot_mot1d_cost_duals")
    return f


def _tuple_costs(inputs, rows, costfn):
    """costfn on each index tuple (the caller's host callable, evaluated on a
    length-K point vector exactly as src/barycenter.py:217-227 does)."""
    pts = [np.asarray(m.points, dtype=np.float64) for m in inputs]
    out = np.empty(len(rows))
    cur = np.empty(len(inputs))
    for t, row in enumerate(rows):
        for q, i in enumerate(row):
            cur[q] = pts[q][i]
        out[t] = float(costfn(cur.copy()))
    return out


def _custom_sweep(inputs, costfn):
    x, a, _, lens = _pack(inputs)
    K, n = a.shape[1], a.shape[2]
    idx, mass, count, status = mot_states_batched(a, lens)
    D.torch().cuda.current_stream().synchronize()
    if int(status[0].item()) == 1:
        raise MassBalanceError("multimarginal sweep needs equal masses")
    c = int(count[0].item())
    rows = D.to_np(idx[0, :c]).astype(np.int64)
    cost = np.zeros((1, idx.shape[1]))
    cost[0, :c] = _tuple_costs(inputs, rows, costfn)
    f = mot_cost_duals_batched(idx, count, cost, K, n, lens)
    fd = D.to_np(f[0])
    m = D.to_np(mass[0, :c])
    keep = m > 0.0
    plan = MultiPlan(rows[keep], m[keep])
    return plan, MultiDual(tuple(fd[q, :lens[q]] for q in range(K)))


def solve_mot_1d(inputs, w=None, costfn=None):
    """Balanced 1-D multimarginal transport (src/barycenter.py:169-233).

    The barycentric squared-Euclidean cost is fused into the sweep kernels; a
    custom ``costfn`` (any host callable on a length-K point vector) is
    evaluated on the tuples of the device sweep (uot_mot1d_states) and the
    duals are formed from those costs on the device (uot_mot1d_cost_duals)."""
    inputs = tuple(inputs)
    if len(inputs) < 2:
        raise ValueError("need at least two measures")
    masses = np.array([m.mass for m in inputs])
    if float(masses.max() - masses.min()) > MASS_TOL * float(masses.max()):
        raise MassBalanceError(f"multimarginal sweep needs equal masses, got {masses.tolist()}")
    if costfn is not None:
        wf = getattr(costfn, "weights", None)
        if wf is None:
            return _custom_sweep(inputs, costfn)
        w = wf
    if w is None:
        raise ValueError("need barycentric weights when costfn is omitted")
    x, a, _, lens = _pack(inputs)
    f, idx, mass, count, status = solve_mot_1d_batched(x, a, w, lens)
    st = int(status[0].item())
    if st == 1:
        raise MassBalanceError("multimarginal sweep needs equal masses")
    if st != 0:
        raise ValueError("multimarginal sweep failed (bucket capacity)")
    fd = D.to_np(f[0])
    plan = _plan_from(idx[0], mass[0], count[0].item())
    return plan, MultiDual(tuple(fd[q, :lens[q]] for q in range(len(inputs))))


def barycentric_cost_fn(w):
    """Tuple cost Cc(x) = sum_k w_k (x_k - B)^2 (src/barycenter.py:159-166)."""
    w = np.asarray(w, dtype=np.float64)

    def costfn(points):
        return multimarginal_cost(points, w)[0]

    costfn.weights = w
    return costfn


def mot_certify_batched(x, a, omega, f, idx, mass, count, lens=None, stream=None):
    """uot_mot_certify on device tensors (layout of solve_mot_1d_batched):
    returns out [B, 6] = (primal, dual, support violation, marginal
    violation, exhaustive feasibility violation, exhaustive-sweep flag)."""
    t = D.torch()
    lib = _lib.load()
    x, a, f = (D.to_dev(v, t.float64) for v in (x, a, f))
    B, K, n = x.shape
    idx = D.to_dev(idx, t.int32)
    mass = D.to_dev(mass, t.float64)
    count = D.to_dev(count, t.int32)
    out = t.zeros((B, 6), dtype=t.float64, device=x.device)
    om = np.ascontiguousarray(np.asarray(omega, dtype=np.float64))
    ln = None if lens is None else np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
    ws = D.workspace(64 * K + 512)
    _lib.check(lib.uot_mot_certify(
        B, K, n, ln.ctypes.data_as(ctypes.c_void_p) if ln is not None else None, _lib.ptr(x),
        _lib.ptr(a), om.ctypes.data_as(ctypes.c_void_p), _lib.ptr(f), _lib.ptr(idx),
        _lib.ptr(mass), _lib.ptr(count), _lib.ptr(out), _lib.ptr(ws), ctypes.c_size_t(64 * K + 512),
        _lib.stream_handle(stream)), "uot_mot_certify")
    D.torch().cuda.current_stream().synchronize()
    return out


def _certify_inputs(inputs, w, plan, duals, costfn=None, grid=True):
    """uot_mot_certify (barycentric cost, weights w) or, for a custom costfn,
    uot_mot_certify_costs with costfn evaluated on the plan tuples and (grid)
    on the whole index grid when it holds at most EXHAUSTIVE_LIMIT tuples."""
    inputs = tuple(inputs)
    x, a, f, lens = _pack(inputs, extra=tuple(duals))
    K, n = x.shape[1], x.shape[2]
    cap = K * (n - 1) + 1
    idx = np.zeros((1, cap, K), dtype=np.int32)
    mass = np.zeros((1, cap))
    e = len(plan)
    if e > cap:
        raise ValueError("plan has more entries than a monotone sweep can produce")
    idx[0, :e] = plan.indices
    mass[0, :e] = plan.mass
    if costfn is None:
        out = mot_certify_batched(x, a, w, f, idx, mass, np.array([e], dtype=np.int32), lens)
        return D.to_np(out[0], readonly=False)
    t = D.torch()
    lib = _lib.load()
    ecost = np.zeros((1, cap))
    ecost[0, :e] = _tuple_costs(inputs, np.asarray(plan.indices, dtype=np.int64), costfn)
    gsize = int(np.prod([len(m) for m in inputs], dtype=np.float64))
    gcost = None
    if grid and gsize <= EXHAUSTIVE_LIMIT:
        rows = np.array(list(np.ndindex(*[len(m) for m in inputs])), dtype=np.int64)
        gcost = D.to_dev(_tuple_costs(inputs, rows, costfn)[None], t.float64)
    ad, fd = D.to_dev(a, t.float64), D.to_dev(f, t.float64)
    idd, md = D.to_dev(idx, t.int32), D.to_dev(mass, t.float64)
    cnt = D.to_dev(np.array([e], dtype=np.int32), t.int32)
    ed = D.to_dev(ecost, t.float64)
    out = t.zeros((1, 6), dtype=t.float64, device=ad.device)
    ws = D.workspace(64 * K + 512)
    _lib.check(lib.uot_mot_certify_costs(
        1, K, n, lens.ctypes.data_as(ctypes.c_void_p), _lib.ptr(ad), _lib.ptr(fd), _lib.ptr(idd),
        _lib.ptr(md), _lib.ptr(cnt), _lib.ptr(ed), _lib.ptr(gcost) if gcost is not None else None,
        _lib.ptr(out), _lib.ptr(ws), ctypes.c_size_t(64 * K + 512), None),
        "uot_mot_certify_costs")
    t.cuda.current_stream().synchronize()
    return D.to_np(out[0], readonly=False)


def _weights_of(costfn, w):
    """Barycentric weights of a built-in cost, or None for a custom costfn."""
    if costfn is None:
        if w is None:
            raise ValueError("need barycentric weights when costfn is omitted")
        return np.asarray(w, dtype=np.float64)
    return getattr(costfn, "weights", None)


def _custom(costfn, w):
    return costfn if (costfn is not None and w is None) else None


def plan_cost(plan, inputs, costfn):
    """sum_e mass_e Cc(tuple_e) (src/barycenter.py:236-240), on the device."""
    inputs = tuple(inputs)
    w = _weights_of(costfn, None)
    duals = MultiDual(tuple(np.zeros(len(m)) for m in inputs))
    return float(_certify_inputs(inputs, w, plan, duals, _custom(costfn, w), grid=False)[0])


def dual_feasibility_exhaustive(inputs, duals, costfn):
    """max over the whole index grid of sum_k f_k - Cc (positive = violation)
    (src/barycenter.py:243-258); grids up to 1e5 tuples, on the device."""
    inputs = tuple(inputs)
    if int(np.prod([len(m) for m in inputs], dtype=np.float64)) > EXHAUSTIVE_LIMIT:
        raise ValueError("grid too large for the exhaustive check")
    w = _weights_of(costfn, None)
    plan = MultiPlan(np.zeros((1, len(inputs)), dtype=np.int64), np.array([1.0]))
    v = _certify_inputs(inputs, w, plan, duals, _custom(costfn, w))
    return float(v[4])


def mot_certificate(inputs, w, plan, duals, costfn=None, rel_tol=1e-9):
    """Optimality certificate of a balanced multi-marginal solution
    (src/barycenter.py:261-295): primal = plan cost, dual = sum_k <a_k, f_k>,
    violation = max(support, marginal, exhaustive feasibility when the grid
    has at most 1e5 tuples), tolerance rel_tol (1 + |primal|)."""
    inputs = tuple(inputs)
    wv = _weights_of(costfn, w)
    v = _certify_inputs(inputs, wv, plan, duals, _custom(costfn, wv))
    primal, dual = float(v[0]), float(v[1])
    violation = max(float(v[2]), float(v[3]), float(v[4]))
    return assemble_certificate(primal, dual, violation, rel_tol * (1.0 + abs(primal)))


def multimarginal_lambda(duals, inputs, w, rho):
    """Optimal zero-sum translation (src/barycenter.py:298-317):
    rho_k q_k - (rho_k / sum rho) sum_j rho_j q_j, q_k = log <a_k, e^(-f_k/rho_k)>."""
    from .duality import kl_scalars

    w = np.asarray(w, dtype=np.float64)
    rhos = w * float(rho)
    q = []
    for fk, m, rk in zip(duals.potentials, inputs, rhos):
        out = kl_scalars(m.weights, m.weights, fk, fk, rk, rk)
        q.append(-float(out[0, 2].item()) / rk)  # Smin = -rho LSE
    q = np.array(q)
    if not np.all(np.isfinite(q)):
        raise ValueError("zero-mass input or diverging reduction")
    rho_tot = float(rhos.sum())
    return rhos * q - (rhos / rho_tot) * float(np.dot(rhos, q))


@dataclass
class BaryBatchResult:
    f: object
    h0: object
    fw_gap: object
    pd_gap: object
    iterations: object
    idx: object
    mass: object
    count: object
    summary: object
    status: object
    supp_hash: object = None
    supp_nnz: object = None
    replay: object = None


def fw_barycenter_batched(x, a, omega, rho=1.0, max_iters=1000, step="linesearch",
                          gap_tol=1e-6, early_exit=False, f0=None, lens=None, stream=None,
                          step_in=None, trace_support=False):
    """Batched KL barycenter FW on device: x, a [B, K, n] (sorted rows).
    Returns device tensors; f is translated (report.final).  ``step_in``
    [B, max_iters] replays given step sizes (the reference's gamma_t);
    ``trace_support`` records every iteration's plan-support hash / count."""
    t = D.torch()
    lib = _lib.load()
    x = D.to_dev(x, t.float64)
    a = D.to_dev(a, t.float64)
    B, K, n = x.shape
    cap = K * (n - 1) + 1
    f = t.zeros((B, K, n), dtype=t.float64, device=x.device) if f0 is None else \
        D.to_dev(f0, t.float64).clone()
    r = BaryBatchResult(
        f=f, h0=D.empty((B, max_iters), t.float64), fw_gap=D.empty((B, max_iters), t.float64),
        pd_gap=D.empty((B, max_iters), t.float64), iterations=D.empty((B,), t.int32),
        idx=D.empty((B, cap, K), t.int32), mass=D.empty((B, cap), t.float64),
        count=D.empty((B,), t.int32), summary=D.empty((B, 2), t.float64),
        status=D.empty((B,), t.int32))
    om = np.ascontiguousarray(np.asarray(omega, dtype=np.float64))
    ln = None if lens is None else np.ascontiguousarray(np.asarray(lens, dtype=np.int32))
    desc = _lib.BaryDesc(
        batch=B, k=K, n=n, omega=om.ctypes.data_as(ctypes.c_void_p),
        lens=ln.ctypes.data_as(ctypes.c_void_p) if ln is not None else None, rho=float(rho),
        step=_lib.STEP_LINESEARCH if step == "linesearch" else _lib.STEP_HARMONIC,
        max_iters=int(max_iters), gap_tol=float(gap_tol), early_exit=1 if early_exit else 0,
        x=_lib.ptr(x), a=_lib.ptr(a), f=_lib.ptr(f), h0=_lib.ptr(r.h0),
        fw_gap=_lib.ptr(r.fw_gap), pd_gap=_lib.ptr(r.pd_gap), iterations=_lib.ptr(r.iterations),
        idx=_lib.ptr(r.idx), mass=_lib.ptr(r.mass), count=_lib.ptr(r.count),
        summary=_lib.ptr(r.summary), status=_lib.ptr(r.status))
    from .fw import _trace_args

    _trace_args(desc, r, B, max_iters, step_in, None, trace_support, x.device)
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_bary_workspace_size(ctypes.byref(desc), ctypes.byref(size)))
    ws = D.workspace(size.value)
    _lib.check(lib.uot_bary_run(ctypes.byref(desc), _lib.ptr(ws), ctypes.c_size_t(size.value),
                                _lib.stream_handle(stream)), "uot_bary_run")
    t.cuda.current_stream().synchronize()  # omega / lens are host buffers of this frame
    return r


def fw_barycenter(problem, config=FwConfig(), init=None):
    """Frank-Wolfe on the invariant dual of the KL multimarginal problem
    (src/barycenter.py:330-430).  Returns ``(report, plan)``.

    The certificate's feasibility term is the exhaustive grid check when the
    index grid holds <= 1e5 tuples, else 0 (:416-418), evaluated on the
    device on the translated potentials (the translation sums to zero,
    :298-317, so the grid maximum is the same).  ``step="pairwise"`` takes
    the line-search branch, as the reference's step dispatch does (:397-407:
    anything but "harmonic" runs the ternary line search)."""
    if problem.rho is None:
        raise ValueError("balanced barycenters route directly through solve_mot_1d")
    step = "linesearch" if config.step == "pairwise" else config.step
    inputs = problem.inputs
    pots0 = None
    if init is not None:
        pots0 = [np.asarray(f, dtype=np.float64) for f in init.potentials]
        if any(p.size != len(m) for p, m in zip(pots0, inputs)):
            raise ValueError("initial potentials do not match the inputs")
    x, a, f0, lens = _pack(inputs, pots0)
    tic = time.perf_counter_ns()
    r = fw_barycenter_batched(x, a, problem.omega, problem.rho, config.max_iters, step,
                              config.gap_tol, early_exit=True, f0=f0, lens=lens)
    st = int(r.status[0].item())
    if st == 1:
        raise MassBalanceError("translated masses disagree; translation broken")
    if st != 0:
        raise ValueError("barycenter sweep failed (bucket capacity)")
    its = int(r.iterations[0].item())
    wall = (time.perf_counter_ns() - tic) // max(its, 1)
    pd = D.to_np(r.pd_gap[0, :its], readonly=False)
    trace = {"h0": D.to_np(r.h0[0, :its], readonly=False),
             "fw_gap": D.to_np(r.fw_gap[0, :its], readonly=False), "pd_gap": pd,
             "wall_ns": np.full(its, wall, dtype=np.int64)}
    converged = bool(its > 0 and pd[-1] < config.gap_tol)
    fd = D.to_np(r.f[0])
    final = MultiDual(tuple(fd[q, :lens[q]] for q in range(len(inputs))))
    plan = _plan_from(r.idx[0], r.mass[0], r.count[0].item())
    primal, dual = (float(v) for v in D.to_np(r.summary[0]))
    feas = 0.0
    if int(np.prod([len(m) for m in inputs], dtype=np.float64)) <= EXHAUSTIVE_LIMIT:
        feas = dual_feasibility_exhaustive(inputs, final, barycentric_cost_fn(problem.omega))
    cert = assemble_certificate(primal, dual, feas, config.gap_tol)
    report = SolverReport(final=final, iterations=its, converged=converged, trace=trace,
                          certificate=cert, plan=plan)
    return report, plan


def extract_barycenter(plan, inputs, w):
    """One atom per plan entry at <w, tuple points> with the entry's mass;
    coincident atoms merge (src/barycenter.py:433-443).  Host-side gather of
    the (already computed) plan."""
    w = np.asarray(w, dtype=np.float64)
    pts = np.stack([inputs[k].points[plan.indices[:, k]] for k in range(plan.k)], axis=1)
    return DiscreteMeasure(pts @ w, plan.mass)


# File formats (paper_2201_00730_b200/formats.py), re-exported where the reference defines them.


def write_multiplan_csv(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.write_multiplan_csv`."""
    from . import formats as _F

    return _F.write_multiplan_csv(*args, **kwargs)


def read_multiplan_csv(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.read_multiplan_csv`."""
    from . import formats as _F

    return _F.read_multiplan_csv(*args, **kwargs)
