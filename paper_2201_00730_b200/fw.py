"""Frank-Wolfe for unregularised 1-D UOT on the B200 (mirror of src/fw.py).

``fw_solve(prob, config, init, reference)`` keeps the reference signature and
``SolverReport``; ``fw_solve_batched`` runs a batch of independent problems
(BASELINE config 2) in one launch of ``csrc/fw1d.cu``: one CTA per problem,
every iteration (tilt, oracle, gaps, Newton line search, update) on chip.
``step="pairwise"`` runs pairwise FW (src/fw.py:255-357) with the atom store
in the device workspace.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .certify import assemble_certificate
from .duality import DualPair
from .entropies import KL, Berg
from .exceptions import InfeasibleDualError, MassBalanceError, UnsupportedEntropyError
from .measures import PowerDistance
from .ot1d import SparsePlan
from .sinkhorn import SolverReport

FEAS_TOL = 1e-9  # src/fw.py:48


@dataclass(frozen=True)
class FwConfig:
    """Step rule ('harmonic', 'linesearch', 'pairwise'), budget, gap target."""

    step: str = "linesearch"
    max_iters: int = 5000
    gap_tol: float = 1e-6

    def __post_init__(self):
        if self.step not in ("harmonic", "linesearch", "pairwise"):
            raise ValueError("step must be 'harmonic', 'linesearch', or 'pairwise'")
        if self.gap_tol <= 0:
            raise ValueError("gap_tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be positive")


@dataclass
class FwBatchResult:
    """Device tensors of a batched run (see fw_solve_batched)."""

    f: object
    g: object
    h0: object
    fw_gap: object
    pd_gap: object
    iterations: object
    ei: object
    ej: object
    em: object
    count: object
    summary: object
    status: object
    step_size: object
    natoms: object = None  # pairwise: active atoms after each iteration


def fw_solve_batched(x, y, a, b, rho1=1.0, rho2=1.0, p=2.0, max_iters=500, step="linesearch",
                     gap_tol=1e-6, early_exit=False, f0=None, g0=None, stream=None):
    """Batched FW on device: x, a [B, N]; y, b [B, M] sorted supports.

    ``early_exit=False`` runs exactly ``max_iters`` iterations per problem
    (BASELINE fixed-iteration configs); True applies fw.py:220-222 per
    problem.  f/g come back translated by lambda* (report.final)."""
    t = D.torch()
    lib = _lib.load()
    x, y, a, b = (D.to_dev(v, t.float64) for v in (x, y, a, b))
    if x.ndim == 1:
        x, y, a, b = (v.unsqueeze(0) for v in (x, y, a, b))
    B, n = x.shape
    m = y.shape[1]
    f = t.zeros((B, n), dtype=t.float64, device=x.device) if f0 is None else \
        D.to_dev(f0, t.float64).reshape(B, n).clone()
    g = t.zeros((B, m), dtype=t.float64, device=x.device) if g0 is None else \
        D.to_dev(g0, t.float64).reshape(B, m).clone()
    r = FwBatchResult(
        f=f, g=g, h0=D.empty((B, max_iters), t.float64), fw_gap=D.empty((B, max_iters), t.float64),
        pd_gap=D.empty((B, max_iters), t.float64), iterations=D.empty((B,), t.int32),
        ei=D.empty((B, n + m - 1), t.int32), ej=D.empty((B, n + m - 1), t.int32),
        em=D.empty((B, n + m - 1), t.float64), count=D.empty((B,), t.int32),
        summary=D.empty((B, 3), t.float64), status=D.empty((B,), t.int32),
        step_size=t.zeros((B, max_iters), dtype=t.float64, device=x.device),
        natoms=t.zeros((B, max_iters), dtype=t.int32, device=x.device) if step == "pairwise"
        else None)
    if step not in ("linesearch", "harmonic", "pairwise"):
        raise ValueError("step must be 'harmonic', 'linesearch', or 'pairwise'")
    code = {"linesearch": _lib.STEP_LINESEARCH, "harmonic": _lib.STEP_HARMONIC,
            "pairwise": _lib.STEP_PAIRWISE}[step]
    desc = _lib.FwDesc(
        batch=B, n=n, m=m, p=float(p), rho1=float(rho1), rho2=float(rho2),
        step=code,
        max_iters=int(max_iters), gap_tol=float(gap_tol), early_exit=1 if early_exit else 0,
        x=_lib.ptr(x), y=_lib.ptr(y), a=_lib.ptr(a), b=_lib.ptr(b), f=_lib.ptr(f), g=_lib.ptr(g),
        h0=_lib.ptr(r.h0), fw_gap=_lib.ptr(r.fw_gap), pd_gap=_lib.ptr(r.pd_gap),
        iterations=_lib.ptr(r.iterations), ei=_lib.ptr(r.ei), ej=_lib.ptr(r.ej),
        em=_lib.ptr(r.em), count=_lib.ptr(r.count), summary=_lib.ptr(r.summary),
        status=_lib.ptr(r.status), step_size=_lib.ptr(r.step_size),
        natoms=_lib.ptr(r.natoms) if r.natoms is not None else None)
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_fw1d_workspace_size(ctypes.byref(desc), ctypes.byref(size)))
    ws = D.workspace(size.value)
    _lib.check(lib.uot_fw1d_run(ctypes.byref(desc), _lib.ptr(ws), ctypes.c_size_t(size.value),
                                _lib.stream_handle(stream)), "uot_fw1d_run")
    return r


def feasibility_violation(x, y, f, g, p=2.0, stream=None):
    """max(0, max_ij f_i + g_j - |x_i - y_j|^p) per problem (device, fp64)."""
    t = D.torch()
    lib = _lib.load()
    x, y, f, g = (D.to_dev(v, t.float64) for v in (x, y, f, g))
    if x.ndim == 1:
        x, y, f, g = (v.unsqueeze(0) for v in (x, y, f, g))
    out = D.empty((x.shape[0],), t.float64)
    _lib.check(lib.uot_feasibility_1d(x.shape[0], x.shape[1], y.shape[1], _lib.ptr(x),
                                      _lib.ptr(y), ctypes.c_double(p), _lib.ptr(f), _lib.ptr(g),
                                      _lib.ptr(out), _lib.stream_handle(stream)))
    return out


def _check_problem(prob):
    if prob.eps != 0:
        raise ValueError("frank-wolfe solves the unregularized problem; need eps = 0")
    for spec in (prob.ent1, prob.ent2):
        if not isinstance(spec, (KL, Berg)):
            raise UnsupportedEntropyError("frank-wolfe needs strictly convex conjugates (KL or Berg)")
        if not isinstance(spec, KL):
            raise UnsupportedEntropyError("the B200 FW path runs KL penalties")
    if not isinstance(prob.cost, PowerDistance):
        raise UnsupportedEntropyError("the B200 FW path runs |x - y|^p costs")


def fw_solve(prob, config=FwConfig(), init=None, reference=None):
    """Maximise the invariant dual at eps = 0 (src/fw.py:176-232)."""
    _check_problem(prob)
    n, m = len(prob.alpha), len(prob.beta)
    d = init if init is not None else DualPair.zeros(n, m)
    prob.check_pair(d)
    x, y = prob.alpha.points, prob.beta.points
    p = prob.cost.p
    viol = float(feasibility_violation(x, y, d.f, d.g, p)[0].item())
    if viol > FEAS_TOL:
        raise InfeasibleDualError("initial pair violates f + g <= C")
    if reference is not None:
        raise UnsupportedEntropyError("err_f tracing is not on the B200 FW path")
    tic = time.perf_counter_ns()
    r = fw_solve_batched(x, y, prob.alpha.weights, prob.beta.weights, prob.ent1.rho,
                         prob.ent2.rho, p, config.max_iters, config.step, config.gap_tol,
                         early_exit=True, f0=d.f, g0=d.g)
    st = int(r.status[0].item())
    if st == 1:
        raise MassBalanceError("reweighted marginal masses disagree; optimal translation looks broken")
    its = int(r.iterations[0].item())
    wall = (time.perf_counter_ns() - tic) // max(its, 1)
    h0 = D.to_np(r.h0[0, :its], readonly=False)
    pd = D.to_np(r.pd_gap[0, :its], readonly=False)
    fg = D.to_np(r.fw_gap[0, :its], readonly=False)
    converged = bool(its > 0 and pd[-1] < config.gap_tol)
    k = int(r.count[0].item())
    plan = SparsePlan(D.to_np(r.ei[0, :k]), D.to_np(r.ej[0, :k]), D.to_np(r.em[0, :k]))
    primal, dual, lam = (float(v) for v in D.to_np(r.summary[0]))
    fin_f = D.to_np(r.f[0])
    fin_g = D.to_np(r.g[0])
    # feasibility of the untranslated iterate (f - lam, g + lam) (fw.py:238-240)
    feas = float(feasibility_violation(x, y, fin_f - lam, fin_g + lam, p)[0].item())
    cert = assemble_certificate(primal, dual, feas, config.gap_tol)
    trace = {"h0": h0, "fw_gap": fg, "pd_gap": pd,
             "wall_ns": np.full(its, wall, dtype=np.int64)}
    return SolverReport(final=DualPair(fin_f, fin_g), iterations=its, converged=converged,
                        trace=trace, certificate=cert, plan=plan)
