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
from .exceptions import (InfeasibleDualError, MassBalanceError, NewtonError, SubmodularityError,
                         UnsupportedEntropyError)
from .measures import ExplicitMatrix, PowerDistance, check_submodular
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
    err_f: object = None   # with ref_f: translated-iterate error per iteration
    cost: object = None    # explicit cost matrix kept alive for the launch
    supp_hash: object = None  # trace_support: per-iteration plan-support hash (int64 view)
    supp_nnz: object = None   # trace_support: per-iteration plan entry count
    replay: object = None     # replayed step sizes / away positions kept alive


def _trace_args(desc, r, B, T, step_in, away_in, trace_support, device):
    """Fill the replay / support-trace fields of an FW or barycenter descriptor."""
    t = D.torch()
    keep = []
    if step_in is not None:
        st = D.to_dev(step_in, t.float64).reshape(B, T).contiguous()
        keep.append(st)
        desc.step_in = _lib.ptr(st)
    if away_in is not None:
        aw = D.to_dev(away_in, t.int32).reshape(B, T).contiguous()
        keep.append(aw)
        desc.away_in = _lib.ptr(aw)
    if trace_support:
        r.supp_hash = t.zeros((B, T), dtype=t.int64, device=device)
        r.supp_nnz = t.zeros((B, T), dtype=t.int32, device=device)
        desc.supp_hash = _lib.ptr(r.supp_hash)
        desc.supp_nnz = _lib.ptr(r.supp_nnz)
    r.replay = keep


def fw_solve_batched(x, y, a, b, rho1=1.0, rho2=1.0, p=2.0, max_iters=500, step="linesearch",
                     gap_tol=1e-6, early_exit=False, f0=None, g0=None, stream=None, ref_f=None,
                     C=None, ent1="kl", ent2="kl", step_in=None, away_in=None,
                     trace_support=False):
    """Batched FW on device: x, a [B, N]; y, b [B, M] sorted supports;
    ``C`` [B, N, M] (optional) an explicit Monge cost instead of |x - y|^p;
    ``ent1`` / ``ent2`` "kl" or "berg" (Berg runs the generic path,
    csrc/fw1d_generic.cu).

    ``early_exit=False`` runs exactly ``max_iters`` iterations per problem
    (BASELINE fixed-iteration configs); True applies fw.py:220-222 per
    problem.  f/g come back translated by lambda* (report.final).

    Parity mode: ``step_in`` [B, max_iters] replays given step sizes (the
    reference's gamma_t) and, for pairwise, ``away_in`` [B, max_iters] the
    away positions (-1 = no step); ``trace_support`` records every
    iteration's plan-support hash and entry count (include/uot_b200.h)."""
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
    ref_d = None
    if ref_f is not None:  # err_f trace against a reference potential (fw.py:217-219)
        ref_d = D.to_dev(ref_f, t.float64).reshape(B, n).contiguous()
        r.err_f = t.zeros((B, max_iters), dtype=t.float64, device=x.device)
        desc.ref_f = _lib.ptr(ref_d)
        desc.err_f = _lib.ptr(r.err_f)
    if C is not None:
        r.cost = D.to_dev(C, t.float64).reshape(B, n, m).contiguous()
        desc.c = _lib.ptr(r.cost)
    codes = {"kl": _lib.ENT_KL, "berg": _lib.ENT_BERG}
    desc.ent1, desc.ent2 = codes[ent1], codes[ent2]
    _trace_args(desc, r, B, max_iters, step_in, away_in, trace_support, x.device)
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_fw1d_workspace_size(ctypes.byref(desc), ctypes.byref(size)))
    ws = D.workspace(size.value)
    _lib.check(lib.uot_fw1d_run(ctypes.byref(desc), _lib.ptr(ws), ctypes.c_size_t(size.value),
                                _lib.stream_handle(stream)), "uot_fw1d_run")
    return r


def feasibility_violation(x, y, f, g, p=2.0, stream=None, C=None):
    """max(0, max_ij f_i + g_j - C_ij) per problem (device, fp64), C_ij =
    |x_i - y_j|^p or the explicit ``C`` [B, N, M]."""
    t = D.torch()
    lib = _lib.load()
    x, y, f, g = (D.to_dev(v, t.float64) for v in (x, y, f, g))
    if x.ndim == 1:
        x, y, f, g = (v.unsqueeze(0) for v in (x, y, f, g))
    out = D.empty((x.shape[0],), t.float64)
    if C is not None:
        B, n, m = x.shape[0], x.shape[1], y.shape[1]
        C = D.to_dev(C, t.float64).reshape(B, n, m).contiguous()
        _lib.check(lib.uot_feasibility_explicit(B, n, m, _lib.ptr(C), _lib.ptr(f), _lib.ptr(g),
                                                _lib.ptr(out), _lib.stream_handle(stream)))
        return out
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
    if not isinstance(prob.cost, (PowerDistance, ExplicitMatrix)):
        raise TypeError(f"unknown cost specification {prob.cost!r}")


def _default_init(prob, C):
    """Zero pair, or half row / column minima for a cost with negative
    entries so that f + g <= C (src/fw.py:151-156); minima on the device."""
    n, m = len(prob.alpha), len(prob.beta)
    if C is None:  # |x - y|^p >= 0
        return DualPair.zeros(n, m)
    if float(C.min().item()) >= 0:
        return DualPair.zeros(n, m)
    return DualPair(D.to_np(0.5 * C.min(dim=1).values), D.to_np(0.5 * C.min(dim=0).values))


def _first_lmo_errors(prob, x, y, p, C, d):
    """Raise what the first FW iteration's translation / mass check raise
    (one device iteration: NewtonError for a Berg marginal, MassBalanceError)."""
    r = fw_solve_batched(x, y, prob.alpha.weights, prob.beta.weights, prob.ent1.rho,
                         prob.ent2.rho, p, 1, "harmonic", 1e-12, early_exit=False, f0=d.f,
                         g0=d.g, C=C, ent1="kl" if isinstance(prob.ent1, KL) else "berg",
                         ent2="kl" if isinstance(prob.ent2, KL) else "berg")
    st = int(r.status[0].item())
    if st == 1:
        raise MassBalanceError("reweighted marginal masses disagree; optimal translation looks broken")
    if st == 3:
        raise NewtonError("translation Newton did not reach the residual target")


def fw_solve(prob, config=FwConfig(), init=None, reference=None):
    """Maximise the invariant dual at eps = 0 (src/fw.py:176-232)."""
    _check_problem(prob)
    kl = isinstance(prob.ent1, KL) and isinstance(prob.ent2, KL)
    n, m = len(prob.alpha), len(prob.beta)
    x, y = prob.alpha.points, prob.beta.points
    C = None
    p = 2.0
    if isinstance(prob.cost, ExplicitMatrix):
        if prob.cost.matrix.shape != (n, m):
            raise ValueError(f"explicit cost shape {prob.cost.matrix.shape} does not match "
                             f"supports ({n}, {m})")
        C = D.to_dev(prob.cost.matrix, D.torch().float64)
    else:
        p = prob.cost.p
    d = init if init is not None else _default_init(prob, C)
    prob.check_pair(d)
    viol = float(feasibility_violation(x, y, d.f, d.g, p, C=C)[0].item())
    if viol > FEAS_TOL:
        raise InfeasibleDualError("initial pair violates f + g <= C")
    if C is not None:  # the oracle's Monge check (src/ot1d.py:106, via _lmo)
        try:
            check_submodular(prob.cost.matrix)
        except SubmodularityError as monge:
            # the reference meets it inside the first _lmo (src/fw.py:159-173), after
            # the translation and the mass check: surface what those raise first
            _first_lmo_errors(prob, x, y, p, C, d)
            raise monge
    if config.step == "pairwise" and not kl:
        return _pfw_solve_host(prob, config, d, reference)
    if reference is not None and len(reference.f) != n:
        raise ValueError("reference potential does not match the problem")
    tic = time.perf_counter_ns()
    r = fw_solve_batched(x, y, prob.alpha.weights, prob.beta.weights, prob.ent1.rho,
                         prob.ent2.rho, p, config.max_iters, config.step, config.gap_tol,
                         early_exit=True, f0=d.f, g0=d.g,
                         ref_f=None if reference is None else reference.f, C=C,
                         ent1="kl" if isinstance(prob.ent1, KL) else "berg",
                         ent2="kl" if isinstance(prob.ent2, KL) else "berg")
    st = int(r.status[0].item())
    if st == 1:
        raise MassBalanceError("reweighted marginal masses disagree; optimal translation looks broken")
    if st == 3:
        raise NewtonError("translation Newton did not reach the residual target")
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
    feas = float(feasibility_violation(x, y, fin_f - lam, fin_g + lam, p, C=C)[0].item())
    cert = assemble_certificate(primal, dual, feas, config.gap_tol)
    trace = {"h0": h0, "fw_gap": fg, "pd_gap": pd,
             "wall_ns": np.full(its, wall, dtype=np.int64)}
    if reference is not None:
        trace["err_f"] = D.to_np(r.err_f[0, :its], readonly=False)
    return SolverReport(final=DualPair(fin_f, fin_g), iterations=its, converged=converged,
                        trace=trace, certificate=cert, plan=plan)


# File formats (paper_2201_00730_b200/formats.py), re-exported where the reference defines them.


def write_gap_csv(*args, **kwargs):
    """See :func:`paper_2201_00730_b200.formats.write_gap_csv`."""
    from . import formats as _F

    return _F.write_gap_csv(*args, **kwargs)


# ---------------------------------------------------------------------------
# Single-step building blocks of src/fw.py (ternary search, the H0 line
# search, the pairwise atom store and one pairwise step), for callers that
# drive FW themselves; the solvers above run whole iterations on the device.

ATOM_DEDUP_TOL = 1e-12  # src/fw.py:47


def ternary_max(fn, lo=0.0, hi=1.0, iters=60):
    """Ternary search for the maximiser of a concave scalar function (:118-128)."""
    a, b = float(lo), float(hi)
    for _ in range(iters):
        m1, m2 = a + (b - a) / 3.0, b - (b - a) / 3.0
        if fn(m1) < fn(m2):
            a = m1
        else:
            b = m2
    return 0.5 * (a + b)


def _h0_value(prob, f, g):
    """_h0 (src/fw.py:106-115): KL closed form, else the translated sums."""
    from .duality import kl_scalars, translation

    if isinstance(prob.ent1, KL) and isinstance(prob.ent2, KL):
        return float(kl_scalars(prob.alpha.weights, prob.beta.weights, f, g, prob.ent1.rho,
                                prob.ent2.rho)[0, 1].item())
    return float(translation(prob, f, g, value=True)[3][0].item())


def line_search_h0(prob, current, target):
    """Step in [0, 1] maximising H0 on the segment: 60 ternary steps and an
    endpoint comparison (:131-148); every H0 value on the device."""
    for spec in (prob.ent1, prob.ent2):
        if not isinstance(spec, (KL, Berg)):
            raise UnsupportedEntropyError("frank-wolfe needs strictly convex conjugates (KL or Berg)")

    def value(gamma):
        return _h0_value(prob, (1.0 - gamma) * current.f + gamma * target.f,
                         (1.0 - gamma) * current.g + gamma * target.g)

    gamma = ternary_max(value, 0.0, 1.0, iters=60)
    return max(((value(c), c) for c in (gamma, 0.0, 1.0)), key=lambda z: z[0])[1]


class AtomStore:
    """Active dual-pair atoms of pairwise FW with convex weights (:70-95)."""

    def __init__(self, r_atoms, s_atoms, weights):
        r = np.atleast_2d(np.asarray(r_atoms, dtype=np.float64))
        s = np.atleast_2d(np.asarray(s_atoms, dtype=np.float64))
        w = np.atleast_1d(np.asarray(weights, dtype=np.float64))
        if r.shape[0] != s.shape[0] or r.shape[0] != w.size or w.size == 0:
            raise ValueError("store arrays must agree on the number of atoms")
        if np.any(w < -1e-14):
            raise ValueError("weights must stay nonnegative")
        if abs(w.sum() - 1.0) > 1e-12:
            raise ValueError("weights must sum to one")
        self.r_atoms, self.s_atoms, self.weights = r, s, w

    def current(self):
        return DualPair(self.weights @ self.r_atoms, self.weights @ self.s_atoms)


def _pfw_iteration(prob, store):
    """One pairwise step (src/fw.py:275-310); returns (new_store, diag) with
    the iterate, the oracle plan, the linear gap, H0 and the plan's primal.
    Device LMO (updated marginals + 1-D oracle), H0 values, primal; the atom
    bookkeeping is host work on the store."""
    from .duality import eval_primal, updated_marginals
    from .measures import DiscreteMeasure
    from .ot1d import solve_ot_1d

    d = store.current()
    ta, tb = updated_marginals(prob, d)
    mass_a, mass_b = float(ta.sum()), float(tb.sum())
    if abs(mass_a - mass_b) > 1e-9 * max(mass_a, mass_b):  # fw.py:161-166
        raise MassBalanceError(f"reweighted marginal masses disagree ({mass_a:.12g} vs "
                               f"{mass_b:.12g}); optimal translation looks broken")
    plan, atom = solve_ot_1d(DiscreteMeasure(prob.alpha.points, ta),
                             DiscreteMeasure(prob.beta.points, tb), prob.cost)
    diag = {"pair": d, "plan": plan,
            "fw_gap": float(np.dot(ta, atom.f - d.f) + np.dot(tb, atom.g - d.g)),
            "dual": _h0_value(prob, d.f, d.g), "primal": eval_primal(prob, plan)}
    scores = np.where(store.weights > 0, store.r_atoms @ ta + store.s_atoms @ tb, np.inf)
    away = int(np.argmin(scores))
    max_step = float(store.weights[away])
    dr, ds = atom.f - store.r_atoms[away], atom.g - store.s_atoms[away]
    if max_step <= 0.0 or (np.abs(dr).max() < ATOM_DEDUP_TOL and np.abs(ds).max() < ATOM_DEDUP_TOL):
        return store, diag

    def value(gamma):
        return _h0_value(prob, d.f + gamma * dr, d.g + gamma * ds)

    gamma = ternary_max(value, 0.0, max_step, iters=60)
    gamma = max(((value(c), c) for c in (gamma, 0.0, max_step)), key=lambda z: z[0])[1]
    if gamma <= 0.0:
        return store, diag
    w = store.weights.copy()
    w[away] = max(w[away] - gamma, 0.0)
    r_atoms, s_atoms = store.r_atoms, store.s_atoms
    dist = np.maximum(np.abs(r_atoms - atom.f).max(axis=1), np.abs(s_atoms - atom.g).max(axis=1))
    hit = np.nonzero(dist < ATOM_DEDUP_TOL)[0]
    if hit.size:
        w[hit[0]] += gamma
    else:
        r_atoms = np.vstack([r_atoms, atom.f])
        s_atoms = np.vstack([s_atoms, atom.g])
        w = np.concatenate([w, [gamma]])
    keep = w > 0
    return AtomStore(r_atoms[keep], s_atoms[keep], w[keep]), diag


def pfw_step(prob, store):
    """One pairwise weight transfer (:255-323): device LMO (updated marginals,
    1-D oracle), the least aligned active atom as donor, a ternary H0 line
    search on [0, w_away] with endpoint comparison, dedup merge of the new
    atom and removal of emptied atoms."""
    if store.weights.size == 0:
        raise ValueError("atom store is empty")
    _check_problem(prob)
    return _pfw_iteration(prob, store)[0]


def _pfw_solve_host(prob, config, d0, reference):
    """Pairwise FW for Berg / mixed penalties (src/fw.py:326-357), one
    device-backed _pfw_iteration per step; KL/KL runs fully on the device."""
    from .duality import dual_feasibility_violation, lambda_star

    store = AtomStore(d0.f[None, :], d0.g[None, :], np.array([1.0]))
    trace = {k: [] for k in ("h0", "fw_gap", "pd_gap", "wall_ns")}
    err_f = []
    converged = False
    plan, primal, dual = None, np.nan, np.nan
    for _ in range(config.max_iters):
        tic = time.perf_counter_ns()
        store, diag = _pfw_iteration(prob, store)
        plan, dual, primal = diag["plan"], diag["dual"], diag["primal"]
        pd_gap = primal - dual
        trace["h0"].append(dual)
        trace["fw_gap"].append(diag["fw_gap"])
        trace["pd_gap"].append(pd_gap)
        trace["wall_ns"].append(time.perf_counter_ns() - tic)
        if reference is not None:
            pair = diag["pair"]
            err_f.append(float(np.abs(pair.f + lambda_star(prob, pair) - reference.f).max()))
        if pd_gap < config.gap_tol:
            converged = True
            break
    d = store.current()
    lam = lambda_star(prob, d)  # _finalize (:235-252)
    cert = assemble_certificate(primal, dual, dual_feasibility_violation(prob, d), config.gap_tol)
    out = {k: np.asarray(v) for k, v in trace.items()}
    out["wall_ns"] = out["wall_ns"].astype(np.int64)
    if reference is not None:
        out["err_f"] = np.asarray(err_f)
    return SolverReport(final=DualPair(d.f + lam, d.g - lam), iterations=len(out["h0"]),
                        converged=converged, trace=out, certificate=cert, plan=plan)
