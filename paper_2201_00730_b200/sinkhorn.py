"""F- and H-Sinkhorn on the B200 (mirror of src/sinkhorn.py:59-163, :246-315).

``run(prob, config, init, reference)`` keeps the reference signature and
report; the iterations execute in the fused sm_100a kernels of
``csrc/sinkhorn.cu`` through ``uot_sinkhorn_run``.  ``sinkhorn_batched`` is
the new batched / point-cloud entry point (BASELINE configs 3 and 4).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from .duality import DualPair, UotProblem, kl_scalars
from .entropies import KL, Berg, ent_code, ent_rho, require_kl

_ENT_NAME = {0: "kl", 1: "berg", 2: "balanced"}


def _ents(prob):
    return _ENT_NAME[ent_code(prob.ent1)], _ENT_NAME[ent_code(prob.ent2)]
from .exceptions import UnsupportedEntropyError
from .measures import ExplicitMatrix, PowerDistance, SqEuclideanPoints, check_submodular  # noqa: F401


@dataclass(frozen=True)
class AndersonConfig:
    """Anderson window depth and ridge (src/sinkhorn.py:45-56); the window
    lives on the device (csrc/anderson.cu), depth <= 32 there."""

    depth: int = 4
    reg: float = 1e-7

    def __post_init__(self):
        if self.depth < 1:
            raise ValueError("depth must be at least 1")
        if self.reg < 0:
            raise ValueError("regularization must be nonnegative")


@dataclass(frozen=True)
class SinkhornConfig:
    """variant in {"f", "g", "h"}, iteration budget, delta_f tolerance.

    ``precision`` is new: "fp64" (default, the reference's arithmetic) or
    "fp32" (log2-domain MUFU kernels; tolerance 1e-4 * eps on potentials)."""

    variant: str = "f"
    max_iters: int = 100_000
    tol: float = 1e-9
    anderson: AndersonConfig | None = None
    precision: str = "fp64"

    def __post_init__(self):
        if self.variant not in ("f", "g", "h"):
            raise ValueError("variant must be one of 'f', 'g', 'h'")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be positive")
        if self.precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")


@dataclass
class SolverReport:
    """Outcome of an iterative run plus its per-iteration trace."""

    final: DualPair
    iterations: int
    converged: bool
    trace: dict = field(default_factory=dict)
    certificate: object = None
    plan: object = None


def _geometry(prob):
    """(cost kind, d, p, x, y, C) of a problem for the kernels."""
    cost = prob.cost
    if isinstance(cost, PowerDistance):
        return _lib.COST_POWER, 1, float(cost.p), prob.alpha.points, prob.beta.points, None
    if isinstance(cost, ExplicitMatrix):
        if cost.matrix.shape != (len(prob.alpha), len(prob.beta)):
            raise ValueError(f"explicit cost shape {cost.matrix.shape} does not match supports "
                             f"({len(prob.alpha)}, {len(prob.beta)})")
        return (_lib.COST_EXPLICIT, 1, 2.0, prob.alpha.points, prob.beta.points, cost.matrix)
    if isinstance(cost, SqEuclideanPoints):
        if cost.X.shape[0] != len(prob.alpha) or cost.Y.shape[0] != len(prob.beta):
            raise ValueError("point clouds do not match the measures")
        return _lib.COST_SQEUCLID, cost.d, 2.0, cost.X, cost.Y, None
    raise TypeError(f"unknown cost specification {cost!r}")


def sinkhorn_batched(x, y, a, b, eps, rho1, rho2, iters, variant="h", cost="sqeuclid", p=2.0,
                     c=None, f0=None, tol=None, precision="fp32", stream=None, comm=None,
                     nranks=1, rank=0, shard_rows=None, g0=None, ent1="kl", ent2="kl",
                     lam0=None, ws=None, warm_shifts=False):
    """Batched Sinkhorn on device.

    x [B, N, d], y [B, M, d] (or [B, N] / [B, M] for 1-D costs), a [B, N],
    b [B, M]; ``cost`` in {"sqeuclid", "power", "explicit"} (explicit needs
    c [B, N, M]).  Returns (f [B, N], g [B, M], delta [B, iters] fp64,
    iterations [B] int32) as device tensors; f and g are in ``precision``.

    Row sharding (one problem): with ``comm`` (a handle from
    ``distributed.NcclComm``) the x / a / f0 given are this rank's rows and
    the returned f is this rank's slice; with ``comm=None, nranks > 1`` and
    ``shard_rows`` the same protocol runs for all shards in this process.
    Variant "g" (src/sinkhorn.py:117-134) starts from lambda*(f0, g0) and
    returns the overparameterised pair (plain potentials (f + lam, g - lam)).
    ``ent1`` / ``ent2`` in {"kl", "berg", "balanced"} select the marginal
    penalties (rho1 / rho2 are their strengths; "h" needs KL/KL).
    ``ws`` (a one-element list holding the workspace tensor, filled on first
    use) and ``warm_shifts`` continue a run chunk by chunk: the stale
    log-sum-exp shifts of the previous call on the same workspace seed this
    one.
    """
    t = D.torch()
    lib = _lib.load()
    dt = t.float32 if precision == "fp32" else t.float64
    kind = {"sqeuclid": _lib.COST_SQEUCLID, "power": _lib.COST_POWER,
            "explicit": _lib.COST_EXPLICIT}[cost]
    a = D.to_dev(a, dt)
    b = D.to_dev(b, dt)
    if a.ndim == 1:
        a, b = a.unsqueeze(0), b.unsqueeze(0)
    B, n = a.shape
    m = b.shape[1]
    x = D.to_dev(x, dt).reshape(B, n, -1)
    y = D.to_dev(y, dt).reshape(B, m, -1)
    d = x.shape[2]
    cm = ct = None
    if kind == _lib.COST_EXPLICIT:
        cm = D.to_dev(c, dt).reshape(B, n, m)
        ct = cm.transpose(1, 2).contiguous()
    f = D.empty((B, n), dt)
    g = D.empty((B, m), dt)
    if f0 is not None:
        f.copy_(D.to_dev(f0, dt).reshape(B, n))
        if variant == "g":
            if g0 is None:
                g.zero_()
            else:
                g.copy_(D.to_dev(g0, dt).reshape(B, m))
    if variant not in ("f", "g", "h"):
        raise ValueError("variant must be one of 'f', 'g', 'h'")
    trace = D.empty((B, iters), t.float64)
    its = D.empty((B,), t.int32)
    desc = _lib.SinkhornDesc(
        variant={"h": _lib.SINKHORN_H, "f": _lib.SINKHORN_F, "g": _lib.SINKHORN_G}[variant],
        dtype=_lib.F32 if dt == t.float32 else _lib.F64, cost=kind, batch=B, n=n, m=m,
        d=1 if kind != _lib.COST_SQEUCLID else d, p=float(p), eps=float(eps),
        rho1=float(rho1), rho2=float(rho2), x=_lib.ptr(x), y=_lib.ptr(y), c=_lib.ptr(cm),
        ct=_lib.ptr(ct), a=_lib.ptr(a), b=_lib.ptr(b), f=_lib.ptr(f), g=_lib.ptr(g),
        init_given=1 if f0 is not None else 0, iters=int(iters),
        tol=float(tol) if tol is not None else 0.0, use_tol=1 if tol is not None else 0,
        trace_delta=_lib.ptr(trace), iterations=_lib.ptr(its), nccl_comm=comm,
        nranks=int(nranks), rank=int(rank), shard_rows=None,
        ent1={"kl": _lib.ENT_KL, "berg": _lib.ENT_BERG, "balanced": _lib.ENT_BALANCED}[ent1],
        ent2={"kl": _lib.ENT_KL, "berg": _lib.ENT_BERG, "balanced": _lib.ENT_BALANCED}[ent2],
        lam_given=0 if lam0 is None else 1, lam0=0.0 if lam0 is None else float(lam0))
    rows_arr = None
    if shard_rows is not None:
        import numpy as _np

        rows_arr = _np.ascontiguousarray(_np.asarray(shard_rows, dtype=_np.int32))
        desc.shard_rows = rows_arr.ctypes.data_as(ctypes.c_void_p)
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_sinkhorn_workspace_size(ctypes.byref(desc), ctypes.byref(size)),
               "sinkhorn workspace")
    holder = ws if ws is not None else [None]
    if holder[0] is None or holder[0].numel() < size.value:
        holder[0] = D.workspace(size.value)
        warm_shifts = False
    ws = holder[0]
    desc.warm_shifts = 1 if warm_shifts else 0
    status = None
    if variant == "g" and "berg" in (ent1, ent2):  # lambda* by Newton: NewtonError possible
        status = t.zeros((B,), dtype=t.int32, device=a.device)
        desc.status = _lib.ptr(status)
    _lib.check(lib.uot_sinkhorn_run(ctypes.byref(desc), _lib.ptr(ws), ctypes.c_size_t(size.value),
                                    _lib.stream_handle(stream)), "uot_sinkhorn_run")
    del rows_arr  # host array read during the (synchronous) enqueue only
    if status is not None:
        raise_newton_status(status)
    return f, g, trace, its


_NEWTON_MESSAGES = {  # src/duality.py:188-189, :220-229, :247
    1: "empty translation domain for Berg conjugates",
    2: "failed to bracket the optimal translation",
    3: "translation Newton did not reach the residual target",
}


def raise_newton_status(status):
    """Raise the reference's NewtonError for the first failed problem of a
    per-problem status vector (uot_sinkhorn_run / uot_translation codes)."""
    from .exceptions import NewtonError

    st = D.to_np(status, readonly=False)
    bad = np.nonzero(st)[0]
    if bad.size:
        code = int(st[bad[0]])
        raise NewtonError(_NEWTON_MESSAGES.get(code, f"translation Newton failed ({code})"))


def verify_batched(x, y, a, b, f, g, eps, rho1, rho2, cost="sqeuclid", p=2.0, c=None,
                   precision="fp64", stream=None):
    """uot_sinkhorn_verify on a batch of given pairs: returns the device
    tensor out [B, 8] (res_g, log <a x b, e^((f+g-C)/eps)>, res_f, -, lambda*,
    Smin_a(f), Smin_b(g), -) -- two on-the-fly cost passes, no N x M matrix."""
    t = D.torch()
    lib = _lib.load()
    dt = t.float32 if precision == "fp32" else t.float64
    kind = {"sqeuclid": _lib.COST_SQEUCLID, "power": _lib.COST_POWER,
            "explicit": _lib.COST_EXPLICIT}[cost]
    a = D.to_dev(a, dt)
    b = D.to_dev(b, dt)
    if a.ndim == 1:
        a, b = a.unsqueeze(0), b.unsqueeze(0)
    B, n = a.shape
    m = b.shape[1]
    x = D.to_dev(x, dt).reshape(B, n, -1)
    y = D.to_dev(y, dt).reshape(B, m, -1)
    d = x.shape[2]
    cm = ct = None
    if kind == _lib.COST_EXPLICIT:
        cm = D.to_dev(c, dt).reshape(B, n, m)
        ct = cm.transpose(1, 2).contiguous()
    fd = D.to_dev(f, dt).reshape(B, n).contiguous()
    gd = D.to_dev(g, dt).reshape(B, m).contiguous()
    out = t.zeros((B, 8), dtype=t.float64, device=fd.device)
    desc = _lib.SinkhornDesc(
        variant=_lib.SINKHORN_F, dtype=_lib.F32 if dt == t.float32 else _lib.F64, cost=kind,
        batch=B, n=n, m=m, d=1 if kind != _lib.COST_SQEUCLID else d, p=float(p), eps=float(eps),
        rho1=float(rho1), rho2=float(rho2), x=_lib.ptr(x), y=_lib.ptr(y), c=_lib.ptr(cm),
        ct=_lib.ptr(ct), a=_lib.ptr(a), b=_lib.ptr(b), f=_lib.ptr(fd), g=_lib.ptr(gd),
        init_given=1, iters=1, tol=0.0, use_tol=0, trace_delta=None, iterations=None,
        nccl_comm=None, nranks=1, rank=0, shard_rows=None)
    size = ctypes.c_size_t(0)
    _lib.check(lib.uot_sinkhorn_workspace_size(ctypes.byref(desc), ctypes.byref(size)),
               "sinkhorn workspace")
    ws = D.workspace(size.value)
    _lib.check(lib.uot_sinkhorn_verify(ctypes.byref(desc), _lib.ptr(ws),
                                       ctypes.c_size_t(size.value), _lib.stream_handle(stream),
                                       _lib.ptr(out)), "uot_sinkhorn_verify")
    return out


def _verify_prob(prob, d):
    if prob.eps <= 0:
        raise ValueError("the entropic terms need eps > 0")
    require_kl(prob.ent1, prob.ent2, what="dual objective")
    costname, p, x, y, C = _step_inputs(prob)
    out = verify_batched(x, y, prob.alpha.weights, prob.beta.weights, d.f, d.g, prob.eps,
                         prob.ent1.rho, prob.ent2.rho, cost=costname, p=p, c=C)
    return D.to_np(out[0], readonly=False)


def h_optimality_residual(prob, d, side="f"):
    """Sup-norm stationarity residual of the invariant dual at the pair
    (src/sinkhorn.py:166-189), computed on the device without C."""
    prob.check_pair(d)
    if not (isinstance(prob.ent1, KL) and isinstance(prob.ent2, KL)):
        raise UnsupportedEntropyError("residual defined for kl penalties only")
    if side not in ("f", "g"):
        raise ValueError("side must be 'f' or 'g'")
    v = _verify_prob(prob, d)
    return float(v[2] if side == "f" else v[0])


def _require_positive_eps(prob):
    if prob.eps <= 0:
        raise ValueError("sinkhorn iterations need eps > 0")


def _step_inputs(prob):
    kind, d, p, x, y, C = _geometry(prob)
    costname = {_lib.COST_POWER: "power", _lib.COST_EXPLICIT: "explicit",
                _lib.COST_SQEUCLID: "sqeuclid"}[kind]
    return costname, p, x, y, C


def _one_step(prob, d, variant):
    _require_positive_eps(prob)
    prob.check_pair(d)
    if variant == "h":
        require_kl(prob.ent1, prob.ent2, what="h-sinkhorn")
    e1, e2 = _ents(prob)
    costname, p, x, y, C = _step_inputs(prob)
    f, g, _, _ = sinkhorn_batched(x, y, prob.alpha.weights, prob.beta.weights, prob.eps,
                                  ent_rho(prob.ent1), ent_rho(prob.ent2), 1, variant=variant,
                                  cost=costname, p=p, c=C, f0=d.f, precision="fp64", ent1=e1,
                                  ent2=e2)
    return DualPair(D.to_np(f[0]), D.to_np(g[0]))


def f_sinkhorn_step(prob, d):
    """One plain step, g then f (src/sinkhorn.py:103-114); KL, Berg or
    Balanced marginals (aprox per entropy, entropies.py:203-263)."""
    return _one_step(prob, d, "f")


def g_sinkhorn_step(prob, d, lam):
    """One translated step at the incoming translation lam
    (src/sinkhorn.py:117-134); returns (pair, new_lam) with new_lam =
    lambda_star(pair, initial=lam).  KL or Berg marginals: the device G run
    starts from the given lam (descriptor lam_given) instead of
    lambda*(f, g); the translation after the step is the closed form (KL/KL)
    or the bracketed Newton (uot_translation)."""
    from .duality import lambda_star

    _require_positive_eps(prob)
    prob.check_pair(d)
    if not all(isinstance(e, (KL, Berg)) for e in (prob.ent1, prob.ent2)):
        raise UnsupportedEntropyError(
            "optimal translation needs strictly convex conjugates (KL or Berg)")
    e1, e2 = _ents(prob)
    costname, p, x, y, C = _step_inputs(prob)
    f, g, _, _ = sinkhorn_batched(x, y, prob.alpha.weights, prob.beta.weights, prob.eps,
                                  ent_rho(prob.ent1), ent_rho(prob.ent2), 1, variant="g",
                                  cost=costname, p=p, c=C, f0=d.f, g0=d.g, precision="fp64",
                                  ent1=e1, ent2=e2, lam0=float(lam))
    pair = DualPair(D.to_np(f[0]), D.to_np(g[0]))
    return pair, lambda_star(prob, pair, initial=float(lam))


def h_sinkhorn_step(prob, d):
    """One translation-invariant step, g then f (src/sinkhorn.py:137-163)."""
    _require_positive_eps(prob)
    if not (isinstance(prob.ent1, KL) and isinstance(prob.ent2, KL)):
        raise UnsupportedEntropyError("h-sinkhorn requires kl penalties on both marginals")
    return _one_step(prob, d, "h")


def run(prob, config, init=None, reference=None):
    """Iterate the configured variant until ||f_t - f_{t-1}||_inf < tol
    (src/sinkhorn.py:246-315).  ``wall_ns`` holds the mean device time per
    iteration of each launch chunk.  With ``reference`` the iterates are
    advanced one step per launch so that err_f / err_g (translated iterates
    vs the reference pair) can be traced exactly like the reference."""
    _require_positive_eps(prob)
    n, m = len(prob.alpha), len(prob.beta)
    d = init if init is not None else DualPair.zeros(n, m)
    prob.check_pair(d)
    if config.variant == "h" and not (isinstance(prob.ent1, KL) and isinstance(prob.ent2, KL)):
        raise UnsupportedEntropyError("h-sinkhorn requires kl penalties on both marginals")
    if config.variant == "g" and not all(isinstance(e, (KL, Berg)) for e in (prob.ent1, prob.ent2)):
        raise UnsupportedEntropyError(
            "optimal translation needs strictly convex conjugates (KL or Berg)")
    e1, e2 = _ents(prob)
    if config.anderson is not None:
        return _run_anderson(prob, config, d, reference, e1, e2)
    t = D.torch()
    costname, p, x, y, C = _step_inputs(prob)
    deltas, walls, err_f, err_g = [], [], [], []
    f_cur = d.f
    g_cur = d.g
    done = 0
    converged = False
    chunk = 1 if reference is not None else 256
    ws = [None]  # filled by the first (largest) chunk, then reused: stale shifts carried
    while done < config.max_iters and not converged:
        k = min(chunk, config.max_iters - done)
        t0 = time.perf_counter_ns()
        f, g, tr, its = sinkhorn_batched(
            x, y, prob.alpha.weights, prob.beta.weights, prob.eps, ent_rho(prob.ent1),
            ent_rho(prob.ent2), k, variant=config.variant, cost=costname, p=p, c=C, f0=f_cur,
            tol=config.tol, precision=config.precision,
            g0=g_cur if config.variant == "g" else None, ent1=e1, ent2=e2, ws=ws,
            warm_shifts=done > 0)
        t.cuda.synchronize()
        el = time.perf_counter_ns() - t0
        got = int(its[0].item())
        dl = D.to_np(tr[0, :got], readonly=False)
        deltas.extend(dl.tolist())
        walls.extend([el // max(got, 1)] * got)
        f_cur = D.to_np(f[0]).astype(np.float64)
        g_cur = D.to_np(g[0]).astype(np.float64)
        done += got
        if got < k or (got > 0 and dl[-1] < config.tol):
            converged = True
        if reference is not None:
            if config.variant == "f":
                lam = 0.0
            else:  # translated iterate (sinkhorn.py:276-280): closed form or Newton
                from .duality import lambda_star

                lam = lambda_star(prob, DualPair(f_cur, g_cur))
            err_f.append(float(np.abs(f_cur + lam - reference.f).max()))
            err_g.append(float(np.abs(g_cur - lam - reference.g).max()))
    trace = {"delta_f": np.asarray(deltas), "wall_ns": np.asarray(walls, dtype=np.int64)}
    if reference is not None:
        trace["err_f"] = np.asarray(err_f)
        trace["err_g"] = np.asarray(err_g)
    return SolverReport(final=DualPair(f_cur, g_cur), iterations=len(deltas), converged=converged,
                        trace=trace)


def anderson_weights(U, r):
    """Window weights c with (U'U + r I) c proportional to 1 and sum c = 1
    (src/sinkhorn.py:197-212), computed on the device (uot_anderson_weights:
    block-reduced Gram, pivoted elimination).  Raises LinAlgError on a
    singular window like the reference."""
    U = np.asarray(U, dtype=np.float64)
    if U.ndim != 2 or U.shape[1] < 1:
        raise ValueError("U must be a matrix with at least one column")
    t = D.torch()
    lib = _lib.load()
    rows, k = U.shape
    Ud = D.to_dev(U, t.float64)
    c = D.empty((k,), t.float64)
    st = t.zeros((1,), dtype=t.int32, device=Ud.device)
    _lib.check(lib.uot_anderson_weights(rows, k, _lib.ptr(Ud), float(r), _lib.ptr(c), _lib.ptr(st),
                                        _lib.stream_handle()), "uot_anderson_weights")
    if int(st.item()) != 0:
        raise np.linalg.LinAlgError("singular or degenerate Anderson window")
    return D.to_np(c, readonly=False)


class AndersonWindow:
    """Device-resident Anderson state for ``batch`` windows over vectors of
    length ``length`` (mirror of src/sinkhorn.py:215-243 _AndersonState)."""

    def __init__(self, batch, length, depth, reg, stream=None):
        self.lib = _lib.load()
        self.batch, self.length, self.depth, self.reg = int(batch), int(length), int(depth), float(reg)
        size = ctypes.c_size_t(0)
        _lib.check(self.lib.uot_anderson_workspace_size(self.batch, self.length, self.depth,
                                                        ctypes.byref(size)), "anderson workspace")
        self.nbytes = size.value
        self.ws = D.workspace(self.nbytes)
        t = D.torch()
        self.delta = D.empty((self.batch,), t.float64)
        self.status = t.zeros((self.batch,), dtype=t.int32, device=self.ws.device)
        self.stream = stream
        _lib.check(self.lib.uot_anderson_reset(self.batch, self.length, self.depth,
                                               _lib.ptr(self.ws), self.nbytes,
                                               _lib.stream_handle(stream)), "uot_anderson_reset")

    def step(self, z, tz, znew, nf):
        """push(z, tz) + extrapolate into znew (device fp64 [batch, length]);
        returns the device tensors (delta_f [batch], status [batch])."""
        _lib.check(self.lib.uot_anderson_step(
            self.batch, self.length, int(nf), self.depth, self.reg, _lib.ptr(z), _lib.ptr(tz),
            _lib.ptr(znew), _lib.ptr(self.delta), _lib.ptr(self.status), _lib.ptr(self.ws),
            self.nbytes, _lib.stream_handle(self.stream)), "uot_anderson_step")
        return self.delta, self.status


def _run_anderson(prob, config, d, reference, e1, e2):
    """run() with ``config.anderson`` (src/sinkhorn.py:281-292): each
    iteration is one device step of the variant from the current f (and, for
    "g", the carried lambda), then the device window's push + extrapolation
    of the concatenated (f, g).  The reference's step maps read g only
    through lambda, so the extrapolated g is carried for "g" and returned."""
    t = D.torch()
    n, m = len(prob.alpha), len(prob.beta)
    from .duality import lambda_star

    variant = config.variant

    def lam_of(zz, initial=0.0):  # translation of a device (f | g) row, closed form or Newton
        return lambda_star(prob, DualPair(D.to_np(zz[:n]), D.to_np(zz[n:])), initial=initial)

    r1, r2 = ent_rho(prob.ent1), ent_rho(prob.ent2)
    aw, bw = prob.alpha.weights, prob.beta.weights
    costname, p, x, y, C = _step_inputs(prob)
    f64 = t.float64
    z = D.to_dev(np.concatenate([np.asarray(d.f, np.float64), np.asarray(d.g, np.float64)]),
                 f64).reshape(1, n + m)
    tz = t.empty_like(z)
    win = AndersonWindow(1, n + m, config.anderson.depth, config.anderson.reg)
    lam = lam_of(z[0]) if variant == "g" else 0.0
    deltas, walls, err_f, err_g = [], [], [], []
    converged = False
    for _ in range(config.max_iters):
        t0 = time.perf_counter_ns()
        gv = variant == "g"  # the device G step starts at the carried lambda (g_sinkhorn_step)
        f1, g1, _, _ = sinkhorn_batched(x, y, aw, bw, prob.eps, r1, r2, 1, variant=variant,
                                        cost=costname, p=p, c=C, f0=z[0, :n],
                                        g0=z[0, n:] if gv else None,
                                        precision=config.precision, ent1=e1, ent2=e2,
                                        lam0=lam if gv else None)
        tz[0, :n].copy_(f1[0])
        tz[0, n:].copy_(g1[0])
        if variant == "g":
            lam = lam_of(tz[0], lam)
        delta, status = win.step(z, tz, z, n)
        dl = float(delta[0].item())
        if int(status[0].item()) != 0:
            raise np.linalg.LinAlgError("singular Anderson window (anderson_weights)")
        walls.append(time.perf_counter_ns() - t0)
        deltas.append(dl)
        if reference is not None:
            shift = 0.0
            if variant != "f":
                shift = lam_of(z[0], lam)
            fz = D.to_np(z[0, :n])
            gz = D.to_np(z[0, n:])
            err_f.append(float(np.abs(fz + shift - reference.f).max()))
            err_g.append(float(np.abs(gz - shift - reference.g).max()))
        if dl < config.tol:
            converged = True
            break
    trace = {"delta_f": np.asarray(deltas), "wall_ns": np.asarray(walls, dtype=np.int64)}
    if reference is not None:
        trace["err_f"] = np.asarray(err_f)
        trace["err_g"] = np.asarray(err_g)
    final = DualPair(D.to_np(z[0, :n]).copy(), D.to_np(z[0, n:]).copy())
    return SolverReport(final=final, iterations=len(deltas), converged=converged, trace=trace)


def estimate_rate(errors):
    """Empirical contraction factor exp(median_t log(e_{t+1}/e_t))
    (src/sinkhorn.py:318-335): trailing entries below 1e-13 (noise floor) are
    dropped first; fewer than two usable ratios raise ValueError.  Host
    statistic over a trace the device produced."""
    e = np.asarray(errors, dtype=np.float64)
    if e.ndim != 1 or e.size < 3:
        raise ValueError("need at least three error values")
    if (e <= 0).any():
        raise ValueError("errors must be strictly positive")
    keep = e.size
    while keep > 0 and e[keep - 1] < 1e-13:
        keep -= 1
    if keep < 3:
        raise ValueError("fewer than 2 usable ratios after truncation")
    return float(np.exp(np.median(np.diff(np.log(e[:keep])))))


def write_trace_csv(report, path_or_buf):
    """``iter,delta_f,err_f,err_g,wall_ns`` rows (src/sinkhorn.py:349-373)."""
    from .formats import write_trace_csv as _w

    _w(report, path_or_buf)


def birkhoff_rate_bound(prob):
    """tanh(D / (4 eps)) with D the cost's quadruple diameter
    (src/sinkhorn.py:338-346): the contraction bound of the softmin in the
    Hilbert seminorm; D computed on the device."""
    from .measures import build_cost_matrix, cost_quadruple_diameter

    _require_positive_eps(prob)
    if isinstance(prob.cost, PowerDistance):
        C = build_cost_matrix(prob.alpha, prob.beta, prob.cost)
    elif isinstance(prob.cost, ExplicitMatrix):
        C = prob.cost.matrix
    else:
        raise UnsupportedEntropyError("birkhoff_rate_bound needs a 1-D or explicit cost")
    return float(np.tanh(cost_quadruple_diameter(C) / (4.0 * prob.eps)))
