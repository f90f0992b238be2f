"""Generate the BASELINE-scale fixtures (cfg3, cfg4, cfg5) from the fp64 ORACLE.

TEST INFRASTRUCTURE.  The reference cannot run these sizes (cfg3 would need a
32 GiB dense cost plus N x M temporaries, src/entropies.py:87-91; cfg5's
_finalize overflows, src/barycenter.py:417), so, as SURVEY.md §8c prescribes,
the fixtures come from the oracle restatement, which tests/test_oracle_golden.py
pins to the reference's own outputs at sizes the reference can run.  Inputs are
NOT stored: the tests regenerate them from the seeded generators in
paper_2201_00730_b200/synthetic.py; only the oracle's outputs are committed.

    python tests/golden/make_scale.py cfg3      # ~1 h on one core
    python tests/golden/make_scale.py cfg4      # a few minutes
    python tests/golden/make_scale.py cfg5      # a few minutes

cfg3 and cfg4 use oracle/csrc/scale.c (the softmin of oracle.c with SIMD
lanes; only the summation order differs), compiled here by
``oracle/Makefile scale``.  cfg5 runs oracle.fw_barycenter_fixed (the
reference loop body, barycenter.py:361-411) and records the line-search step
sizes gamma_t so the device can replay them (tests/test_scale_gpu.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2201_00730_b200 import synthetic as S  # noqa: E402

_SCALE = None


def scale_lib():
    global _SCALE
    if _SCALE is None:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "scale"], check=True)
        L = ctypes.CDLL(os.path.join(ROOT, "oracle", "_oracle_scale.so"))
        dp = ctypes.POINTER(ctypes.c_double)
        L.scale_smin_sq.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, dp, dp,
                                    ctypes.c_double, dp]
        L.scale_smin_sq.restype = None
        _SCALE = L
    return _SCALE


class FastPointCost:
    """Squared-Euclidean point-cloud cost with the vectorised softmin
    (same interface as oracle.PointCost)."""

    def __init__(self, x, y):
        self.x = np.ascontiguousarray(x, dtype=np.float64)
        self.y = np.ascontiguousarray(y, dtype=np.float64)
        self.xt = np.ascontiguousarray(self.x.T)
        self.yt = np.ascontiguousarray(self.y.T)
        self.n, self.d = self.x.shape
        self.m = self.y.shape[0]

    def _run(self, rt, o, nred, nout, pot, w, eps):
        out = np.empty(nout)
        scale_lib().scale_smin_sq(nred, nout, self.d, O._dp(rt), O._dp(o),
                                  O._dp(O._c64(pot)), O._dp(O._c64(w)), eps, O._dp(out))
        return out

    def smin_cols(self, f, eps, aw):
        return self._run(self.xt, self.y, self.n, self.m, f, aw, eps)

    def smin_rows(self, g, eps, bw):
        return self._run(self.yt, self.x, self.m, self.n, g, bw, eps)


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


def h_run(cost, a, b, eps, rho, iters, keep=()):
    """sinkhorn.py:246-315 with the early exit removed: exactly ``iters``
    H steps (oracle.h_sinkhorn_step = sinkhorn.py:137-163) from zeros."""
    f, g = np.zeros(cost.n), np.zeros(cost.m)
    delta = np.empty(iters)
    snaps = {}
    t0 = time.time()
    for t in range(iters):
        fn, gn = O.h_sinkhorn_step(cost, a, b, f, g, eps, rho, rho)
        delta[t] = float(np.abs(fn - f).max())
        f, g = fn, gn
        if t + 1 in keep:
            snaps[t + 1] = (f.copy(), g.copy())
        if t % 10 == 0:
            print(f"  it {t + 1}/{iters} delta {delta[t]:.3e} ({time.time() - t0:.0f}s)",
                  flush=True)
    return f, g, delta, snaps


def dual_h(cost, a, b, f, g, eps, rho):
    """eval_H (duality.py:256-290) with the eps term (:124-132)."""
    return O.eval_h_kl(a, b, f, g, rho, rho, eps,
                       smin_fn=lambda ff, e: cost.smin_cols(ff, e, a))


def gen_cfg3(iters=200):
    c = S.cfg3_inputs()
    cost = FastPointCost(c.x, c.y)
    f, g, delta, snaps = h_run(cost, c.alpha, c.beta, c.eps, c.rho, iters, keep=(1,))
    out = dict(eps=c.eps, rho=c.rho, iters=iters, f=f, g=g, delta=delta,
               lam=O.lambda_star_kl(c.alpha, c.beta, f, g, c.rho, c.rho),
               dual=dual_h(cost, c.alpha, c.beta, f, g, c.eps, c.rho))
    for t, (ft, gt) in snaps.items():
        out[f"f{t}"], out[f"g{t}"] = ft, gt
    save("cfg3_full.npz", **out)


def gen_cfg4(iters=300, problems=(0, 1)):
    out = {"iters": iters, "eps": S.CFG4_EPS, "rho": S.CFG4_RHO,
           "problems": np.array(problems)}
    for p in problems:
        x, y, a, b = S.cfg4_batch(start=p, count=1)
        cost = FastPointCost(x[0], y[0])
        f, g, delta, _ = h_run(cost, a[0], b[0], S.CFG4_EPS, S.CFG4_RHO, iters)
        out[f"p{p}_f"], out[f"p{p}_g"], out[f"p{p}_delta"] = f, g, delta
        out[f"p{p}_lam"] = O.lambda_star_kl(a[0], b[0], f, g, S.CFG4_RHO, S.CFG4_RHO)
        out[f"p{p}_dual"] = dual_h(cost, a[0], b[0], f, g, S.CFG4_EPS, S.CFG4_RHO)
    save("cfg4_full.npz", **out)


def gen_cfg5(iters=200, problems=(0, 1)):
    out = {"iters": iters, "problems": np.array(problems)}
    for p in problems:
        x, w = S.cfg5_batch(start=p, count=1)
        k = x.shape[1]
        om = np.full(k, 1.0 / k)
        for step in ("harmonic", "linesearch"):
            t0 = time.time()
            r = O.fw_barycenter_fixed(list(x[0]), list(w[0]), om, 1.0, iters, step=step)
            tag = f"p{p}_{step[0]}"
            pots = np.stack(r["pots"])  # translated by the final lambda (barycenter.py:413-414)
            # every 8th atom of every list (fixture size) + per-list sums of all atoms
            out[f"{tag}_pots8"] = pots[:, ::8].copy()
            out[f"{tag}_potsum"] = pots.sum(axis=1)
            for key in ("h0", "fw_gap", "pd_gap", "gamma", "nnz", "supp_hash"):
                out[f"{tag}_{key}"] = r[key]
            print(f"  cfg5 problem {p} {step}: {time.time() - t0:.0f}s", flush=True)
    save("cfg5_full.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg5", "cfg4", "cfg3"]
    for name in which:
        t0 = time.time()
        print(f"{name} ...", flush=True)
        globals()[f"gen_{name}"]()
        print(f"{name} done in {time.time() - t0:.0f}s", flush=True)
