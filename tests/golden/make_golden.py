"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``uotkit`` read-only from /root/reference/pkg/src and drives the
reference's own step / oracle functions with fixed iteration counts (the
reference's ``run``/``fw_solve``/``fw_barycenter`` exit early once a gap or
delta tolerance is met -- sinkhorn.py:304-306, fw.py:220-222,
barycenter.py:394-396 -- so the loops below call the step functions
directly, as SURVEY.md §8c prescribes).  The fixtures are small .npz files
(no pickles); tests/test_oracle_golden.py pins the oracle against them and
the GPU parity tests compare the CUDA path against them.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import uotkit as U  # noqa: E402
from uotkit import barycenter as UB  # noqa: E402
from uotkit import fw as UF  # noqa: E402
from uotkit import sinkhorn as US  # noqa: E402

import oracle as O  # noqa: E402  (plan_hash only)
from paper_2201_00730_b200 import synthetic as S  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1024:.1f} KiB)")


def ref_sinkhorn(prob, variant, iters, d0=None):
    d = U.DualPair.zeros(len(prob.alpha), len(prob.beta)) if d0 is None else d0
    deltas = []
    if variant == "g":  # run(): lam = lambda_star(d0), then g_sinkhorn_step (:263-271)
        lam = U.lambda_star(prob, d)
        for _ in range(iters):
            new, lam = US.g_sinkhorn_step(prob, d, lam)
            deltas.append(float(np.abs(new.f - d.f).max()))
            d = new
        return d.f, d.g, np.asarray(deltas)
    step = US.h_sinkhorn_step if variant == "h" else US.f_sinkhorn_step
    for _ in range(iters):
        new = step(prob, d)
        deltas.append(float(np.abs(new.f - d.f).max()))
        d = new
    return d.f, d.g, np.asarray(deltas)


def gen_sinkhorn_ent():
    """F and G steps with Berg / Balanced penalties (entropies.py:203-263,
    duality.py:182-247), small 1-D problems."""
    rng = np.random.default_rng(53)
    out = {}
    combos = [("f", "berg", "berg"), ("f", "kl", "berg"), ("f", "berg", "balanced"),
              ("f", "balanced", "kl"), ("g", "berg", "kl"), ("g", "berg", "berg"),
              ("g", "kl", "berg"), ("f", "berg", "berg")]
    names = {"kl": U.KL, "berg": U.Berg}
    for k, (var, e1, e2) in enumerate(combos):
        n, m = int(rng.integers(3, 30)), int(rng.integers(3, 30))
        p = [1.0, 2.0][k % 2]
        eps = [0.1, 0.5][k % 2]
        r1, r2 = float(rng.uniform(0.5, 2.0)), float(rng.uniform(0.5, 2.0))
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        wa = rng.uniform(0.1, 1.0, n)
        wb = rng.uniform(0.1, 1.0, m)
        if "balanced" in (e1, e2):
            wb *= wa.sum() / wb.sum()
        ent = [names[e](r) if e != "balanced" else U.Balanced() for e, r in ((e1, r1), (e2, r2))]
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(p), ent[0], ent[1], eps=eps)
        f, g, dl = ref_sinkhorn(prob, var, 25)
        out[f"c{k}_f"], out[f"c{k}_g"], out[f"c{k}_delta"] = f, g, dl
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_par"] = np.array([p, eps, r1, r2, 25])
        out[f"c{k}_spec"] = np.array([var, e1, e2])
    out["cases"] = np.arange(len(combos))
    save("sinkhorn_ent.npz", **out)


def gen_sinkhorn_g():
    """G-Sinkhorn (sinkhorn.py:117-134) on small 1-D problems, from zeros and
    from a nonzero initial pair, plus the cfg1 setting."""
    rng = np.random.default_rng(41)
    out = {}
    cases = []
    for k in range(8):
        n, m = int(rng.integers(3, 40)), int(rng.integers(3, 40))
        p = [1.0, 2.0, 1.5][k % 3]
        eps = [0.05, 0.5, 0.2][k % 3]
        r1, r2 = float(rng.uniform(0.3, 2.0)), float(rng.uniform(0.3, 2.0))
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        wa = rng.uniform(0.1, 1.0, n)
        wb = rng.uniform(0.1, 1.0, m) * 1.7
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(p), U.KL(r1), U.KL(r2), eps=eps)
        f0 = g0 = None
        if k % 2 == 1:  # feasible nonzero start: half the row / column minima
            C = np.abs(x[:, None] - y[None, :]) ** p
            f0, g0 = 0.5 * C.min(axis=1) + 0.1, 0.5 * C.min(axis=0) - 0.1
        d0 = None if f0 is None else U.DualPair(f0, g0)
        f, g, dl = ref_sinkhorn(prob, "g", 40, d0)
        out[f"c{k}_f"], out[f"c{k}_g"], out[f"c{k}_delta"] = f, g, dl
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_f0"] = np.zeros(n) if f0 is None else f0
        out[f"c{k}_g0"] = np.zeros(m) if g0 is None else g0
        out[f"c{k}_par"] = np.array([p, eps, r1, r2, 40, 0.0 if f0 is None else 1.0])
        cases.append(k)
    c = S.cfg1_inputs()
    prob = U.UotProblem(U.DiscreteMeasure(c.x, c.alpha), U.DiscreteMeasure(c.y, c.beta),
                        U.PowerDistance(2.0), U.KL(c.rho), U.KL(c.rho), eps=c.eps)
    f, g, dl = ref_sinkhorn(prob, "g", c.iters)
    k = 8
    out[f"c{k}_f"], out[f"c{k}_g"], out[f"c{k}_delta"] = f, g, dl
    out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = c.x, c.y, c.alpha, c.beta
    out[f"c{k}_f0"], out[f"c{k}_g0"] = np.zeros(len(c.x)), np.zeros(len(c.y))
    out[f"c{k}_par"] = np.array([2.0, c.eps, c.rho, c.rho, c.iters, 0.0])
    cases.append(k)
    out["cases"] = np.array(cases)
    save("sinkhorn_g.npz", **out)


def gen_cfg1():
    c = S.cfg1_inputs()
    a = U.DiscreteMeasure(c.x, c.alpha)
    b = U.DiscreteMeasure(c.y, c.beta)
    prob = U.UotProblem(a, b, U.PowerDistance(2.0), U.KL(c.rho), U.KL(c.rho), eps=c.eps)
    out = dict(x=c.x, y=c.y, alpha=c.alpha, beta=c.beta, eps=c.eps, rho=c.rho)
    for v in ("h", "f"):
        f, g, dl = ref_sinkhorn(prob, v, c.iters)
        out[f"{v}_f"], out[f"{v}_g"], out[f"{v}_delta"] = f, g, dl
        lam = U.lambda_star(prob, U.DualPair(f, g))
        out[f"{v}_lam"] = lam
        out[f"{v}_dual"] = U.eval_H(prob, U.DualPair(f, g))
    save("cfg1.npz", **out)


def gen_sinkhorn_small():
    rng = np.random.default_rng(7)
    out = {}
    cases = []
    for k in range(12):
        n, m = int(rng.integers(3, 40)), int(rng.integers(3, 40))
        p = [1.0, 2.0, 1.5][k % 3]
        eps = [0.05, 0.5, 0.2][k % 3]
        r1, r2 = float(rng.uniform(0.3, 2.0)), float(rng.uniform(0.3, 2.0))
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        wa = rng.uniform(0.1, 1.0, n)
        wb = rng.uniform(0.1, 1.0, m) * 1.7
        if k % 4 == 3:  # zero-weight atoms are masked out of every reduction
            wa[rng.integers(0, n)] = 0.0
            wb[rng.integers(0, m)] = 0.0
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(p), U.KL(r1), U.KL(r2), eps=eps)
        iters = 40
        for v in ("h", "f"):
            f, g, dl = ref_sinkhorn(prob, v, iters)
            out[f"c{k}_{v}_f"], out[f"c{k}_{v}_g"], out[f"c{k}_{v}_delta"] = f, g, dl
            out[f"c{k}_{v}_dual"] = U.eval_H(prob, U.DualPair(f, g))
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_par"] = np.array([p, eps, r1, r2, iters])
        cases.append(k)
    out["cases"] = np.array(cases)
    save("sinkhorn_small.npz", **out)


def gen_points_sinkhorn(name, x, y, wa, wb, eps, rho, iters):
    C = ((x[:, None, :] - y[None, :, :]) ** 2).sum(axis=2)
    n, m = len(x), len(y)
    prob = U.UotProblem(U.DiscreteMeasure(np.arange(n, dtype=float), wa),
                        U.DiscreteMeasure(np.arange(m, dtype=float), wb),
                        U.ExplicitMatrix(C), U.KL(rho), U.KL(rho), eps=eps)
    t0 = time.time()
    f, g, dl = ref_sinkhorn(prob, "h", iters)
    dual = U.eval_H(prob, U.DualPair(f, g))
    print(f"  {name}: reference H-sinkhorn {n}x{m} x{iters} in {time.time() - t0:.1f}s")
    save(name, x=x, y=y, alpha=wa, beta=wb, eps=eps, rho=rho, iters=iters, f=f, g=g,
         delta=dl, dual=dual)


def gen_cfg3_small():
    c = S.cfg3_inputs(n=384, seed=2023)
    gen_points_sinkhorn("cfg3_small.npz", c.x, c.y, c.alpha, c.beta, c.eps, c.rho, c.iters)


def gen_cfg4_small():
    x, y, a, b = S.cfg4_batch(batch=2, n=256, m=256, d=64)
    gen_points_sinkhorn("cfg4_small.npz", x[0], y[0], a[0], b[0], S.CFG4_EPS, S.CFG4_RHO, 300)


def gen_ot1d():
    rng = np.random.default_rng(11)
    out = {}
    cases = []

    def add(k, x, y, wa, wb, p):
        a = U.DiscreteMeasure(x, wa)
        b = U.DiscreteMeasure(y, wb)
        plan, d = U.solve_ot_1d(a, b, U.PowerDistance(p))
        out[f"c{k}_x"], out[f"c{k}_y"] = a.points, b.points
        out[f"c{k}_a"], out[f"c{k}_b"] = a.weights, b.weights
        out[f"c{k}_p"] = np.array(p)
        out[f"c{k}_i"], out[f"c{k}_j"], out[f"c{k}_m"] = plan.source_idx, plan.target_idx, plan.mass
        out[f"c{k}_f"], out[f"c{k}_g"] = d.f, d.g
        cases.append(k)

    # reference known-answer cases: tests/test_ot1d.py:32-38, :47-58, :71-76
    add(0, [0.0], [1.0], [1.0], [1.0], 1.0)
    add(1, [0.0, 1.0], [0.0, 1.0], [0.7, 0.3], [0.4, 0.6], 1.0)
    add(2, [0.0, 0.5, 1.0], [0.2, 0.9], [0.5, 0.0, 0.5], [0.6, 0.4], 2.0)
    k = 3
    for _ in range(60):  # tests/test_ot1d.py:60-69 style, zero weights allowed
        n, m = rng.integers(1, 51, 2)
        p = float(rng.choice([1.0, 2.0]))
        wa = rng.uniform(0.0, 1.0, n)
        wb = rng.uniform(0.0, 1.0, m)
        wb *= wa.sum() / wb.sum()
        add(k, np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m)), wa, wb, p)
        k += 1
    for n, m in ((1024, 1024), (1000, 777), (4096, 4096)):  # cfg2-scale sweeps
        wa = rng.exponential(1.0, n)
        wb = rng.exponential(1.0, m)
        wb *= wa.sum() / wb.sum()
        add(k, np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m)), wa, wb, 2.0)
        k += 1
    out["cases"] = np.array(cases)
    save("ot1d.npz", **out)


def ref_fw(prob, iters, step):
    """fw.py:176-232 loop body with the early exit removed."""
    d = UF._default_init(prob)
    tr = {k: [] for k in ("h0", "fw_gap", "pd_gap")}
    plan = None
    for t in range(iters):
        ta, tb, plan, atom, fw_gap = UF._lmo(prob, d)
        dual = UF._h0(prob, d.f, d.g)
        primal = U.eval_primal(prob, plan)
        tr["h0"].append(dual)
        tr["fw_gap"].append(fw_gap)
        tr["pd_gap"].append(primal - dual)
        gamma = 2.0 / (2.0 + t) if step == "harmonic" else UF.line_search_h0(prob, d, atom)
        d = U.DualPair((1.0 - gamma) * d.f + gamma * atom.f, (1.0 - gamma) * d.g + gamma * atom.g)
    lam = U.lambda_star(prob, d)
    return d, lam, plan, {k: np.asarray(v) for k, v in tr.items()}


def gen_fw():
    out = {}
    cases = []
    rng = np.random.default_rng(13)
    specs = []
    for k in range(6):  # small random problems, both step rules
        n, m = int(rng.integers(20, 70)), int(rng.integers(20, 70))
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        wa = rng.exponential(1.0, n)
        wa *= rng.uniform(0.5, 2.0) / wa.sum()
        wb = rng.exponential(1.0, m)
        wb *= rng.uniform(0.5, 2.0) / wb.sum()
        r1, r2 = float(rng.uniform(0.3, 2.0)), float(rng.uniform(0.3, 2.0))
        p = [2.0, 1.0][k % 2]
        specs.append((x, y, wa, wb, r1, r2, p, 120, ["linesearch", "harmonic"][k % 2]))
    x2, y2, a2, b2 = S.cfg2_batch(count=3)
    for q in range(3):  # the first problems of the seeded cfg2 batch, full shape
        specs.append((x2[q], y2[q], a2[q], b2[q], 1.0, 1.0, 2.0, 500,
                      "harmonic" if q == 2 else "linesearch"))
    for k, (x, y, wa, wb, r1, r2, p, iters, step) in enumerate(specs):
        t0 = time.time()
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(p), U.KL(r1), U.KL(r2), eps=0.0)
        d, lam, plan, tr = ref_fw(prob, iters, step)
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_par"] = np.array([r1, r2, p, iters, 1.0 if step == "linesearch" else 0.0])
        out[f"c{k}_f_raw"], out[f"c{k}_g_raw"] = d.f, d.g
        out[f"c{k}_f"], out[f"c{k}_g"] = d.f + lam, d.g - lam
        out[f"c{k}_i"], out[f"c{k}_j"], out[f"c{k}_m"] = plan.source_idx, plan.target_idx, plan.mass
        for kk, v in tr.items():
            out[f"c{k}_{kk}"] = v
        cases.append(k)
        print(f"  fw case {k}: {len(x)}x{len(y)} {step} x{iters} in {time.time() - t0:.1f}s")
    out["cases"] = np.array(cases)
    save("fw.npz", **out)


def ref_pfw(prob, iters):
    """fw.py:326-357 (_pfw_solve) loop body with the early exit removed; the
    step size is read back from the weight transfer."""
    d0 = UF._default_init(prob)
    store = UF.AtomStore(d0.f[None, :], d0.g[None, :], np.array([1.0]))
    tr = {k: [] for k in ("h0", "fw_gap", "pd_gap", "natoms")}
    plan = None
    for _ in range(iters):
        store, diag = UF._pfw_iteration(prob, store)
        plan = diag["plan"]
        tr["h0"].append(diag["dual"])
        tr["fw_gap"].append(diag["fw_gap"])
        tr["pd_gap"].append(diag["primal"] - diag["dual"])
        tr["natoms"].append(store.weights.size)
    d = store.current()
    lam = U.lambda_star(prob, d)
    return d, lam, plan, {k: np.asarray(v) for k, v in tr.items()}


def gen_pfw():
    out = {}
    cases = []
    rng = np.random.default_rng(29)
    specs = []
    for k in range(5):  # small random problems
        n, m = int(rng.integers(20, 70)), int(rng.integers(20, 70))
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        wa = rng.exponential(1.0, n)
        wa *= rng.uniform(0.5, 2.0) / wa.sum()
        wb = rng.exponential(1.0, m)
        wb *= rng.uniform(0.5, 2.0) / wb.sum()
        r1, r2 = float(rng.uniform(0.3, 2.0)), float(rng.uniform(0.3, 2.0))
        p = [2.0, 1.0][k % 2]
        specs.append((x, y, wa, wb, r1, r2, p, 80))
    x2, y2, a2, b2 = S.cfg2_batch(count=1)
    specs.append((x2[0], y2[0], a2[0], b2[0], 1.0, 1.0, 2.0, 150))  # cfg2 shape
    for k, (x, y, wa, wb, r1, r2, p, iters) in enumerate(specs):
        t0 = time.time()
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(p), U.KL(r1), U.KL(r2), eps=0.0)
        d, lam, plan, tr = ref_pfw(prob, iters)
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_par"] = np.array([r1, r2, p, iters])
        out[f"c{k}_f_raw"], out[f"c{k}_g_raw"] = d.f, d.g
        out[f"c{k}_f"], out[f"c{k}_g"] = d.f + lam, d.g - lam
        out[f"c{k}_i"], out[f"c{k}_j"], out[f"c{k}_m"] = plan.source_idx, plan.target_idx, plan.mass
        for kk, v in tr.items():
            out[f"c{k}_{kk}"] = v
        cases.append(k)
        print(f"  pfw case {k}: {len(x)}x{len(y)} x{iters} atoms {tr['natoms'][-1]} "
              f"in {time.time() - t0:.1f}s")
    out["cases"] = np.array(cases)
    save("pfw.npz", **out)


def gen_mot():
    rng = np.random.default_rng(17)
    out = {}
    cases = []

    def add(k, inputs, w):
        plan, duals = U.solve_mot_1d(inputs, w)
        kk = len(inputs)
        out[f"c{k}_k"] = np.array(kk)
        out[f"c{k}_w"] = np.asarray(w, dtype=float)
        for q, mq in enumerate(inputs):
            out[f"c{k}_x{q}"], out[f"c{k}_a{q}"] = mq.points, mq.weights
            out[f"c{k}_f{q}"] = duals.potentials[q]
        out[f"c{k}_idx"], out[f"c{k}_m"] = plan.indices, plan.mass
        cases.append(k)

    # tests/test_barycenter.py:58-66 (single atoms) and :95-105 (zero weights)
    add(0, [U.DiscreteMeasure([float(q)], [1.0]) for q in range(3)], np.full(3, 1 / 3))
    add(1, [U.DiscreteMeasure([0.0, 0.4, 1.0], [0.5, 0.0, 0.5]),
            U.DiscreteMeasure([0.1, 0.9], [0.6, 0.4]),
            U.DiscreteMeasure([0.2, 0.8], [0.3, 0.7])], np.full(3, 1 / 3))
    k = 2
    for _ in range(40):  # random families, K in 2..5, ragged sizes
        kk = int(rng.integers(2, 6))
        inputs = []
        for _q in range(kk):
            n = int(rng.integers(2, 30))
            wq = rng.uniform(0.1, 1.0, n)
            wq *= 1.3 / wq.sum()
            inputs.append(U.DiscreteMeasure(np.sort(rng.uniform(0, 1, n)), wq))
        w = rng.uniform(0.2, 1.0, kk)
        w /= w.sum()
        add(k, inputs, w)
        k += 1
    # one cfg5-shaped family (K = 16) at reduced N
    xs, ws = S.cfg5_batch(count=1, n=256)
    inputs = [U.DiscreteMeasure(xs[0, q], ws[0, q] * (1.0 / ws[0, q].sum())) for q in range(16)]
    add(k, inputs, np.full(16, 1 / 16))
    out["cases"] = np.array(cases + [k])
    save("mot.npz", **out)


def gen_mot_cert():
    """mot_certificate (barycenter.py:261-295) of every mot.npz solution, and
    of a perturbed dual (failing certificate) for each case."""
    z = np.load(os.path.join(HERE, "mot.npz"))
    out = {}
    done = []
    for k in z["cases"]:
        kk = int(z[f"c{k}_k"])
        if kk > 8:  # np.prod of the grid overflows int64 to 0 and the reference
            continue  # then attempts the exhaustive sweep (TiB allocation)
        inputs = [U.DiscreteMeasure(z[f"c{k}_x{q}"], z[f"c{k}_a{q}"]) for q in range(kk)]
        w = z[f"c{k}_w"]
        plan = UB.MultiPlan(z[f"c{k}_idx"], z[f"c{k}_m"])
        duals = UB.MultiDual(tuple(z[f"c{k}_f{q}"] for q in range(kk)))
        cert = UB.mot_certificate(inputs, w, plan, duals)
        out[f"c{k}_cert"] = np.array([cert.primal, cert.dual, cert.gap, cert.feasibility_violation,
                                      1.0 if cert.passed else 0.0])
        bad = UB.MultiDual(tuple(z[f"c{k}_f{q}"] + (0.01 if q == 0 else 0.0) for q in range(kk)))
        cb = UB.mot_certificate(inputs, w, plan, bad)
        out[f"c{k}_bad"] = np.array([cb.primal, cb.dual, cb.gap, cb.feasibility_violation,
                                     1.0 if cb.passed else 0.0])
        done.append(k)
    out["cases"] = np.array(done)
    save("mot_cert.npz", **out)


def ref_barycenter(problem, iters, step):
    """barycenter.py:361-414 with the early exit removed and no _finalize."""
    inputs, w = problem.inputs, problem.omega
    rhos = problem.rhos()
    costfn = UB.barycentric_cost_fn(w)
    pots = [np.zeros(len(a)) for a in inputs]
    tr = {k: [] for k in ("h0", "fw_gap", "pd_gap")}
    plan = None
    for t in range(iters):
        lam = UB.multimarginal_lambda(UB.MultiDual(tuple(pots)), inputs, w, problem.rho)
        tilted = [a.weights * np.exp(-(f + lk) / rk) for a, f, lk, rk in zip(inputs, pots, lam, rhos)]
        plan, atoms = UB.solve_mot_1d([U.DiscreteMeasure(a.points, tw) for a, tw in zip(inputs, tilted)],
                                      w, costfn)
        fw_gap = float(sum(np.dot(tw, r - f) for tw, r, f in zip(tilted, atoms.potentials, pots)))
        dual = UB._h_value(inputs, rhos, pots)
        primal = UB.plan_cost(plan, inputs, costfn) + float(sum(
            U.divergence(U.KL(rk), plan.marginal(q, len(a)), a.weights)
            for q, (a, rk) in enumerate(zip(inputs, rhos))))
        tr["h0"].append(dual)
        tr["fw_gap"].append(fw_gap)
        tr["pd_gap"].append(primal - dual)
        if step == "harmonic":
            gamma = 2.0 / (2.0 + t)
        else:
            def value(g):
                return UB._h_value(inputs, rhos, [(1.0 - g) * f + g * r for f, r in zip(pots, atoms.potentials)])
            gamma = UF.ternary_max(value, 0.0, 1.0, iters=60)
            gamma = max(((value(c), c) for c in (gamma, 0.0, 1.0)), key=lambda z: z[0])[1]
        pots = [(1.0 - gamma) * f + gamma * r for f, r in zip(pots, atoms.potentials)]
    lam = UB.multimarginal_lambda(UB.MultiDual(tuple(pots)), inputs, w, problem.rho)
    return pots, lam, plan, {k: np.asarray(v) for k, v in tr.items()}


def gen_barycenter():
    rng = np.random.default_rng(19)
    out = {}
    specs = []
    for k in range(4):
        kk = [3, 4, 2, 5][k]
        inputs = []
        for _q in range(kk):
            n = int(rng.integers(8, 40))
            wq = rng.uniform(0.05, 1.0, n)
            wq *= rng.uniform(0.5, 2.0) / wq.sum()
            inputs.append(U.DiscreteMeasure(np.sort(rng.uniform(0, 1, n)), wq))
        w = rng.uniform(0.2, 1.0, kk)
        w /= w.sum()
        specs.append((inputs, w, float(rng.uniform(0.5, 2.0)), 60, ["linesearch", "harmonic"][k % 2]))
    xs, ws = S.cfg5_batch(count=1, n=128)
    specs.append(([U.DiscreteMeasure(xs[0, q], ws[0, q]) for q in range(16)], np.full(16, 1 / 16),
                  1.0, 40, "linesearch"))
    cases = []
    for k, (inputs, w, rho, iters, step) in enumerate(specs):
        t0 = time.time()
        problem = U.BarycenterProblem(tuple(inputs), w, rho)
        pots, lam, plan, tr = ref_barycenter(problem, iters, step)
        out[f"c{k}_k"] = np.array(len(inputs))
        out[f"c{k}_w"] = w
        out[f"c{k}_par"] = np.array([rho, iters, 1.0 if step == "linesearch" else 0.0])
        for q, mq in enumerate(inputs):
            out[f"c{k}_x{q}"], out[f"c{k}_a{q}"] = mq.points, mq.weights
            out[f"c{k}_f{q}"] = pots[q] + lam[q]
            out[f"c{k}_fraw{q}"] = pots[q]
        out[f"c{k}_idx"], out[f"c{k}_m"] = plan.indices, plan.mass
        bar = U.extract_barycenter(plan, inputs, w)
        out[f"c{k}_bar_x"], out[f"c{k}_bar_w"] = bar.points, bar.weights
        for kk_, v in tr.items():
            out[f"c{k}_{kk_}"] = v
        cases.append(k)
        print(f"  barycenter case {k}: K={len(inputs)} x{iters} {step} in {time.time() - t0:.1f}s")
    out["cases"] = np.array(cases)
    save("barycenter.npz", **out)


def gen_duality():
    """Known answers: tests/test_duality.py:64-75, :134-144, :185-200 style."""
    rng = np.random.default_rng(23)
    out = {}
    for k in range(8):
        n, m = int(rng.integers(2, 30)), int(rng.integers(2, 30))
        wa = rng.uniform(0.0, 1.0, n)
        wb = rng.uniform(0.1, 1.0, m)
        f = rng.normal(0, 1, n)
        g = rng.normal(0, 1, m)
        r1, r2 = float(rng.uniform(0.2, 3.0)), float(rng.uniform(0.2, 3.0))
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb), U.PowerDistance(2.0),
                            U.KL(r1), U.KL(r2), eps=0.3)
        d = U.DualPair(f, g)
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_f"], out[f"c{k}_g"] = f, g
        out[f"c{k}_par"] = np.array([r1, r2, 0.3])
        out[f"c{k}_lam"] = U.lambda_star(prob, d)
        out[f"c{k}_H"] = U.eval_H(prob, d)
        ta, tb = U.updated_marginals(prob, d)
        out[f"c{k}_ta"], out[f"c{k}_tb"] = ta, tb
        out[f"c{k}_sa"] = U.softmin(prob.alpha, r1, f)
    out["cases"] = np.arange(8)
    save("duality.npz", **out)


def gen_anderson():
    """Anderson-extrapolated runs (sinkhorn.py:197-243, :281-292) through the
    reference's own ``run`` (tol 1e-300 so the budget is spent unless delta_f
    hits exactly 0), plus ``anderson_weights`` known answers."""
    from uotkit.synthetic import mixture_measure

    out = {}
    cases = []
    # the reference's own acceleration test problem (tests/test_sinkhorn.py:260-271)
    a, _ = mixture_measure(20, 55)
    b, _ = mixture_measure(20, 56)
    specs = [(a.points, a.weights, b.points, b.weights, 2.0, 0.1, 5.0, 5.0, "f", 200, 4, 1e-7,
              "kl", None)]
    rng = np.random.default_rng(97)
    combos = [("f", 4, 1e-7, "kl"), ("h", 4, 1e-7, "kl"), ("g", 4, 1e-7, "kl"),
              ("f", 1, 1e-7, "kl"), ("f", 2, 1e-3, "kl"), ("h", 7, 1e-7, "kl"),
              ("f", 5, 0.0, "kl"), ("f", 4, 1e-7, "berg"), ("g", 3, 1e-6, "kl"),
              ("h", 3, 1e-5, "kl")]
    for k, (var, depth, reg, ent) in enumerate(combos):
        n, m = int(rng.integers(4, 48)), int(rng.integers(4, 48))
        p = [2.0, 1.0, 1.5][k % 3]
        eps = [0.1, 0.3, 0.05][k % 3]
        r1, r2 = float(rng.uniform(0.5, 3.0)), float(rng.uniform(0.5, 3.0))
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        wa = rng.uniform(0.1, 1.0, n)
        wb = rng.uniform(0.1, 1.0, m) * 1.4
        start = None
        if k % 2 == 1:
            C = np.abs(x[:, None] - y[None, :]) ** p
            start = (0.5 * C.min(axis=1) + 0.05, 0.5 * C.min(axis=0) - 0.05)
        specs.append((x, wa, y, wb, p, eps, r1, r2, var, 60, depth, reg, ent, start))
    c = S.cfg1_inputs()
    specs.append((c.x, c.alpha, c.y, c.beta, 2.0, c.eps, c.rho, c.rho, "f", 300, 4, 1e-7, "kl",
                  None))
    for k, (x, wa, y, wb, p, eps, r1, r2, var, iters, depth, reg, ent, start) in enumerate(specs):
        E = U.KL if ent == "kl" else U.Berg
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(p), E(r1), E(r2), eps=eps)
        init = None if start is None else U.DualPair(*start)
        cfg = US.SinkhornConfig(var, iters, 1e-300, US.AndersonConfig(depth, reg))
        rep = US.run(prob, cfg, init=init)
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_f0"] = np.zeros(len(x)) if start is None else start[0]
        out[f"c{k}_g0"] = np.zeros(len(y)) if start is None else start[1]
        out[f"c{k}_f"], out[f"c{k}_g"] = rep.final.f, rep.final.g
        out[f"c{k}_delta"] = rep.trace["delta_f"]
        out[f"c{k}_par"] = np.array([p, eps, r1, r2, iters, depth, reg,
                                     {"f": 0, "h": 1, "g": 2}[var], 0 if ent == "kl" else 1])
        cases.append(k)
    out["cases"] = np.array(cases)
    # anderson_weights known answers (tests/test_sinkhorn.py:243-258) + random windows
    wins = [(np.array([[1.0], [2.0]]), 1e-7), (np.tile(np.array([[1.0], [2.0]]), (1, 3)), 1e-7),
            (np.array([[np.sqrt(2.0), 0.0], [0.0, 1.0]]), 0.0)]
    for k in range(6):
        wins.append((rng.normal(size=(int(rng.integers(3, 200)), k % 5 + 2)), [0.0, 1e-7, 1e-2][k % 3]))
    for k, (Um, r) in enumerate(wins):
        out[f"w{k}_U"], out[f"w{k}_r"] = Um, np.array(r)
        out[f"w{k}_c"] = US.anderson_weights(Um, r)
    out["nwin"] = np.array(len(wins))
    save("anderson.npz", **out)


def gen_formats():
    """Reference writer outputs (measures / plans / traces, src/measures.py:185-254,
    src/ot1d.py:188-215, src/barycenter.py:446-475, src/sinkhorn.py:349-373,
    src/fw.py:360-381) and `uotkit gen` stdout, as text fixtures."""
    import contextlib
    import io

    from uotkit import cli as UC
    from uotkit import measures as UM
    from uotkit import ot1d as UO

    out = {}

    def text(fn, *args):
        buf = io.StringIO()
        fn(*args, buf)
        return buf.getvalue()

    for k, (kind, n, seed) in enumerate([("mixture", 40, 9), ("uniform", 3, 5), ("mixture", 5, 1),
                                         ("uniform", 17, 123)]):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert UC.main(["gen", "--kind", kind, "--n", str(n), "--seed", str(seed)]) == 0
        out[f"gen{k}_args"] = np.array([kind, str(n), str(seed)])
        out[f"gen{k}_text"] = np.array(buf.getvalue())
    rng = np.random.default_rng(5)
    a = U.DiscreteMeasure(rng.uniform(0, 1, 7), rng.uniform(0.1, 1, 7))
    b = U.DiscreteMeasure(rng.uniform(0, 1, 5), rng.uniform(0.1, 1, 5) * 0.0 + a.mass / 5)
    out["ma_x"], out["ma_w"] = a.points, a.weights
    out["mb_x"], out["mb_w"] = b.points, b.weights
    out["ma_csv"] = np.array(UM.measure_to_csv_text(a, ["one", "two three"]))
    out["ma_json"] = np.array(text(UM.write_measure_json, a))
    plan, _ = U.solve_ot_1d(a, b, U.PowerDistance(2.0))
    out["plan_i"], out["plan_j"], out["plan_m"] = plan.source_idx, plan.target_idx, plan.mass
    out["plan_csv"] = np.array(text(UO.write_plan_csv, plan))
    mp = UB.MultiPlan(np.array([[0, 0, 0], [0, 1, 0], [1, 1, 2]]), np.array([0.25, 0.5, 1e-17]))
    out["mp_idx"], out["mp_mass"] = mp.indices, mp.mass
    out["mp_csv"] = np.array(text(UB.write_multiplan_csv, mp))
    tr = {"delta_f": np.array([0.5, 1e-3, 2.5e-17]), "wall_ns": np.array([10, 20, 30])}
    rep = US.SolverReport(final=U.DualPair.zeros(1, 1), iterations=3, converged=True, trace=tr)
    out["tr_delta"], out["tr_wall"] = tr["delta_f"], tr["wall_ns"]
    out["trace_csv"] = np.array(text(US.write_trace_csv, rep))
    tr2 = dict(tr, err_f=np.array([1.0, 0.1, 0.01]), err_g=np.array([2.0, 0.2, 1e-300]))
    rep2 = US.SolverReport(final=U.DualPair.zeros(1, 1), iterations=3, converged=True, trace=tr2)
    out["tr_errf"], out["tr_errg"] = tr2["err_f"], tr2["err_g"]
    out["trace_ref_csv"] = np.array(text(US.write_trace_csv, rep2))
    tg = {"h0": np.array([0.1, 0.2]), "fw_gap": np.array([1.0, 1e-9]),
          "pd_gap": np.array([2.0, -1e-18]), "wall_ns": np.array([5, 7])}
    rep3 = US.SolverReport(final=U.DualPair.zeros(1, 1), iterations=2, converged=True, trace=tg)
    out["gap_h0"], out["gap_fw"], out["gap_pd"], out["gap_wall"] = (tg["h0"], tg["fw_gap"],
                                                                    tg["pd_gap"], tg["wall_ns"])
    out["gap_csv"] = np.array(text(UF.write_gap_csv, rep3))
    save("formats.npz", **out)


def gen_dense():
    """Dense / plan-level API helpers: build_cost_matrix, cost_quadruple_diameter,
    birkhoff_rate_bound, updated_marginals, eval_primal (sparse and dense plans,
    eps = 0 and eps > 0, KL and Balanced, an infinite case), and the certify
    norms / scalar oracle (src/measures.py:125-184, src/sinkhorn.py:338-346,
    src/duality.py:293-344, src/certify.py:73-118)."""
    from uotkit import certify as UC
    from uotkit import duality as UD
    from uotkit import measures as UM

    rng = np.random.default_rng(311)
    out = {}
    k = 0
    for p, (n, m) in zip([1.0, 2.0, 1.5, 2.0], [(7, 9), (33, 20), (12, 12), (60, 45)]):
        x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
        a, b = rng.uniform(0.1, 1, n), rng.uniform(0.1, 1, m)
        b *= a.sum() / b.sum()
        A, Bm = U.DiscreteMeasure(x, a), U.DiscreteMeasure(y, b)
        C = UM.build_cost_matrix(A, Bm, U.PowerDistance(p))
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, a, b
        out[f"c{k}_p"] = np.array(p)
        out[f"c{k}_C"] = C
        out[f"c{k}_diam"] = np.array(UM.cost_quadruple_diameter(C))
        r1, r2 = float(rng.uniform(0.5, 2)), float(rng.uniform(0.5, 2))
        eps = [0.05, 0.2, 0.1, 0.3][k]
        prob = U.UotProblem(A, Bm, U.PowerDistance(p), U.KL(r1), U.KL(r2), eps=eps)
        out[f"c{k}_par"] = np.array([r1, r2, eps])
        out[f"c{k}_birkhoff"] = np.array(US.birkhoff_rate_bound(prob))
        f, g = rng.normal(size=n) * 0.3, rng.normal(size=m) * 0.3
        out[f"c{k}_f"], out[f"c{k}_g"] = f, g
        ta, tb = UD.updated_marginals(prob, U.DualPair(f, g))
        out[f"c{k}_ta"], out[f"c{k}_tb"] = ta, tb
        # sparse plan (the balanced 1-D OT plan) at eps = 0 and eps > 0
        plan, _ = U.solve_ot_1d(A, Bm, U.PowerDistance(p))
        out[f"c{k}_pi"], out[f"c{k}_pj"], out[f"c{k}_pm"] = (plan.source_idx, plan.target_idx,
                                                              plan.mass)
        prob0 = U.UotProblem(A, Bm, U.PowerDistance(p), U.KL(r1), U.KL(r2), eps=0.0)
        out[f"c{k}_primal0"] = np.array(UD.eval_primal(prob0, plan))
        out[f"c{k}_primal_eps"] = np.array(UD.eval_primal(prob, plan))
        dense = rng.uniform(0, 1, (n, m)) * (rng.uniform(0, 1, (n, m)) < 0.3) / (n * m)
        out[f"c{k}_dense"] = dense
        out[f"c{k}_primal_dense"] = np.array(UD.eval_primal(prob, dense))
        probB = U.UotProblem(A, Bm, U.PowerDistance(p), U.Balanced(), U.KL(r2), eps=0.0)
        out[f"c{k}_primal_bal"] = np.array(UD.eval_primal(probB, plan))
        k += 1
    out["ncases"] = np.array(k)
    # infinite: mass on a zero-weight atom
    x = np.linspace(0, 1, 5)
    a = np.array([0.2, 0.0, 0.3, 0.2, 0.3])
    A = U.DiscreteMeasure(x, a)
    prob = U.UotProblem(A, A, U.PowerDistance(2.0), U.KL(1.0), U.KL(1.0), eps=0.0)
    dense = np.diag([0.2, 0.1, 0.3, 0.2, 0.2])
    out["inf_primal"] = np.array(UD.eval_primal(prob, dense))
    v = rng.normal(size=17)
    w = rng.normal(size=9)
    out["norm_f"], out["norm_g"] = v, w
    out["hilbert"] = np.array(UC.hilbert_norm(v))
    out["dstar"] = np.array(UC.double_star_norm(v, w))
    xm, vm = UC.scalar_max_oracle(lambda t: -(t - 0.37) ** 2 + 0.5 * np.sin(3 * t), (0.0, 1.0))
    out["oracle_x"], out["oracle_v"] = np.array(xm), np.array(vm)
    save("dense.npz", **out)


def gen_entropy_api():
    """Entropy-family functions (src/entropies.py:67-263), the FW single-step
    API (line_search_h0, pfw_step on an AtomStore, src/fw.py:118-323) and the
    certify grid oracles (src/certify.py:121-177), from the reference."""
    from uotkit import certify as UC
    from uotkit import entropies as UE

    rng = np.random.default_rng(2718)
    out = {}
    v = rng.normal(size=40) * 3
    w = rng.uniform(0, 1, 40)
    w[::7] = 0.0
    out["v"], out["w"] = v, w
    out["lde_flat"] = np.array(UE.logdotexp(v, w))
    M = rng.normal(size=(6, 40))
    out["M"] = M
    out["lde_ax1"] = UE.logdotexp(M, w, axis=1)
    M0 = rng.normal(size=(40, 5))
    out["M0"] = M0
    out["lde_ax0"] = UE.logdotexp(M0, w, axis=0)
    out["lde_zero"] = np.array(UE.logdotexp(v, np.zeros(40)))
    A = U.DiscreteMeasure(np.arange(40.0), np.where(w > 0, w, 0.5))
    out["aw"] = A.weights
    out["softmin"] = np.array(UE.softmin(A, 0.3, v))
    x = rng.normal(size=25)
    out["x"] = x
    specs = {"kl": U.KL(1.7), "berg": U.Berg(2.5), "bal": U.Balanced()}
    for name, sp in specs.items():
        xs = np.minimum(x, 2.4) if name == "berg" else x
        out[f"{name}_x"] = xs
        out[f"{name}_conj"] = UE.conj(sp, xs)
        out[f"{name}_grad"] = UE.conj_grad(sp, xs)
        out[f"{name}_hess"] = UE.conj_hess(sp, xs)
        out[f"{name}_aprox"] = UE.aprox(sp, 0.2, xs)
        mu = rng.uniform(0, 1, 30)
        nu = rng.uniform(0, 1, 30)
        nu[3] = 0.0
        if name == "berg":
            mu[5] = 0.7
        out[f"{name}_mu"], out[f"{name}_nu"] = mu, nu
        out[f"{name}_div"] = np.array(UE.divergence(sp, mu, nu))
        mu2 = mu.copy()
        mu2[3] = 0.0
        out[f"{name}_mu2"] = mu2
        out[f"{name}_div2"] = np.array(UE.divergence(sp, mu2, nu))
        out[f"{name}_div_same"] = np.array(UE.divergence(sp, nu, nu))
    # FW single steps on a small problem
    n, m = 30, 24
    xx, yy = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
    a, b = rng.uniform(0.1, 1, n), rng.uniform(0.1, 1, m) * 1.3
    prob = U.UotProblem(U.DiscreteMeasure(xx, a), U.DiscreteMeasure(yy, b), U.PowerDistance(2.0),
                        U.KL(1.2), U.KL(0.8), eps=0.0)
    out["fw_x"], out["fw_y"], out["fw_a"], out["fw_b"] = xx, yy, a, b
    cur = U.DualPair(np.zeros(n), np.zeros(m))
    _, _, _, atom, _ = UF._lmo(prob, cur)
    out["ls_gamma"] = np.array(UF.line_search_h0(prob, cur, atom))
    store = UF.AtomStore(np.zeros((1, n)), np.zeros((1, m)), np.array([1.0]))
    for it in range(4):
        store = UF.pfw_step(prob, store)
        out[f"pfw{it}_r"], out[f"pfw{it}_s"], out[f"pfw{it}_w"] = (store.r_atoms, store.s_atoms,
                                                                    store.weights)
    # fw_solve with a reference pair: the err_f trace (src/fw.py:217-219)
    ref = UF.fw_solve(prob, UF.FwConfig("harmonic", 400, 1e-12)).final
    rep = UF.fw_solve(prob, UF.FwConfig("harmonic", 30, 1e-300), reference=ref)
    out["fw_ref_f"], out["fw_ref_g"] = ref.f, ref.g
    out["fw_err_f"] = rep.trace["err_f"]
    f = rng.normal(size=11)
    g = rng.normal(size=7)
    out["gf"], out["gg"] = f, g
    out["hgrid"] = np.array(UC.hilbert_norm_grid(f))
    out["dgrid"] = np.array(UC.double_star_norm_grid(f, g))
    gx, gv = UC.grid_max_scalar(lambda t: -(t - 0.123) ** 2, 0.0, 1.0)
    out["gmax"] = np.array([gx, gv])
    save("entropy_api.npz", **out)


def _monge(rng, x, y, kind):
    """Submodular (Monge) cost families for the ExplicitMatrix path."""
    d = x[:, None] - y[None, :]
    u = rng.normal(size=x.size)
    v = rng.normal(size=y.size)
    if kind == 0:  # convex |d|^1.5 plus separable terms
        return np.abs(d) ** 1.5 + u[:, None] + v[None, :]
    if kind == 1:  # -x y (submodular for sorted supports), negative entries
        return -3.0 * x[:, None] * y[None, :] + 0.1 * u[:, None]
    if kind == 2:  # barycentric two-marginal cost, tests/test_barycenter.py:68-80
        return 0.3 * 0.7 * d ** 2
    return d ** 2 - 0.5  # tests/test_fw.py:86-91 (negative entries)


def gen_explicit():
    """ExplicitMatrix costs through solve_ot_1d (src/ot1d.py:92-109) and
    fw_solve (src/fw.py:151-232, :326-357 incl. the half-minima default
    init for negative costs), from the reference."""
    rng = np.random.default_rng(4242)
    out = {}
    ot_cases, fw_cases = [], []
    k = 0
    for kind in range(4):
        for _ in range(6):
            n, m = (int(v) for v in rng.integers(1, 40, 2))
            x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
            wa = rng.uniform(0.0, 1.0, n)
            if n > 3:
                wa[1] = 0.0  # zero-weight atoms keep their recursion values
            wb = rng.uniform(0.0, 1.0, m)
            wb *= wa.sum() / wb.sum()
            C = _monge(rng, x, y, kind)
            plan, d = U.solve_ot_1d(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                                    U.ExplicitMatrix(C))
            out[f"o{k}_x"], out[f"o{k}_y"], out[f"o{k}_a"], out[f"o{k}_b"] = x, y, wa, wb
            out[f"o{k}_C"] = C
            out[f"o{k}_i"], out[f"o{k}_j"], out[f"o{k}_m"] = (plan.source_idx, plan.target_idx,
                                                              plan.mass)
            out[f"o{k}_f"], out[f"o{k}_g"] = d.f, d.g
            ot_cases.append(k)
            k += 1
    k = 0
    for kind, step, iters in ((0, "linesearch", 60), (1, "harmonic", 80), (1, "linesearch", 60),
                              (3, "harmonic", 50), (0, "pairwise", 40), (1, "pairwise", 40)):
        n, m = int(rng.integers(20, 50)), int(rng.integers(20, 50))
        x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
        wa = rng.exponential(1.0, n)
        wa *= rng.uniform(0.5, 2.0) / wa.sum()
        wb = rng.exponential(1.0, m)
        wb *= rng.uniform(0.5, 2.0) / wb.sum()
        r1, r2 = float(rng.uniform(0.3, 2.0)), float(rng.uniform(0.3, 2.0))
        C = _monge(rng, x, y, kind)
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.ExplicitMatrix(C), U.KL(r1), U.KL(r2), eps=0.0)
        d0 = UF._default_init(prob)
        if step == "pairwise":
            d, lam, plan, tr = ref_pfw(prob, iters)
        else:
            d, lam, plan, tr = ref_fw(prob, iters, step)
        out[f"w{k}_x"], out[f"w{k}_y"], out[f"w{k}_a"], out[f"w{k}_b"] = x, y, wa, wb
        out[f"w{k}_C"] = C
        out[f"w{k}_par"] = np.array([r1, r2, iters, ["harmonic", "linesearch", "pairwise"].index(step)])
        out[f"w{k}_f0"], out[f"w{k}_g0"] = d0.f, d0.g
        out[f"w{k}_f"], out[f"w{k}_g"] = d.f + lam, d.g - lam
        out[f"w{k}_i"], out[f"w{k}_j"], out[f"w{k}_m"] = plan.source_idx, plan.target_idx, plan.mass
        for kk, v in tr.items():
            out[f"w{k}_{kk}"] = v
        fw_cases.append(k)
        k += 1
    # tests/test_fw.py:86-91 end to end: the reference's own fw_solve report
    a4 = U.DiscreteMeasure(np.sort(rng.uniform(0, 1, 4)), rng.uniform(0.2, 1, 4))
    b4 = U.DiscreteMeasure(np.sort(rng.uniform(0, 1, 4)), rng.uniform(0.2, 1, 4))
    C4 = (a4.points[:, None] - b4.points[None, :]) ** 2 - 0.5
    rep = U.fw_solve(U.UotProblem(a4, b4, U.ExplicitMatrix(C4), U.KL(1.0), U.KL(1.0), eps=0.0),
                     U.FwConfig("linesearch", 2000, 1e-8))
    out["e_x"], out["e_y"], out["e_a"], out["e_b"], out["e_C"] = (a4.points, b4.points,
                                                                  a4.weights, b4.weights, C4)
    out["e_f"], out["e_g"] = rep.final.f, rep.final.g
    out["e_iters"] = np.array(rep.iterations)
    out["e_passed"] = np.array(bool(rep.certificate.passed))
    out["ot_cases"], out["fw_cases"] = np.array(ot_cases), np.array(fw_cases)
    save("explicit.npz", **out)


def gen_bary_api():
    """The reference's own fw_barycenter report (src/barycenter.py:330-430):
    pairwise (= the line-search branch, :397-407) and harmonic, with the
    exhaustive feasibility term of the certificate (:416-418)."""
    rng = np.random.default_rng(77)
    out = {}
    k = 0
    for K, step, iters in ((3, "pairwise", 25), (3, "linesearch", 25), (2, "harmonic", 40),
                           (4, "pairwise", 15)):
        inputs = []
        for _q in range(K):
            n = int(rng.integers(6, 18))
            wq = rng.uniform(0.05, 1.0, n)
            wq *= rng.uniform(0.5, 2.0) / wq.sum()
            inputs.append(U.DiscreteMeasure(np.sort(rng.uniform(0, 1, n)), wq))
        w = rng.uniform(0.2, 1.0, K)
        w /= w.sum()
        rho = float(rng.uniform(0.5, 2.0))
        rep, plan = U.fw_barycenter(U.BarycenterProblem(tuple(inputs), w, rho),
                                    U.FwConfig(step, iters, 1e-9))
        out[f"c{k}_k"] = np.array(K)
        out[f"c{k}_w"] = w
        out[f"c{k}_par"] = np.array([rho, iters, ["harmonic", "linesearch", "pairwise"].index(step)])
        for q, mq in enumerate(inputs):
            out[f"c{k}_x{q}"], out[f"c{k}_a{q}"] = mq.points, mq.weights
            out[f"c{k}_f{q}"] = rep.final.potentials[q]
        out[f"c{k}_h0"] = np.asarray(rep.trace["h0"])
        out[f"c{k}_pd_gap"] = np.asarray(rep.trace["pd_gap"])
        c = rep.certificate
        out[f"c{k}_cert"] = np.array([c.primal, c.dual, c.gap, c.feasibility_violation, float(c.passed)])
        out[f"c{k}_iters"] = np.array(rep.iterations)
        k += 1
    out["cases"] = np.arange(k)
    save("bary_api.npz", **out)


def gen_berg():
    """Berg / mixed penalties off the KL closed form: the bracketed-Newton
    translation, updated marginals, F / G / H values, the primal with the
    Berg divergence (src/duality.py:135-303, src/entropies.py:104-138) and
    fixed-iteration FW runs (src/fw.py:106-232), from the reference."""
    from uotkit import duality as UD

    rng = np.random.default_rng(9001)
    out = {}
    specs = [(U.Berg(1.0), U.Berg(1.0)), (U.KL(0.8), U.Berg(1.4)), (U.Berg(0.6), U.KL(1.3)),
             (U.Berg(2.5), U.Berg(0.4))]
    for k, (e1, e2) in enumerate(specs):
        n, m = int(rng.integers(4, 30)), int(rng.integers(4, 30))
        x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
        wa, wb = rng.uniform(0.0, 1.0, n), rng.uniform(0.0, 1.0, m)
        wa[0] = 0.0
        f, g = rng.uniform(-0.3, 0.3, n), rng.uniform(-0.3, 0.3, m)
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(2.0), e1, e2, eps=0.0)
        d = U.DualPair(f, g)
        out[f"d{k}_x"], out[f"d{k}_y"], out[f"d{k}_a"], out[f"d{k}_b"] = x, y, wa, wb
        out[f"d{k}_f"], out[f"d{k}_g"] = f, g
        out[f"d{k}_ent"] = np.array([0 if isinstance(e1, U.KL) else 1, e1.rho,
                                     0 if isinstance(e2, U.KL) else 1, e2.rho])
        lam = U.lambda_star(prob, d)
        out[f"d{k}_lam"] = np.array(lam)
        ta, tb = U.updated_marginals(prob, d)
        out[f"d{k}_ta"], out[f"d{k}_tb"] = ta, tb
        # F / G / H at eps = 0 on a feasible pair, and F at eps > 0
        C = np.abs(x[:, None] - y[None, :]) ** 2
        fs = np.minimum(f, (C - g[None, :]).min(axis=1))
        dfs = U.DualPair(fs, g)
        out[f"d{k}_fs"] = fs
        out[f"d{k}_F"] = np.array(UD.eval_F(prob, dfs))
        out[f"d{k}_G"] = np.array(UD.eval_G(prob, dfs, 0.07))
        out[f"d{k}_H"] = np.array(UD.eval_H(prob, dfs))
        pe = U.UotProblem(prob.alpha, prob.beta, prob.cost, e1, e2, eps=0.3)
        out[f"d{k}_Feps"] = np.array(UD.eval_F(pe, d))
        # primal of a plan with full support on the positive-weight atoms
        plan, _ = U.solve_ot_1d(U.DiscreteMeasure(x, ta), U.DiscreteMeasure(y, tb))
        out[f"d{k}_pi"], out[f"d{k}_pj"], out[f"d{k}_pm"] = (plan.source_idx, plan.target_idx,
                                                             plan.mass)
        out[f"d{k}_primal"] = np.array(U.eval_primal(prob, plan))
        out[f"d{k}_primal_eps"] = np.array(U.eval_primal(pe, plan))
    fw_specs = [(U.Berg(1.0), U.Berg(1.0), "linesearch", 40), (U.KL(0.8), U.Berg(1.4), "harmonic", 60),
                (U.Berg(0.7), U.KL(1.1), "linesearch", 40), (U.Berg(1.5), U.Berg(0.5), "harmonic", 50)]
    for k, (e1, e2, step, iters) in enumerate(fw_specs):
        n, m = int(rng.integers(15, 45)), int(rng.integers(15, 45))
        x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
        wa = rng.exponential(1.0, n)
        wa *= rng.uniform(0.5, 2.0) / wa.sum()
        wb = rng.exponential(1.0, m)
        wb *= rng.uniform(0.5, 2.0) / wb.sum()
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(2.0), e1, e2, eps=0.0)
        dd, lam, plan, tr = ref_fw(prob, iters, step)
        out[f"w{k}_x"], out[f"w{k}_y"], out[f"w{k}_a"], out[f"w{k}_b"] = x, y, wa, wb
        out[f"w{k}_par"] = np.array([0 if isinstance(e1, U.KL) else 1, e1.rho,
                                     0 if isinstance(e2, U.KL) else 1, e2.rho, iters,
                                     1.0 if step == "linesearch" else 0.0])
        out[f"w{k}_f"], out[f"w{k}_g"] = dd.f + lam, dd.g - lam
        out[f"w{k}_i"], out[f"w{k}_j"], out[f"w{k}_m"] = plan.source_idx, plan.target_idx, plan.mass
        for kk, v in tr.items():
            out[f"w{k}_{kk}"] = v
    # tests/test_fw.py:121-125: the reference's own report on a Berg instance
    xa, xb = np.sort(rng.uniform(0, 1, 10)), np.sort(rng.uniform(0, 1, 9))
    wa = rng.uniform(0.2, 1.0, 10)
    wb = rng.uniform(0.2, 1.0, 9)
    wb *= wa.sum() / wb.sum()
    prob = U.UotProblem(U.DiscreteMeasure(xa, wa), U.DiscreteMeasure(xb, wb),
                        U.PowerDistance(2.0), U.Berg(1.0), U.Berg(1.0), eps=0.0)
    rep = U.fw_solve(prob, U.FwConfig("linesearch", 3000, 1e-7))
    out["e_x"], out["e_y"], out["e_a"], out["e_b"] = xa, xb, wa, wb
    out["e_f"], out["e_g"] = rep.final.f, rep.final.g
    out["e_iters"] = np.array(rep.iterations)
    out["e_h0"] = np.asarray(rep.trace["h0"])
    out["e_passed"] = np.array(bool(rep.certificate.passed))
    out["d_cases"], out["w_cases"] = np.arange(len(specs)), np.arange(len(fw_specs))
    save("berg.npz", **out)


def gen_sk_trace():
    """run(prob, config, reference=...) error traces for penalties off the
    KL closed form (src/sinkhorn.py:246-315): F with Berg / Balanced (no
    translation) and G with a Berg marginal (Newton translation)."""
    rng = np.random.default_rng(606)
    out = {}
    specs = [("f", U.Berg(1.0), U.Berg(0.7)), ("f", U.KL(0.9), U.Balanced()),
             ("g", U.KL(0.8), U.Berg(1.2)), ("g", U.Berg(1.5), U.Berg(0.6))]
    for k, (variant, e1, e2) in enumerate(specs):
        n, m = int(rng.integers(8, 30)), int(rng.integers(8, 30))
        x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
        wa = rng.uniform(0.1, 1.0, n)
        wb = rng.uniform(0.1, 1.0, m)
        if isinstance(e2, U.Balanced):
            wb *= wa.sum() / wb.sum()
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(2.0), e1, e2, eps=0.2)
        ref = US.run(prob, U.SinkhornConfig("f", 20000, 1e-13)).final
        rep = US.run(prob, U.SinkhornConfig(variant, 25, 1e-15), reference=ref)
        code = {U.KL: 0, U.Berg: 1, U.Balanced: 2}
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_par"] = np.array([0 if variant == "f" else 1, code[type(e1)],
                                     getattr(e1, "rho", 1.0), code[type(e2)],
                                     getattr(e2, "rho", 1.0)])
        out[f"c{k}_ref_f"], out[f"c{k}_ref_g"] = ref.f, ref.g
        for key in ("delta_f", "err_f", "err_g"):
            out[f"c{k}_{key}"] = np.asarray(rep.trace[key])
        out[f"c{k}_f"], out[f"c{k}_g"] = rep.final.f, rep.final.g
    out["cases"] = np.arange(len(specs))
    # g_sinkhorn_step at a given lam and Anderson-accelerated G with Berg
    for k, (e1, e2) in enumerate([(U.Berg(1.1), U.Berg(0.8)), (U.KL(0.7), U.Berg(1.3)),
                                  (U.Berg(0.9), U.KL(1.6))]):
        n, m = int(rng.integers(8, 30)), int(rng.integers(8, 30))
        x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
        wa, wb = rng.uniform(0.1, 1.0, n), rng.uniform(0.1, 1.0, m)
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(2.0), e1, e2, eps=0.15)
        f0, g0 = rng.uniform(-0.2, 0.2, n), rng.uniform(-0.2, 0.2, m)
        pair, lam1 = US.g_sinkhorn_step(prob, U.DualPair(f0, g0), 0.13)
        ref = US.run(prob, U.SinkhornConfig("f", 20000, 1e-13)).final
        rep = US.run(prob, U.SinkhornConfig("g", 12, 1e-15, anderson=U.AndersonConfig(3, 1e-9)),
                     reference=ref)
        code = {U.KL: 0, U.Berg: 1}
        out[f"s{k}_x"], out[f"s{k}_y"], out[f"s{k}_a"], out[f"s{k}_b"] = x, y, wa, wb
        out[f"s{k}_par"] = np.array([code[type(e1)], e1.rho, code[type(e2)], e2.rho])
        out[f"s{k}_f0"], out[f"s{k}_g0"] = f0, g0
        out[f"s{k}_f1"], out[f"s{k}_g1"], out[f"s{k}_lam1"] = pair.f, pair.g, np.array(lam1)
        out[f"s{k}_ref_f"], out[f"s{k}_ref_g"] = ref.f, ref.g
        for key in ("delta_f", "err_f", "err_g"):
            out[f"s{k}_and_{key}"] = np.asarray(rep.trace[key])
        out[f"s{k}_and_f"], out[f"s{k}_and_g"] = rep.final.f, rep.final.g
    out["step_cases"] = np.arange(3)
    save("sk_trace.npz", **out)


def gen_berg_pfw():
    """Pairwise FW with Berg / mixed penalties: the reference's own fw_solve
    report (src/fw.py:326-357) and its CLI (uot1d --entropy berg)."""
    import contextlib
    import io
    import tempfile

    from uotkit.cli import main as ref_main

    rng = np.random.default_rng(4747)
    out = {}
    for k, (e1, e2, iters) in enumerate([(U.Berg(1.0), U.Berg(1.0), 40), (U.KL(0.8), U.Berg(1.3), 40),
                                         (U.Berg(0.6), U.KL(1.2), 25)]):
        n, m = int(rng.integers(8, 25)), int(rng.integers(8, 25))
        x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
        wa = rng.uniform(0.1, 1.0, n)
        wb = rng.uniform(0.1, 1.0, m)
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.PowerDistance(2.0), e1, e2, eps=0.0)
        rep = U.fw_solve(prob, U.FwConfig("pairwise", iters, 1e-10))
        code = {U.KL: 0, U.Berg: 1}
        out[f"c{k}_x"], out[f"c{k}_y"], out[f"c{k}_a"], out[f"c{k}_b"] = x, y, wa, wb
        out[f"c{k}_par"] = np.array([code[type(e1)], e1.rho, code[type(e2)], e2.rho, iters])
        out[f"c{k}_h0"] = np.asarray(rep.trace["h0"])
        out[f"c{k}_pd_gap"] = np.asarray(rep.trace["pd_gap"])
        out[f"c{k}_f"], out[f"c{k}_g"] = rep.final.f, rep.final.g
        out[f"c{k}_passed"] = np.array(bool(rep.certificate.passed))
    with tempfile.TemporaryDirectory() as tmp:
        a, b = os.path.join(tmp, "a.csv"), os.path.join(tmp, "b.csv")
        with contextlib.redirect_stdout(io.StringIO()):
            ref_main(["gen", "--n", "12", "--seed", "5", "--out", a])
            ref_main(["gen", "--n", "10", "--seed", "6", "--out", b])
        for method in ("fw-ls", "fw", "pfw"):
            o = os.path.join(tmp, "o.json")
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = ref_main(["uot1d", a, b, "--entropy", "berg", "--method", method,
                               "--gap-tol", "1e-7", "--max-iters", "3000", "--out", o])
            out[f"cli_{method}_rc"] = np.array(rc)
            out[f"cli_{method}_cert"] = np.frombuffer(buf.getvalue().splitlines()[0].encode(),
                                                      dtype=np.uint8)
    out["cases"] = np.arange(3)
    # explicit (negative-entry) Monge cost with Berg / mixed penalties, fixed iterations
    for k, (e1, e2, step) in enumerate([(U.Berg(1.2), U.KL(0.9), "linesearch"),
                                        (U.Berg(0.8), U.Berg(1.1), "harmonic")]):
        n, m = int(rng.integers(10, 30)), int(rng.integers(10, 30))
        x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
        wa = rng.uniform(0.1, 1.0, n)
        wb = rng.uniform(0.1, 1.0, m)
        C = _monge(rng, x, y, 1)
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.ExplicitMatrix(C), e1, e2, eps=0.0)
        try:  # the half-minima init can leave the Berg translation domain empty
            U.fw_solve(prob, U.FwConfig(step, 5, 1e-12))
            out[f"x{k}_big_newton_error"] = np.array(False)
        except U.NewtonError:
            out[f"x{k}_big_newton_error"] = np.array(True)
        out[f"x{k}_Cbig"] = C
        C = 0.2 * C
        prob = U.UotProblem(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                            U.ExplicitMatrix(C), e1, e2, eps=0.0)
        d0 = UF._default_init(prob)
        dd, lam, plan, tr = ref_fw(prob, 30, step)
        out[f"x{k}_x"], out[f"x{k}_y"], out[f"x{k}_a"], out[f"x{k}_b"], out[f"x{k}_C"] = x, y, wa, wb, C
        out[f"x{k}_par"] = np.array([0 if isinstance(e1, U.KL) else 1, e1.rho,
                                     0 if isinstance(e2, U.KL) else 1, e2.rho,
                                     1.0 if step == "linesearch" else 0.0])
        out[f"x{k}_f0"], out[f"x{k}_g0"] = d0.f, d0.g
        out[f"x{k}_f"], out[f"x{k}_g"] = dd.f + lam, dd.g - lam
        out[f"x{k}_h0"] = tr["h0"]
    save("berg_pfw.npz", **out)



# ---------------------------------------------------------------------------
# Replay fixtures (round 2): the reference loops of fw.npz / pfw.npz /
# barycenter.npz re-run with every iteration's step size gamma_t (and, for
# pairwise, the away position) and the hash + entry count of every
# iteration's oracle plan recorded, so the device can replay the reference's
# steps and be compared at every iteration (tests/test_replay_gpu.py).


def _hash_pairs(plan):
    return O.plan_hash(np.stack([plan.source_idx, plan.target_idx], axis=1))


def ref_fw_rec(prob, iters, step):
    """fw.py:176-232 loop body (as ref_fw) recording gamma_t and the plans."""
    d = UF._default_init(prob)
    rec = {k: [] for k in ("h0", "gamma", "hash", "nnz")}
    for t in range(iters):
        ta, tb, plan, atom, fw_gap = UF._lmo(prob, d)
        rec["h0"].append(UF._h0(prob, d.f, d.g))
        h, c = _hash_pairs(plan)
        rec["hash"].append(h)
        rec["nnz"].append(c)
        gamma = 2.0 / (2.0 + t) if step == "harmonic" else UF.line_search_h0(prob, d, atom)
        rec["gamma"].append(gamma)
        d = U.DualPair((1.0 - gamma) * d.f + gamma * atom.f, (1.0 - gamma) * d.g + gamma * atom.g)
    return d, {k: np.asarray(v) for k, v in rec.items()}


def ref_pfw_rec(prob, iters):
    """fw.py:275-310 (_pfw_iteration), restated step by step on the
    reference's own helpers (_lmo, _h0, _active_scores, ternary_max,
    _merge_atom) so the away position and the transfer can be recorded;
    away = -1 when the iteration makes no step (fw.py:291-293, :298-299)."""
    d0 = UF._default_init(prob)
    store = UF.AtomStore(d0.f[None, :], d0.g[None, :], np.array([1.0]))
    rec = {k: [] for k in ("h0", "gamma", "away", "hash", "nnz", "natoms")}
    for _ in range(iters):
        d = store.current()
        ta, tb, plan, atom, fw_gap = UF._lmo(prob, d)
        rec["h0"].append(UF._h0(prob, d.f, d.g))
        h, c = _hash_pairs(plan)
        rec["hash"].append(h)
        rec["nnz"].append(c)
        scores = UF._active_scores(store, ta, tb)
        away = int(np.argmin(scores))
        max_step = float(store.weights[away])
        dr = atom.f - store.r_atoms[away]
        ds = atom.g - store.s_atoms[away]
        gamma = 0.0
        if not (max_step <= 0.0 or (np.abs(dr).max() < UF.ATOM_DEDUP_TOL
                                    and np.abs(ds).max() < UF.ATOM_DEDUP_TOL)):
            def value(gg):
                return UF._h0(prob, d.f + gg * dr, d.g + gg * ds)
            gamma = UF.ternary_max(value, 0.0, max_step, iters=60)
            gamma = max(((value(c_), c_) for c_ in (gamma, 0.0, max_step)), key=lambda z: z[0])[1]
        if gamma > 0.0:
            w = store.weights.copy()
            w[away] = max(w[away] - gamma, 0.0)
            r_atoms, s_atoms, w = UF._merge_atom(store.r_atoms, store.s_atoms, w, atom.f, atom.g,
                                                 gamma)
            keep = w > 0
            if not keep.all():
                r_atoms, s_atoms, w = r_atoms[keep], s_atoms[keep], w[keep]
            store = UF.AtomStore(r_atoms, s_atoms, w)
            rec["away"].append(away)
        else:
            rec["away"].append(-1)
        rec["gamma"].append(gamma)
        rec["natoms"].append(store.weights.size)
    return store.current(), {k: np.asarray(v) for k, v in rec.items()}


def ref_barycenter_rec(problem, iters, step):
    """barycenter.py:361-411 (as ref_barycenter) recording gamma_t and the plans."""
    inputs, w = problem.inputs, problem.omega
    rhos = problem.rhos()
    costfn = UB.barycentric_cost_fn(w)
    pots = [np.zeros(len(a)) for a in inputs]
    rec = {k: [] for k in ("h0", "gamma", "hash", "nnz")}
    for t in range(iters):
        lam = UB.multimarginal_lambda(UB.MultiDual(tuple(pots)), inputs, w, problem.rho)
        tilted = [a.weights * np.exp(-(f + lk) / rk) for a, f, lk, rk in zip(inputs, pots, lam, rhos)]
        plan, atoms = UB.solve_mot_1d([U.DiscreteMeasure(a.points, tw) for a, tw in zip(inputs, tilted)],
                                      w, costfn)
        rec["h0"].append(UB._h_value(inputs, rhos, pots))
        h, c = O.plan_hash(plan.indices)
        rec["hash"].append(h)
        rec["nnz"].append(c)
        if step == "harmonic":
            gamma = 2.0 / (2.0 + t)
        else:
            def value(g):
                return UB._h_value(inputs, rhos, [(1.0 - g) * f + g * r for f, r in zip(pots, atoms.potentials)])
            gamma = UF.ternary_max(value, 0.0, 1.0, iters=60)
            gamma = max(((value(c_), c_) for c_ in (gamma, 0.0, 1.0)), key=lambda z: z[0])[1]
        rec["gamma"].append(gamma)
        pots = [(1.0 - gamma) * f + gamma * r for f, r in zip(pots, atoms.potentials)]
    return pots, {k: np.asarray(v) for k, v in rec.items()}


def gen_replay():
    out = {}
    z = np.load(os.path.join(HERE, "fw.npz"))
    for k in z["cases"]:
        r1, r2, p, iters, ls = z[f"c{k}_par"]
        step = "linesearch" if ls else "harmonic"
        prob = U.UotProblem(U.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"]),
                            U.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"]),
                            U.PowerDistance(p), U.KL(r1), U.KL(r2), eps=0.0)
        t0 = time.time()
        d, rec = ref_fw_rec(prob, int(iters), step)
        out[f"fw{k}_f"], out[f"fw{k}_g"] = d.f, d.g
        for kk, v in rec.items():
            out[f"fw{k}_{kk}"] = v
        print(f"  replay fw {k}: {step} x{int(iters)} in {time.time() - t0:.1f}s", flush=True)
    z = np.load(os.path.join(HERE, "pfw.npz"))
    for k in z["cases"]:
        r1, r2, p, iters = z[f"c{k}_par"]
        prob = U.UotProblem(U.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"]),
                            U.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"]),
                            U.PowerDistance(p), U.KL(r1), U.KL(r2), eps=0.0)
        t0 = time.time()
        d, rec = ref_pfw_rec(prob, int(iters))
        assert np.array_equal(rec["natoms"], z[f"c{k}_natoms"])  # same loop as ref_pfw
        out[f"pfw{k}_f"], out[f"pfw{k}_g"] = d.f, d.g
        for kk, v in rec.items():
            out[f"pfw{k}_{kk}"] = v
        print(f"  replay pfw {k}: x{int(iters)} in {time.time() - t0:.1f}s", flush=True)
    z = np.load(os.path.join(HERE, "barycenter.npz"))
    for k in z["cases"]:
        kk_ = int(z[f"c{k}_k"])
        rho, iters, ls = z[f"c{k}_par"]
        inputs = tuple(U.DiscreteMeasure(z[f"c{k}_x{q}"], z[f"c{k}_a{q}"]) for q in range(kk_))
        problem = U.BarycenterProblem(inputs, z[f"c{k}_w"], float(rho))
        t0 = time.time()
        pots, rec = ref_barycenter_rec(problem, int(iters), "linesearch" if ls else "harmonic")
        for q in range(kk_):
            out[f"bary{k}_f{q}"] = pots[q]
        for kk, v in rec.items():
            out[f"bary{k}_{kk}"] = v
        print(f"  replay barycenter {k}: K={kk_} x{int(iters)} in {time.time() - t0:.1f}s", flush=True)
    out["fw_cases"] = np.load(os.path.join(HERE, "fw.npz"))["cases"]
    out["pfw_cases"] = np.load(os.path.join(HERE, "pfw.npz"))["cases"]
    out["bary_cases"] = np.load(os.path.join(HERE, "barycenter.npz"))["cases"]
    save("replay.npz", **out)


# ---------------------------------------------------------------------------
# Large 1-D problems (round 2): sizes beyond the resident
# on-chip path (n or m > 4096) -- the paper's FW experiment (PAPER.md:589:
# 5.000-sample measures, rho = 0.1) and n = 16384 (m = 12001: no exact ties of the uniform
# cumulative masses; m = 12000 is kept as the structural-tie case).  Inputs come from the
# reference's own generators (uotkit.synthetic, mirrored byte-for-byte by
# paper_2201_00730_b200.synthetic) or oracle.large_ot_inputs, so the fixture
# stores only outputs: potentials, per-iteration gamma / support hashes.


def gen_large():
    from uotkit import synthetic as USyn

    out = {}
    # solve_ot_1d with zero-weight atoms and ties, p = 2 and p = 1
    for k, (n, m, p, seed) in enumerate(((5000, 4999, 2.0, 1), (16384, 16384, 1.0, 2),
                                         (4097, 12000, 2.0, 3))):
        x, y, wa, wb = O.large_ot_inputs(n, m, seed)
        t0 = time.time()
        plan, duals = U.solve_ot_1d(U.DiscreteMeasure(x, wa), U.DiscreteMeasure(y, wb),
                                    U.PowerDistance(p))
        h, c = _hash_pairs(plan)
        out[f"ot{k}_spec"] = np.array([n, m, p, seed])
        out[f"ot{k}_f"], out[f"ot{k}_g"] = duals.f, duals.g
        out[f"ot{k}_hash"], out[f"ot{k}_nnz"] = np.array(h), np.array(c)
        out[f"ot{k}_mass8"] = plan.mass[::8].copy()
        print(f"  large ot {k}: {n}x{m} p={p} entries {c} in {time.time() - t0:.1f}s", flush=True)
    # FW on the paper's 5000-sample mixtures (rho = 0.1) and at n = 16384
    specs = [(5000, 5000, 11, 12, 0.1, "linesearch", 60), (5000, 5000, 11, 12, 0.1, "harmonic", 60),
             (16384, 12001, 13, 14, 1.0, "linesearch", 25)]
    for k, (n, m, sa, sb, rho, step, iters) in enumerate(specs):
        a, _ = USyn.mixture_measure(n, sa)
        b, _ = USyn.mixture_measure(m, sb)
        prob = U.UotProblem(a, b, U.PowerDistance(2.0), U.KL(rho), U.KL(rho), eps=0.0)
        t0 = time.time()
        d, rec = ref_fw_rec(prob, iters, step)
        lam = U.lambda_star(prob, d)
        out[f"fw{k}_spec"] = np.array([n, m, sa, sb, rho, 1.0 if step == "linesearch" else 0.0,
                                       iters])
        out[f"fw{k}_f"], out[f"fw{k}_g"] = d.f + lam, d.g - lam
        for kk, v in rec.items():
            out[f"fw{k}_{kk}"] = v
        print(f"  large fw {k}: {n}x{m} {step} x{iters} in {time.time() - t0:.1f}s", flush=True)
    # pairwise FW on the 5000-sample mixtures
    a, _ = USyn.mixture_measure(5000, 11)
    b, _ = USyn.mixture_measure(5000, 12)
    prob = U.UotProblem(a, b, U.PowerDistance(2.0), U.KL(0.1), U.KL(0.1), eps=0.0)
    t0 = time.time()
    d, rec = ref_pfw_rec(prob, 40)
    lam = U.lambda_star(prob, d)
    out["pfw_f"], out["pfw_g"] = d.f + lam, d.g - lam
    for kk, v in rec.items():
        out[f"pfw_{kk}"] = v
    print(f"  large pfw: 5000x5000 x40 in {time.time() - t0:.1f}s", flush=True)
    # uniform weights on 16384 x 12000 atoms: the cumulative masses of the two
    # sides coincide exactly at every 4096-th / 3000-th atom (structural ties,
    # SURVEY.md §0 finding 8); gamma_t, per-iteration plans (hash) recorded
    a, _ = USyn.mixture_measure(16384, 13)
    b, _ = USyn.mixture_measure(12000, 14)
    prob = U.UotProblem(a, b, U.PowerDistance(2.0), U.KL(1.0), U.KL(1.0), eps=0.0)
    d, rec = ref_fw_rec(prob, 6, "linesearch")
    lam = U.lambda_star(prob, d)
    out["tie_f"], out["tie_g"] = d.f + lam, d.g - lam
    for kk, v in rec.items():
        out[f"tie_{kk}"] = v
    save("large.npz", **out)

def gen_mot_custom():
    """solve_mot_1d / plan_cost / dual_feasibility_exhaustive / mot_certificate
    with custom tuple costs (barycenter.py:169-295, costfn given)."""
    from custom_costs import COSTS

    rng = np.random.default_rng(23)
    out = {}
    cases = []
    names = sorted(COSTS)
    for c in range(18):
        kk = int(rng.integers(2, 6)) if c < 15 else 8
        inputs = []
        for _q in range(kk):
            n = int(rng.integers(1, 25)) if c < 15 else 6
            wq = rng.uniform(0.1, 1.0, n)
            if n > 2 and c % 3 == 0:
                # zero-weight atom (tests/test_barycenter.py:95-105); not the last one: lists
                # ending in zero weights tie at their total masses, which differ in the last
                # ulp, and the reference breaks that tie on its clipped remainders
                # (barycenter.py:216-221) -- the structural near tie of DESIGN.md §2
                wq[rng.integers(0, n - 1)] = 0.0
            wq *= 1.7 / wq.sum()
            inputs.append(U.DiscreteMeasure(np.sort(rng.uniform(-1, 1, n)), wq))
        w = rng.uniform(0.2, 1.0, kk)
        w /= w.sum()
        name = names[c % len(names)]
        costfn = COSTS[name](w)
        plan, duals = UB.solve_mot_1d(inputs, costfn=costfn)
        out[f"c{c}_k"] = np.array(kk)
        out[f"c{c}_cost"] = np.array(name)
        out[f"c{c}_w"] = w
        for q, mq in enumerate(inputs):
            out[f"c{c}_x{q}"], out[f"c{c}_a{q}"] = mq.points, mq.weights
            out[f"c{c}_f{q}"] = duals.potentials[q]
        out[f"c{c}_idx"], out[f"c{c}_m"] = plan.indices, plan.mass
        out[f"c{c}_pc"] = np.array(UB.plan_cost(plan, inputs, costfn))
        cert = UB.mot_certificate(inputs, None, plan, duals, costfn=costfn)
        out[f"c{c}_cert"] = np.array([cert.primal, cert.dual, cert.gap,
                                      cert.feasibility_violation, 1.0 if cert.passed else 0.0])
        bad = UB.MultiDual(tuple(p + (0.01 if q == 0 else 0.0)
                                 for q, p in enumerate(duals.potentials)))
        cb = UB.mot_certificate(inputs, None, plan, bad, costfn=costfn)
        out[f"c{c}_bad"] = np.array([cb.primal, cb.dual, cb.gap, cb.feasibility_violation,
                                     1.0 if cb.passed else 0.0])
        grid = int(np.prod([len(m) for m in inputs], dtype=np.float64))
        out[f"c{c}_dfe"] = np.array(UB.dual_feasibility_exhaustive(inputs, bad, costfn)
                                    if grid <= 10**5 else np.nan)
        cases.append(c)
    out["cases"] = np.array(cases)
    save("mot_custom.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg1", "sinkhorn_small", "cfg3_small", "cfg4_small", "ot1d", "fw",
                             "mot", "barycenter", "duality", "pfw", "sinkhorn_g", "mot_cert",
                             "sinkhorn_ent", "anderson", "formats", "dense", "entropy_api", "explicit", "bary_api", "berg", "sk_trace", "berg_pfw", "replay", "large", "mot_custom"]
    for w in which:
        t0 = time.time()
        globals()[f"gen_{w}"]()
        print(f"[{w}] {time.time() - t0:.1f}s")
