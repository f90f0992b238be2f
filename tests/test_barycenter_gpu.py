"""GPU parity of the K-marginal sweep and the barycenter FW (csrc/mot1d.cu)
against the reference goldens and the CPU oracle."""

import numpy as np
import pytest

import oracle as O
import paper_2201_00730_b200 as P
from conftest import cases, golden
from paper_2201_00730_b200 import _device as D
from paper_2201_00730_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _inputs(z, k):
    kk = int(z[f"c{k}_k"])
    return [P.DiscreteMeasure(z[f"c{k}_x{q}"], z[f"c{k}_a{q}"]) for q in range(kk)], kk


def test_mot_goldens():
    z = golden("mot.npz")
    for k in cases(z):
        inputs, kk = _inputs(z, k)
        plan, duals = P.solve_mot_1d(inputs, z[f"c{k}_w"])
        np.testing.assert_array_equal(plan.indices, z[f"c{k}_idx"], err_msg=str(k))
        tot = float(np.sum(z[f"c{k}_m"]))
        np.testing.assert_allclose(plan.mass, z[f"c{k}_m"], rtol=0, atol=1e-13 * tot)
        scale = max(1e-300, max(np.abs(z[f"c{k}_f{q}"]).max() for q in range(kk)))
        for q in range(kk):
            assert np.abs(duals.potentials[q] - z[f"c{k}_f{q}"]).max() <= 1e-12 * max(scale, 1.0), k


def test_mot_known_answers():
    # tests/test_barycenter.py:58-66 of the reference (single atoms)
    inputs = [P.DiscreteMeasure([float(q)], [1.0]) for q in range(3)]
    w = np.full(3, 1 / 3)
    plan, duals = P.solve_mot_1d(inputs, w)
    assert len(plan) == 1 and plan.mass[0] == 1.0
    cost, _ = P.multimarginal_cost([0.0, 1.0, 2.0], w)
    assert duals.potentials[0][0] == pytest.approx(cost)
    assert duals.potentials[1][0] == 0.0 and duals.potentials[2][0] == 0.0
    with pytest.raises(P.MassBalanceError):
        P.solve_mot_1d([inputs[0], P.DiscreteMeasure([1.0], [2.0])], np.array([0.5, 0.5]))


def test_barycenter_goldens():
    """Fixed-iteration replay (the golden loop has no early exit)."""
    from paper_2201_00730_b200.barycenter import _pack

    z = golden("barycenter.npz")
    tight = 0
    for k in cases(z):
        inputs, kk = _inputs(z, k)
        rho, iters, ls = z[f"c{k}_par"]
        step = "linesearch" if ls else "harmonic"
        x, a, _, lens = _pack(inputs)
        r = P.fw_barycenter_batched(x, a, z[f"c{k}_w"], float(rho), int(iters), step, lens=lens)
        assert int(r.status[0].item()) == 0
        np.testing.assert_allclose(D.to_np(r.h0[0]), z[f"c{k}_h0"], rtol=1e-9, atol=1e-12,
                                   err_msg=str(k))
        f = D.to_np(r.f[0])
        scale = max(np.abs(z[f"c{k}_f{q}"]).max() for q in range(kk))
        err = max(np.abs(f[q, :lens[q]] - z[f"c{k}_f{q}"]).max() for q in range(kk))
        # ternary line search conditioning, see tests/test_fw_gpu.py
        assert err <= (1e-9 if step == "harmonic" else 1e-6) * scale, (k, err / scale)
        if err <= 1e-12 * scale:
            tight += 1
            c = int(r.count[0].item())
            idx = D.to_np(r.idx[0, :c]).astype(np.int64)
            np.testing.assert_array_equal(idx, z[f"c{k}_idx"])
            plan = P.MultiPlan(idx, D.to_np(r.mass[0, :c]))
            bar = P.extract_barycenter(plan, inputs, z[f"c{k}_w"])
            np.testing.assert_allclose(bar.points, z[f"c{k}_bar_x"], rtol=1e-12, atol=1e-14)
    assert tight >= 2


def test_fw_barycenter_api_dirac_inputs():
    # tests/test_barycenter.py:176-186 of the reference: Diracs -> weighted mean
    inputs = (P.DiscreteMeasure([0.0], [1.0]), P.DiscreteMeasure([1.0], [1.0]),
              P.DiscreteMeasure([2.5], [1.0]))
    w = np.array([0.2, 0.3, 0.5])
    rep, plan = P.fw_barycenter(P.BarycenterProblem(inputs, w, 3.0),
                                P.FwConfig("linesearch", 100, 1e-12))
    bar = P.extract_barycenter(plan, inputs, w)
    assert len(bar) == 1
    assert bar.points[0] == pytest.approx(1.55, abs=1e-12)


def test_barycenter_batched_cfg5_shape_vs_oracle():
    xs, ws = S.cfg5_batch(count=3, n=1024)
    w = np.full(16, 1 / 16)
    r = P.fw_barycenter_batched(xs, ws, w, 1.0, 12, "linesearch")
    assert (D.to_np(r.status) == 0).all()
    for p in (0, 2):
        out = O.fw_barycenter_fixed(list(xs[p]), list(ws[p]), w, 1.0, 12)
        np.testing.assert_allclose(D.to_np(r.h0[p]), out["h0"], rtol=1e-9)
        f = D.to_np(r.f[p])
        scale = max(np.abs(v).max() for v in out["pots"])
        err = max(np.abs(f[q] - out["pots"][q]).max() for q in range(16))
        assert err <= 1e-6 * scale
    rh = P.fw_barycenter_batched(xs, ws, w, 1.0, 12, "harmonic")
    out = O.fw_barycenter_fixed(list(xs[1]), list(ws[1]), w, 1.0, 12, step="harmonic")
    f = D.to_np(rh.f[1])
    scale = max(np.abs(v).max() for v in out["pots"])
    assert max(np.abs(f[q] - out["pots"][q]).max() for q in range(16)) <= 1e-9 * scale
    c = int(rh.count[1].item())
    np.testing.assert_array_equal(D.to_np(rh.idx[1, :c]), out["plan"][0])


def test_mot_full_cfg5_size_vs_oracle():
    xs, ws = S.cfg5_batch(count=2)
    w = np.full(16, 1 / 16)
    ws = ws / ws.sum(axis=2, keepdims=True)  # balanced inputs
    f, idx, mass, count, st = P.solve_mot_1d_batched(xs, ws, w)
    for p in range(2):
        ii, mm, pots = O.solve_mot_1d(list(xs[p]), list(ws[p]), w)
        c = int(count[p].item())
        got = D.to_np(idx[p, :c])
        np.testing.assert_array_equal(got, ii)
        np.testing.assert_allclose(D.to_np(mass[p, :c]), mm, rtol=0, atol=1e-13)
        fd = D.to_np(f[p])
        for q in range(16):
            assert np.abs(fd[q] - pots[q]).max() <= 1e-10


# ---------------------------------------------------------------------------
# Multi-marginal certificate at scale (§8f row 3): barycenter.py:236-295


def test_mot_certificate_matches_reference():
    z = golden("mot.npz")
    zc = golden("mot_cert.npz")
    for k in zc["cases"]:
        kk = int(z[f"c{k}_k"])
        inputs = [P.DiscreteMeasure(z[f"c{k}_x{q}"], z[f"c{k}_a{q}"]) for q in range(kk)]
        w = z[f"c{k}_w"]
        plan = P.MultiPlan(z[f"c{k}_idx"], z[f"c{k}_m"])
        for tag, shift in (("cert", 0.0), ("bad", 0.01)):
            duals = P.MultiDual(tuple(z[f"c{k}_f{q}"] + (shift if q == 0 else 0.0)
                                      for q in range(kk)))
            c = P.mot_certificate(inputs, w, plan, duals)
            ref = zc[f"c{k}_{tag}"]
            scale = 1.0 + abs(ref[0])
            assert abs(c.primal - ref[0]) <= 1e-12 * scale
            assert abs(c.dual - ref[1]) <= 1e-12 * scale
            assert abs(c.feasibility_violation - ref[3]) <= 1e-12 * scale
            assert c.passed == bool(ref[4]), (k, tag)


def test_mot_certificate_cfg5_scale():
    """K = 16 lists of 8192 atoms: the reference's int64 grid-size product
    overflows to 0 and it tries a TiB exhaustive sweep; the device certificate
    gates on the true size and checks support / marginals / gap."""
    xs, ws = S.cfg5_batch(count=1)
    inputs = [P.DiscreteMeasure(xs[0, q], ws[0, q] * (1.0 / ws[0, q].sum())) for q in range(16)]
    w = np.full(16, 1 / 16)
    plan, duals = P.solve_mot_1d(inputs, w)
    c = P.mot_certificate(inputs, w, plan, duals)
    assert c.passed
    assert abs(P.plan_cost(plan, inputs, P.barycentric_cost_fn(w)) - c.primal) < 1e-12


@pytest.mark.parametrize("k", range(4))
def test_fw_barycenter_report_vs_reference(k):
    """The reference's own fw_barycenter report (tests/golden/bary_api.npz):
    early exit, the final translated potentials, the certificate including
    its exhaustive feasibility term (src/barycenter.py:416-418); step
    "pairwise" runs the line-search branch (:397-407)."""
    z = golden("bary_api.npz")
    inputs, kk = _inputs(z, k)
    rho, iters, st = z[f"c{k}_par"]
    step = ["harmonic", "linesearch", "pairwise"][int(st)]
    problem = P.BarycenterProblem(tuple(inputs), z[f"c{k}_w"], float(rho))
    rep, plan = P.fw_barycenter(problem, P.FwConfig(step, int(iters), 1e-9))
    assert rep.iterations == int(z[f"c{k}_iters"])
    ref_h0 = z[f"c{k}_h0"]
    np.testing.assert_allclose(rep.trace["h0"], ref_h0, rtol=1e-9, atol=1e-13)
    scale = max(np.abs(z[f"c{k}_f{q}"]).max() for q in range(kk))
    tol = 1e-9 if step == "harmonic" else 1e-6
    for q in range(kk):
        assert np.abs(rep.final.potentials[q] - z[f"c{k}_f{q}"]).max() <= tol * scale
    primal, dual, gap, feas, passed = z[f"c{k}_cert"]
    c = rep.certificate
    assert c.primal == pytest.approx(primal, rel=1e-9)
    assert c.dual == pytest.approx(dual, rel=1e-9)
    assert abs(c.feasibility_violation - feas) <= 1e-12
    assert c.passed == bool(passed)


# ---------------------------------------------------------------------------
# Kernel variants of the sweep (csrc/mot1d.cu): the fine bin sort (default), the
# coarse one (UOT_MOT_COARSEBIN=1, also the path of buckets above 8 events per
# thread) and the merge-path fallback order the events identically (the (value, list, index) order is
# total), and the three update kernels (mot_update_s, the default of small
# batches; mot_update2 with UOT_MOT_UPDATES=0; mot_update with
# UOT_MOT_UPDATE1=1) compute the same iterates; clustered keys (zero-weight runs repeat breakpoints) and ties
# across lists (identical inputs) exercise the fallback and the tie rule.
@pytest.mark.parametrize("env,val", [("UOT_MOT_NOBIN", "1"), ("UOT_MOT_COARSEBIN", "1"),
                                     ("UOT_MOT_UPDATE1", "1"), ("UOT_MOT_UPDATES", "0")])
def test_sweep_variants_agree(monkeypatch, env, val):
    xs, ws = S.cfg5_batch(count=3, n=2048)
    ws[1, :, 100:400] = 0.0          # zero-weight runs: repeated breakpoints
    xs[2, 5] = xs[2, 4]              # two identical lists: cross-list ties
    ws[2, 5] = ws[2, 4]
    w = np.full(16, 1 / 16)
    # the two update kernels associate their block / cluster sums differently:
    # compared on harmonic steps (a fixed gamma schedule); the merge fallback
    # orders the same keys, compared on line-search runs
    step = "linesearch" if env in ("UOT_MOT_NOBIN", "UOT_MOT_COARSEBIN") else "harmonic"
    base = P.fw_barycenter_batched(xs, ws, w, 1.0, 15, step, trace_support=True)
    monkeypatch.setenv(env, val)
    alt = P.fw_barycenter_batched(xs, ws, w, 1.0, 15, step, trace_support=True)
    monkeypatch.delenv(env)
    assert (D.to_np(base.status) == 0).all() and (D.to_np(alt.status) == 0).all()
    np.testing.assert_array_equal(D.to_np(base.supp_hash), D.to_np(alt.supp_hash))
    f0, f1 = D.to_np(base.f), D.to_np(alt.f)
    tol = 1e-14 if env in ("UOT_MOT_NOBIN", "UOT_MOT_COARSEBIN") else 1e-13
    assert np.abs(f0 - f1).max() <= tol * np.abs(f0).max()
    np.testing.assert_allclose(D.to_np(alt.h0), D.to_np(base.h0), rtol=max(tol, 1e-13))
    c = D.to_np(base.count)
    for p in range(3):
        np.testing.assert_array_equal(D.to_np(alt.idx[p, :c[p]]), D.to_np(base.idx[p, :c[p]]))
    # balanced sweep at full size through the fallback as well
    if env == "UOT_MOT_NOBIN":
        xb, wb = S.cfg5_batch(count=1)
        wb = wb / wb.sum(axis=2, keepdims=True)
        r0 = P.solve_mot_1d_batched(xb, wb, w)
        monkeypatch.setenv(env, "1")
        r1 = P.solve_mot_1d_batched(xb, wb, w)
        monkeypatch.delenv(env)
        c0 = int(r0[3][0].item())
        np.testing.assert_array_equal(D.to_np(r0[1][0, :c0]), D.to_np(r1[1][0, :c0]))


# ---------------------------------------------------------------------------
# More than 16 input measures (the reference has no limit, barycenter.py:169-233):
# 16 < K <= 32 runs on clusters of ceil(K/2) CTAs holding two lists each
# (odd K: the last CTA holds one); the balanced sweep needs no cluster at all.
@pytest.mark.parametrize("k,n", [(21, 300), (32, 1000), (24, 129)])
def test_barycenter_many_inputs_vs_oracle(k, n):
    xs, ws = S.cfg5_batch(batch=2, k=k, n=n, count=2)
    w = np.full(k, 1.0 / k)
    rh = P.fw_barycenter_batched(xs, ws, w, 1.0, 10, "harmonic")
    assert (D.to_np(rh.status) == 0).all()
    for p in range(2):
        out = O.fw_barycenter_fixed(list(xs[p]), list(ws[p]), w, 1.0, 10, step="harmonic")
        np.testing.assert_allclose(D.to_np(rh.h0[p]), out["h0"], rtol=1e-9)
        f = D.to_np(rh.f[p])
        scale = max(np.abs(v).max() for v in out["pots"])
        assert max(np.abs(f[q] - out["pots"][q]).max() for q in range(k)) <= 1e-9 * scale
        c = int(rh.count[p].item())
        np.testing.assert_array_equal(D.to_np(rh.idx[p, :c]), out["plan"][0])
    rl = P.fw_barycenter_batched(xs, ws, w, 1.0, 6, "linesearch")
    out = O.fw_barycenter_fixed(list(xs[0]), list(ws[0]), w, 1.0, 6)
    np.testing.assert_allclose(D.to_np(rl.h0[0]), out["h0"], rtol=1e-9)


@pytest.mark.parametrize("k,n", [(24, 300), (32, 2049)])
def test_mot_many_inputs_vs_oracle(k, n):
    xs, ws = S.cfg5_batch(batch=1, k=k, n=n, count=1)
    ws = ws / ws.sum(axis=2, keepdims=True)
    w = np.full(k, 1.0 / k)
    f, idx, mass, count, st = P.solve_mot_1d_batched(xs, ws, w)
    ii, mm, pots = O.solve_mot_1d(list(xs[0]), list(ws[0]), w)
    c = int(count[0].item())
    np.testing.assert_array_equal(D.to_np(idx[0, :c]), ii)
    np.testing.assert_allclose(D.to_np(mass[0, :c]), mm, rtol=0, atol=1e-13)
    fd = D.to_np(f[0])
    assert max(np.abs(fd[q] - pots[q]).max() for q in range(k)) <= 1e-10


def test_too_many_inputs_raise_like_a_limit():
    xs, ws = S.cfg5_batch(batch=1, k=33, n=64, count=1)
    with pytest.raises(ValueError):
        P.fw_barycenter_batched(xs, ws, np.full(33, 1 / 33), 1.0, 2, "harmonic")


# ---------------------------------------------------------------------------
# Lists beyond 16384 atoms (K <= 16): 64 / 128 / 256 atoms per thread with the
# per-atom loops rolled (csrc/mot1d.cu: ept_for), up to 768 buckets per problem.
@pytest.mark.parametrize("k,n", [(4, 20000), (3, 70001), (16, 40000)])
def test_long_lists_vs_oracle(k, n):
    xs, ws = S.cfg5_batch(batch=1, k=k, n=n, count=1, floor=1e-3)
    w = np.full(k, 1.0 / k)
    wb = ws / ws.sum(axis=2, keepdims=True)
    f, idx, mass, count, st = P.solve_mot_1d_batched(xs, wb, w)
    assert int(st[0].item()) == 0
    ii, mm, pots = O.solve_mot_1d(list(xs[0]), list(wb[0]), w)
    c = int(count[0].item())
    np.testing.assert_array_equal(D.to_np(idx[0, :c]), ii)
    np.testing.assert_allclose(D.to_np(mass[0, :c]), mm, rtol=0, atol=1e-13)
    fd = D.to_np(f[0])
    assert max(np.abs(fd[q] - pots[q]).max() for q in range(k)) <= 1e-10
    its = 4
    rh = P.fw_barycenter_batched(xs, ws, w, 1.0, its, "harmonic")
    assert int(rh.status[0].item()) == 0
    out = O.fw_barycenter_fixed(list(xs[0]), list(ws[0]), w, 1.0, its, step="harmonic")
    np.testing.assert_allclose(D.to_np(rh.h0[0]), out["h0"], rtol=1e-9)
    fh = D.to_np(rh.f[0])
    scale = max(np.abs(v).max() for v in out["pots"])
    assert max(np.abs(fh[q] - out["pots"][q]).max() for q in range(k)) <= 1e-9 * scale
    rl = P.fw_barycenter_batched(xs, ws, w, 1.0, 3, "linesearch")
    outl = O.fw_barycenter_fixed(list(xs[0]), list(ws[0]), w, 1.0, 3)
    np.testing.assert_allclose(D.to_np(rl.h0[0]), outl["h0"], rtol=1e-9)


def test_list_length_limit_message():
    xs = np.sort(np.random.default_rng(0).uniform(size=(1, 2, 131073)), axis=2)
    ws = np.full((1, 2, 131073), 1.0 / 131073)
    with pytest.raises(ValueError, match="131072"):
        P.solve_mot_1d_batched(xs, ws, np.full(2, 0.5))
