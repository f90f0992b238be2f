"""GPU parity of ExplicitMatrix costs on the 1-D OT oracle and the batched
Frank-Wolfe kernel (csrc/fw1d_kernel.cuh, cost kind PK = 3) against the
reference's solve_ot_1d / fw_solve on explicit (Monge) matrices
(tests/golden/explicit.npz, src/ot1d.py:92-109, src/fw.py:151-357).
Plan supports bit-exact; potentials 1e-12 relative for the sweep, the FW
tolerances of tests/test_fw_gpu.py for the iterations."""

import numpy as np
import pytest

import oracle as O
import paper_2201_00730_b200 as P
from conftest import golden, rel_err
from paper_2201_00730_b200 import _device as D
from paper_2201_00730_b200 import fw as F
from paper_2201_00730_b200 import synthetic as S

pytestmark = pytest.mark.gpu

STEPS = ["harmonic", "linesearch", "pairwise"]


def test_explicit_ot_goldens():
    z = golden("explicit.npz")
    for k in z["ot_cases"]:
        a = P.DiscreteMeasure(z[f"o{k}_x"], z[f"o{k}_a"])
        b = P.DiscreteMeasure(z[f"o{k}_y"], z[f"o{k}_b"])
        plan, d = P.solve_ot_1d(a, b, P.ExplicitMatrix(z[f"o{k}_C"]))
        np.testing.assert_array_equal(plan.source_idx, z[f"o{k}_i"], err_msg=str(k))
        np.testing.assert_array_equal(plan.target_idx, z[f"o{k}_j"], err_msg=str(k))
        np.testing.assert_allclose(plan.mass, z[f"o{k}_m"], rtol=0,
                                   atol=1e-13 * float(np.sum(z[f"o{k}_a"])))
        assert rel_err(d.f, d.g, z[f"o{k}_f"], z[f"o{k}_g"]) < 1e-12, k


def test_explicit_matches_power_path_at_cfg2_shape():
    """C = (x - y)^2 as an explicit matrix reproduces the |x - y|^2 kernel at
    full cfg2 problem size (1024 x 1024 per problem): the plan (a function
    of the masses only) bit for bit, the potentials to rounding (the power
    kernel contracts d*d - e*e into an FMA, the table lookup cannot)."""
    x, y, a, b = S.cfg2_batch(count=3)
    bal = b * (a.sum(1) / b.sum(1))[:, None]
    C = (x[:, :, None] - y[:, None, :]) ** 2
    r0 = [D.to_np(v) for v in P.solve_ot_1d_batched(x, y, a, bal, 2.0)]
    r1 = [D.to_np(v) for v in P.solve_ot_1d_batched(x, y, a, bal, C=C)]
    for u, v in zip(r0[2:], r1[2:]):  # ei, ej, em, count, status
        assert np.array_equal(u, v)
    for k in range(3):
        assert rel_err(r1[0][k], r1[1][k], r0[0][k], r0[1][k]) < 1e-13
    f0 = F.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, 30, "harmonic")
    f1 = F.fw_solve_batched(x, y, a, b, 1.0, 1.0, 2.0, 30, "harmonic", C=C)
    np.testing.assert_allclose(D.to_np(f1.h0), D.to_np(f0.h0), rtol=1e-12)
    for k in range(3):
        assert rel_err(D.to_np(f1.f[k]), D.to_np(f1.g[k]), D.to_np(f0.f[k]),
                       D.to_np(f0.g[k])) < 1e-11
    for name in ("ei", "ej", "count"):
        assert np.array_equal(D.to_np(getattr(f0, name)), D.to_np(getattr(f1, name))), name


def test_explicit_shift_and_scaled_power_cost():
    """tests/test_ot1d.py:78-88 and :102-106: C + 5 keeps the plan and adds
    5 * mass to its cost; 0.37 * |x - y|^2 is accepted and certified."""
    rng = np.random.default_rng(8)
    x, y = np.sort(rng.uniform(0, 1, 8)), np.sort(rng.uniform(0, 1, 6))
    wa = rng.uniform(0.1, 1, 8)
    wb = rng.uniform(0.1, 1, 6)
    wb *= wa.sum() / wb.sum()
    a, b = P.DiscreteMeasure(x, wa), P.DiscreteMeasure(y, wb)
    C = P.build_cost_matrix(a, b, P.PowerDistance(2.0))
    plan0, _ = P.solve_ot_1d(a, b, P.PowerDistance(2.0))
    plan5, d5 = P.solve_ot_1d(a, b, P.ExplicitMatrix(C + 5.0))
    assert plan0.source_idx.tolist() == plan5.source_idx.tolist()
    assert plan0.target_idx.tolist() == plan5.target_idx.tolist()
    np.testing.assert_allclose(plan0.mass, plan5.mass)
    assert plan5.cost_value(C + 5.0) == pytest.approx(plan0.cost_value(C) + 5.0 * a.mass,
                                                      rel=1e-12)
    C2 = np.asarray(C) * 0.37
    plan, d = P.solve_ot_1d(a, b, P.ExplicitMatrix(C2))
    assert P.check_complementary_slackness(plan, d, C2)


def test_explicit_errors():
    a = P.DiscreteMeasure([0.0, 1.0], [0.5, 0.5])
    with pytest.raises(P.SubmodularityError):  # tests/test_ot1d.py:96-100
        P.solve_ot_1d(a, a, P.ExplicitMatrix(np.array([[1.0, 0.0], [0.0, 1.0]])))
    with pytest.raises(ValueError):
        P.solve_ot_1d(a, a, P.ExplicitMatrix(np.zeros((3, 2))))
    prob = P.UotProblem(a, a, P.ExplicitMatrix(np.array([[1.0, 0.0], [0.0, 1.0]])), P.KL(1.0),
                        P.KL(1.0), eps=0.0)
    with pytest.raises(P.SubmodularityError):
        P.fw_solve(prob)


def test_explicit_sweep_vs_oracle_batched():
    rng = np.random.default_rng(21)
    B, n, m = 16, 300, 211
    x = np.sort(rng.uniform(0, 1, (B, n)), axis=1)
    y = np.sort(rng.uniform(0, 1, (B, m)), axis=1)
    a = rng.exponential(1.0, (B, n))
    a[:, ::9] = 0.0
    b = rng.exponential(1.0, (B, m))
    b *= (a.sum(1) / b.sum(1))[:, None]
    C = (-2.0 * x[:, :, None] * y[:, None, :] + rng.normal(size=(B, n))[:, :, None]
         + np.abs(x[:, :, None] - y[:, None, :]) ** 1.3)
    f, g, ei, ej, em, cnt, st = P.solve_ot_1d_batched(x, y, a, b, C=C)
    for k in range(B):
        ii, jj, mm, fo, go = O.solve_ot_1d(None, None, a[k], b[k], explicit=C[k])
        c = int(cnt[k].item())
        np.testing.assert_array_equal(D.to_np(ei[k, :c]), ii)
        np.testing.assert_array_equal(D.to_np(ej[k, :c]), jj)
        np.testing.assert_allclose(D.to_np(em[k, :c]), mm, rtol=0, atol=1e-13 * a[k].sum())
        assert rel_err(D.to_np(f[k]), D.to_np(g[k]), fo, go) < 1e-12


def _fw_case(z, k):
    r1, r2, iters, st = z[f"w{k}_par"]
    return (z[f"w{k}_x"], z[f"w{k}_y"], z[f"w{k}_a"], z[f"w{k}_b"], z[f"w{k}_C"], float(r1),
            float(r2), int(iters), STEPS[int(st)])


@pytest.mark.parametrize("k", range(6))
def test_explicit_fw_goldens(k):
    """Fixed-iteration FW on explicit costs from the half-minima default init
    (src/fw.py:151-156) vs the reference loop; pairwise as in
    tests/test_pfw_gpu.py (identical while one atom is active, then the
    invariants)."""
    z = golden("explicit.npz")
    x, y, a, b, C, r1, r2, iters, step = _fw_case(z, k)
    r = F.fw_solve_batched(x, y, a, b, r1, r2, 2.0, iters, step, f0=z[f"w{k}_f0"],
                           g0=z[f"w{k}_g0"], C=C)
    assert int(r.status[0].item()) == 0
    h0, pd = D.to_np(r.h0[0]), D.to_np(r.pd_gap[0])
    ref_h0 = z[f"w{k}_h0"]
    scale = np.abs(ref_h0).max()
    if step == "pairwise":
        assert np.abs(h0[:2] - ref_h0[:2]).max() / scale < 1e-9
        assert np.all(np.diff(h0) >= -1e-12 * scale)
        assert pd.min() >= -1e-9 * scale
        assert h0[-1] >= ref_h0[-1] - 1e-9 * scale
        f, g = D.to_np(r.f[0]), D.to_np(r.g[0])
        lam = float(r.summary[0, 2].item())
        viol = float(F.feasibility_violation(x, y, f - lam, g + lam, C=C)[0].item())
        assert viol <= 1e-9
        return
    np.testing.assert_allclose(h0, ref_h0, rtol=1e-9, atol=1e-12 * scale)
    np.testing.assert_allclose(pd, z[f"w{k}_pd_gap"], rtol=0, atol=4e-9 * scale)
    err = rel_err(D.to_np(r.f[0]), D.to_np(r.g[0]), z[f"w{k}_f"], z[f"w{k}_g"])
    assert err < (1e-9 if step == "harmonic" else 1e-6), err
    if err < 1e-12:
        c = int(r.count[0].item())
        np.testing.assert_array_equal(D.to_np(r.ei[0, :c]), z[f"w{k}_i"])
        np.testing.assert_array_equal(D.to_np(r.ej[0, :c]), z[f"w{k}_j"])


def test_explicit_fw_solve_api_default_init():
    """tests/test_fw.py:86-91: negative explicit costs, the default init
    shift, the reference's own fw_solve report."""
    z = golden("explicit.npz")
    a = P.DiscreteMeasure(z["e_x"], z["e_a"])
    b = P.DiscreteMeasure(z["e_y"], z["e_b"])
    prob = P.UotProblem(a, b, P.ExplicitMatrix(z["e_C"]), P.KL(1.0), P.KL(1.0), eps=0.0)
    rep = P.fw_solve(prob, P.FwConfig("linesearch", 2000, 1e-8))
    assert rep.certificate.passed
    assert rep.iterations == int(z["e_iters"])
    assert rel_err(rep.final.f, rep.final.g, z["e_f"], z["e_g"]) < 1e-6
    for k in range(6):  # the default init the solver builds equals the reference's
        x, y, wa, wb, C, r1, r2, _, _ = _fw_case(z, k)
        pr = P.UotProblem(P.DiscreteMeasure(x, wa), P.DiscreteMeasure(y, wb), P.ExplicitMatrix(C),
                          P.KL(r1), P.KL(r2), eps=0.0)
        d0 = F._default_init(pr, D.to_dev(C, D.torch().float64))
        np.testing.assert_array_equal(d0.f, z[f"w{k}_f0"])
        np.testing.assert_array_equal(d0.g, z[f"w{k}_g0"])


def test_two_marginal_sweep_equals_explicit_pairwise():
    """tests/test_barycenter.py:68-80: the K = 2 multi-marginal sweep and the
    pairwise solver on the barycentric cost matrix give the same plan."""
    from paper_2201_00730_b200 import barycenter as PB

    rng = np.random.default_rng(5)
    w = np.array([0.3, 0.7])
    for _ in range(10):
        n, m = (int(v) for v in rng.integers(2, 11, 2))
        a = P.DiscreteMeasure(np.sort(rng.uniform(0, 1, n)), rng.uniform(0.1, 1, n))
        wb = rng.uniform(0.1, 1, m)
        b = P.DiscreteMeasure(np.sort(rng.uniform(0, 1, m)), wb * a.mass / wb.sum())
        plan, _ = PB.solve_mot_1d([a, b], w)
        Cm = w[0] * w[1] * (a.points[:, None] - b.points[None, :]) ** 2
        plan2, _ = P.solve_ot_1d(a, b, P.ExplicitMatrix(Cm))
        assert plan.indices[:, 0].tolist() == plan2.source_idx.tolist()
        assert plan.indices[:, 1].tolist() == plan2.target_idx.tolist()
        v1 = PB.plan_cost(plan, [a, b], PB.barycentric_cost_fn(w))
        v2 = plan2.cost_value(Cm)
        assert abs(v1 - v2) <= 1e-10 * (1 + abs(v1))
