"""Custom tuple costs on the B200 path: solve_mot_1d(inputs, costfn=...),
plan_cost, dual_feasibility_exhaustive and mot_certificate with a caller
costfn (src/barycenter.py:169-295) against the reference's own outputs
(tests/golden/mot_custom.npz, make_golden.py::gen_mot_custom) and the oracle."""

import os
import sys

import numpy as np
import pytest

import oracle as O
import paper_2201_00730_b200 as P
from conftest import cases, golden

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from custom_costs import COSTS, pairwise_pow15, plain_barycentric, spread  # noqa: E402

pytestmark = pytest.mark.gpu


def _case(z, c):
    kk = int(z[f"c{c}_k"])
    inputs = [P.DiscreteMeasure(z[f"c{c}_x{q}"], z[f"c{c}_a{q}"]) for q in range(kk)]
    return inputs, kk, COSTS[str(z[f"c{c}_cost"])](z[f"c{c}_w"])


def test_custom_cost_sweep_goldens():
    z = golden("mot_custom.npz")
    for c in cases(z):
        inputs, kk, costfn = _case(z, c)
        plan, duals = P.solve_mot_1d(inputs, costfn=costfn)
        np.testing.assert_array_equal(plan.indices, z[f"c{c}_idx"], err_msg=str(c))
        tot = float(np.sum(z[f"c{c}_m"]))
        np.testing.assert_allclose(plan.mass, z[f"c{c}_m"], rtol=0, atol=1e-13 * tot)
        scale = max(1.0, max(np.abs(z[f"c{c}_f{q}"]).max() for q in range(kk)))
        for q in range(kk):
            err = np.abs(duals.potentials[q] - z[f"c{c}_f{q}"]).max()
            assert err <= 1e-12 * scale, (c, q, err)


def test_custom_cost_certificates_goldens():
    z = golden("mot_custom.npz")
    for c in cases(z):
        inputs, kk, costfn = _case(z, c)
        plan = P.MultiPlan(z[f"c{c}_idx"], z[f"c{c}_m"])
        duals = P.MultiDual(tuple(z[f"c{c}_f{q}"] for q in range(kk)))
        pc = P.plan_cost(plan, inputs, costfn)
        assert pc == pytest.approx(float(z[f"c{c}_pc"]), rel=1e-12, abs=1e-14)
        for key, d in (("cert", duals),
                       ("bad", P.MultiDual(tuple(p + (0.01 if q == 0 else 0.0)
                                                 for q, p in enumerate(duals.potentials))))):
            cert = P.mot_certificate(inputs, None, plan, d, costfn=costfn)
            ref = z[f"c{c}_{key}"]
            scale = 1.0 + abs(ref[0])
            assert cert.primal == pytest.approx(ref[0], rel=1e-12, abs=1e-14)
            assert cert.dual == pytest.approx(ref[1], rel=1e-12, abs=1e-14)
            assert abs(cert.gap - ref[2]) <= 1e-12 * scale
            assert abs(cert.feasibility_violation - ref[3]) <= 1e-12 * scale
            assert bool(cert.passed) == bool(ref[4]), (c, key)
        dfe = float(z[f"c{c}_dfe"])
        if np.isfinite(dfe):
            bad = P.MultiDual(tuple(p + (0.01 if q == 0 else 0.0)
                                    for q, p in enumerate(duals.potentials)))
            got = P.dual_feasibility_exhaustive(inputs, bad, costfn)
            assert got == pytest.approx(dfe, rel=1e-12, abs=1e-14)


@pytest.mark.parametrize("name", ["pow15", "spread"])
def test_custom_cost_vs_oracle_ragged(name):
    """K = 6 ragged lists (up to 300 atoms, zero weights) vs the oracle's
    restatement of the sweep loop."""
    rng = np.random.default_rng(91 if name == "pow15" else 92)
    xs, ws = [], []
    for _q in range(6):
        n = int(rng.integers(150, 301))
        w = rng.exponential(1.0, n)
        w[rng.random(n) < 0.08] = 0.0
        w *= 2.5 / w.sum()
        xs.append(np.sort(rng.normal(0.0, 1.0, n)))
        ws.append(w)
    costfn = {"pow15": pairwise_pow15, "spread": spread}[name]
    inputs = [P.DiscreteMeasure(x, w) for x, w in zip(xs, ws)]
    plan, duals = P.solve_mot_1d(inputs, costfn=costfn)
    ii, mm, pots = O.solve_mot_1d_custom(xs, ws, costfn)
    np.testing.assert_array_equal(plan.indices, ii)
    np.testing.assert_allclose(plan.mass, mm, rtol=0, atol=1e-13 * 2.5)
    scale = max(1.0, max(np.abs(p).max() for p in pots))
    for q in range(6):
        assert np.abs(duals.potentials[q] - pots[q]).max() <= 1e-11 * scale


def test_custom_barycentric_equals_builtin():
    """The barycentric cost passed as an anonymous callable takes the
    custom-cost path and must reproduce the fused barycentric sweep."""
    from paper_2201_00730_b200 import synthetic as S

    xs, ws = S.cfg5_batch(count=1, n=300)
    ws = ws / ws.sum(axis=2, keepdims=True)
    w = np.full(16, 1 / 16)
    inputs = [P.DiscreteMeasure(xs[0, q], ws[0, q]) for q in range(16)]
    p1, d1 = P.solve_mot_1d(inputs, w)
    p2, d2 = P.solve_mot_1d(inputs, costfn=plain_barycentric(w))
    np.testing.assert_array_equal(p1.indices, p2.indices)
    np.testing.assert_array_equal(p1.mass, p2.mass)
    scale = max(np.abs(p).max() for p in d1.potentials)
    for q in range(16):
        assert np.abs(d1.potentials[q] - d2.potentials[q]).max() <= 1e-12 * scale


def test_custom_cost_mass_balance_error():
    inputs = [P.DiscreteMeasure([0.0, 1.0], [0.5, 0.5]), P.DiscreteMeasure([0.5], [2.0])]
    with pytest.raises(P.MassBalanceError):
        P.solve_mot_1d(inputs, costfn=spread)
