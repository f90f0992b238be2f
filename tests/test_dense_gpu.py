"""Dense / plan-level API helpers on the device (csrc/dense.cu) against the
reference's own values (tests/golden/dense.npz): build_cost_matrix,
cost_quadruple_diameter, birkhoff_rate_bound, updated_marginals, eval_primal."""

import numpy as np
import pytest

import paper_2201_00730_b200 as P
from conftest import golden

pytestmark = pytest.mark.gpu


def _case(z, k):
    A = P.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"])
    B = P.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"])
    r1, r2, eps = z[f"c{k}_par"]
    return A, B, float(z[f"c{k}_p"]), r1, r2, eps


def test_cost_matrix_diameter_and_rate_bound():
    z = golden("dense.npz")
    for k in range(int(z["ncases"])):
        A, B, p, r1, r2, eps = _case(z, k)
        C = P.build_cost_matrix(A, B, P.PowerDistance(p))
        np.testing.assert_allclose(C, z[f"c{k}_C"], rtol=1e-15, atol=1e-17)
        if p in (1.0, 2.0):  # the same arithmetic as numpy: bit-exact
            np.testing.assert_array_equal(C, z[f"c{k}_C"])
        assert P.cost_quadruple_diameter(C) == pytest.approx(float(z[f"c{k}_diam"]), rel=1e-14)
        prob = P.UotProblem(A, B, P.PowerDistance(p), P.KL(r1), P.KL(r2), eps=eps)
        assert P.birkhoff_rate_bound(prob) == pytest.approx(float(z[f"c{k}_birkhoff"]), rel=1e-13)


def test_updated_marginals():
    z = golden("dense.npz")
    for k in range(int(z["ncases"])):
        A, B, p, r1, r2, eps = _case(z, k)
        prob = P.UotProblem(A, B, P.PowerDistance(p), P.KL(r1), P.KL(r2), eps=0.0)
        ta, tb = P.updated_marginals(prob, P.DualPair(z[f"c{k}_f"], z[f"c{k}_g"]))
        np.testing.assert_allclose(ta, z[f"c{k}_ta"], rtol=1e-13)
        np.testing.assert_allclose(tb, z[f"c{k}_tb"], rtol=1e-13)


def test_eval_primal_sparse_dense_balanced_and_inf():
    z = golden("dense.npz")
    for k in range(int(z["ncases"])):
        A, B, p, r1, r2, eps = _case(z, k)
        plan = P.SparsePlan(z[f"c{k}_pi"], z[f"c{k}_pj"], z[f"c{k}_pm"])
        cost = P.PowerDistance(p)
        prob0 = P.UotProblem(A, B, cost, P.KL(r1), P.KL(r2), eps=0.0)
        prob = P.UotProblem(A, B, cost, P.KL(r1), P.KL(r2), eps=eps)
        probB = P.UotProblem(A, B, cost, P.Balanced(), P.KL(r2), eps=0.0)
        assert P.eval_primal(prob0, plan) == pytest.approx(float(z[f"c{k}_primal0"]), rel=1e-12)
        assert P.eval_primal(prob, plan) == pytest.approx(float(z[f"c{k}_primal_eps"]), rel=1e-12)
        assert P.eval_primal(prob, z[f"c{k}_dense"]) == pytest.approx(
            float(z[f"c{k}_primal_dense"]), rel=1e-12)
        assert P.eval_primal(probB, plan) == pytest.approx(float(z[f"c{k}_primal_bal"]), rel=1e-12)
        # explicit costs take the stored matrix
        probE = P.UotProblem(A, B, P.ExplicitMatrix(z[f"c{k}_C"]), P.KL(r1), P.KL(r2), eps=0.0)
        assert P.eval_primal(probE, plan) == pytest.approx(float(z[f"c{k}_primal0"]), rel=1e-12)
    x = np.linspace(0, 1, 5)
    A = P.DiscreteMeasure(x, [0.2, 0.0, 0.3, 0.2, 0.3])
    prob = P.UotProblem(A, A, P.PowerDistance(2.0), P.KL(1.0), P.KL(1.0), eps=0.0)
    assert P.eval_primal(prob, np.diag([0.2, 0.1, 0.3, 0.2, 0.2])) == float(z["inf_primal"])


def test_eval_primal_large_dense_plan():
    """Dense plans with many entries take the grid-parallel path (csrc/dense.cu:
    eval_primal_entries, marginals by fp64 atomics); checked against the formula
    of src/duality.py:320-344 written out in numpy."""
    rng = np.random.default_rng(4)
    n, m, eps, r1, r2 = 900, 1300, 0.07, 0.8, 1.7
    x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
    a, b = rng.exponential(1.0, n), rng.exponential(1.0, m)
    C = (x[:, None] - y[None, :]) ** 2
    plan = np.outer(a, b) * np.exp(-C / eps) * rng.uniform(0.5, 1.5, (n, m))
    prob = P.UotProblem(P.DiscreteMeasure(x, a), P.DiscreteMeasure(y, b), P.PowerDistance(2.0),
                        P.KL(r1), P.KL(r2), eps)

    def kl(p, q):
        return float(np.sum(p * np.log(p / q) - p + q))

    want = (float(np.sum(plan * C)) + eps * kl(plan, np.outer(a, b)) + r1 * kl(plan.sum(1), a)
            + r2 * kl(plan.sum(0), b))
    got = P.eval_primal(prob, plan)
    assert abs(got - want) <= 1e-11 * abs(want)
    big = np.ones((2048, 2048)) / 2048.0 ** 2
    u = np.linspace(0, 1, 2048)
    pb = P.UotProblem(P.DiscreteMeasure(u, np.full(2048, 1 / 2048)),
                      P.DiscreteMeasure(u, np.full(2048, 1 / 2048)), P.PowerDistance(2.0),
                      P.KL(1.0), P.KL(1.0), 0.0)
    v = P.eval_primal(pb, big)  # (the one-CTA kernel needed ~1 s here)
    assert v == pytest.approx(float(np.sum(big * (u[:, None] - u[None, :]) ** 2)), rel=1e-11)
