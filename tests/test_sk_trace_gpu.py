"""run(..., reference=) error traces for penalties off the KL closed form
(src/sinkhorn.py:246-315) vs the reference (tests/golden/sk_trace.npz): F
with Berg / Balanced marginals (untranslated iterates) and G with a Berg
marginal (translated by the Newton lambda*, csrc/fw1d_generic.cu)."""

import numpy as np
import pytest

import paper_2201_00730_b200 as P
from conftest import golden

pytestmark = pytest.mark.gpu


def _ent(code, rho):
    return [P.KL, P.Berg, None][int(code)](float(rho)) if int(code) < 2 else P.Balanced()


@pytest.mark.parametrize("k", range(4))
def test_error_traces_match_reference(k):
    z = golden("sk_trace.npz")
    var, c1, r1, c2, r2 = z[f"c{k}_par"]
    variant = "f" if int(var) == 0 else "g"
    prob = P.UotProblem(P.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"]),
                        P.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"]), P.PowerDistance(2.0),
                        _ent(c1, r1), _ent(c2, r2), eps=0.2)
    ref = P.DualPair(z[f"c{k}_ref_f"], z[f"c{k}_ref_g"])
    rep = P.run(prob, P.SinkhornConfig(variant, 25, 1e-15), reference=ref)
    # the stopping test sits at delta ~ 1e-15 (rounding): compare the common prefix
    want = z[f"c{k}_err_f"]
    L = min(len(want), rep.iterations)
    assert abs(len(want) - rep.iterations) <= 3
    for key in ("delta_f", "err_f", "err_g"):
        np.testing.assert_allclose(rep.trace[key][:L], z[f"c{k}_{key}"][:L], rtol=1e-8, atol=1e-11,
                                   err_msg=key)


def _sprob(z, k):
    c1, r1, c2, r2 = z[f"s{k}_par"]
    return P.UotProblem(P.DiscreteMeasure(z[f"s{k}_x"], z[f"s{k}_a"]),
                        P.DiscreteMeasure(z[f"s{k}_y"], z[f"s{k}_b"]), P.PowerDistance(2.0),
                        _ent(c1, r1), _ent(c2, r2), eps=0.15)


@pytest.mark.parametrize("k", range(3))
def test_g_step_at_given_lambda_berg(k):
    """g_sinkhorn_step(prob, d, lam) with Berg marginals (src/sinkhorn.py:117-134):
    the device G run starts from the given lam (descriptor lam_given)."""
    z = golden("sk_trace.npz")
    prob = _sprob(z, k)
    pair, lam1 = P.g_sinkhorn_step(prob, P.DualPair(z[f"s{k}_f0"], z[f"s{k}_g0"]), 0.13)
    np.testing.assert_allclose(pair.f, z[f"s{k}_f1"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(pair.g, z[f"s{k}_g1"], rtol=0, atol=1e-12)
    assert lam1 == pytest.approx(float(z[f"s{k}_lam1"]), abs=1e-10)


@pytest.mark.parametrize("k", range(3))
def test_anderson_g_berg_traces(k):
    """Anderson-accelerated G (src/sinkhorn.py:281-292) with a Berg marginal:
    the carried lambda is the Newton translation of the stepped pair."""
    z = golden("sk_trace.npz")
    prob = _sprob(z, k)
    ref = P.DualPair(z[f"s{k}_ref_f"], z[f"s{k}_ref_g"])
    rep = P.run(prob, P.SinkhornConfig("g", 12, 1e-15, anderson=P.AndersonConfig(3, 1e-9)),
                reference=ref)
    for key in ("delta_f", "err_f", "err_g"):
        np.testing.assert_allclose(rep.trace[key], z[f"s{k}_and_{key}"], rtol=1e-7, atol=1e-11,
                                   err_msg=key)
    np.testing.assert_allclose(rep.final.f, z[f"s{k}_and_f"], rtol=0, atol=1e-10)


def test_g_sinkhorn_berg_newton_error_like_reference():
    """an empty Berg translation domain (src/duality.py:188-189)
    raises NewtonError from the device G run exactly where the reference
    raises it (checked against uotkit in the build container: Berg/Berg with
    f0 = g0 = -3 raises, Berg/KL from the same start runs)."""
    x = np.linspace(0, 1, 20)
    a, b = np.full(20, 0.05), np.full(20, 0.06)
    init = P.DualPair(np.full(20, -3.0), np.full(20, -3.0))
    prob = P.UotProblem(P.DiscreteMeasure(x, a), P.DiscreteMeasure(x, b), P.PowerDistance(2.0),
                        P.Berg(1.0), P.Berg(1.0), eps=0.05)
    with pytest.raises(P.NewtonError, match="empty translation domain"):
        P.run(prob, P.SinkhornConfig("g", 10, 1e-12), init=init)
    prob = P.UotProblem(P.DiscreteMeasure(x, a), P.DiscreteMeasure(x, b), P.PowerDistance(2.0),
                        P.Berg(1.0), P.KL(1.0), eps=0.05)
    rep = P.run(prob, P.SinkhornConfig("g", 10, 1e-12), init=init)
    assert np.isfinite(rep.final.f).all() and np.isfinite(rep.final.g).all()
