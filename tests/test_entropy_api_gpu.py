"""Entropy-family functions (logdotexp, softmin, conj / conj_grad / conj_hess,
aprox, divergence) and the FW single-step API (line_search_h0, pfw_step) on
the device, against the reference's own values (tests/golden/entropy_api.npz)."""

import math

import numpy as np
import pytest

import paper_2201_00730_b200 as P
from conftest import golden
from paper_2201_00730_b200 import entropies as E
from paper_2201_00730_b200 import fw as F

pytestmark = pytest.mark.gpu


def test_logdotexp_and_softmin():
    z = golden("entropy_api.npz")
    assert E.logdotexp(z["v"], z["w"]) == pytest.approx(float(z["lde_flat"]), rel=1e-14)
    np.testing.assert_allclose(E.logdotexp(z["M"], z["w"], axis=1), z["lde_ax1"], rtol=1e-14)
    np.testing.assert_allclose(E.logdotexp(z["M0"], z["w"], axis=0), z["lde_ax0"], rtol=1e-14)
    assert E.logdotexp(z["v"], np.zeros(40)) == -math.inf == float(z["lde_zero"])
    A = P.DiscreteMeasure(np.arange(40.0), z["aw"])
    assert E.softmin(A, 0.3, z["v"]) == pytest.approx(float(z["softmin"]), rel=1e-14)
    with pytest.raises(ValueError):
        E.softmin(A, 0.0, z["v"])


@pytest.mark.parametrize("name", ["kl", "berg", "bal"])
def test_conjugates_aprox_divergence(name):
    z = golden("entropy_api.npz")
    sp = {"kl": P.KL(1.7), "berg": P.Berg(2.5), "bal": P.Balanced()}[name]
    x = z[f"{name}_x"]
    np.testing.assert_allclose(E.conj(sp, x), z[f"{name}_conj"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(E.conj_grad(sp, x), z[f"{name}_grad"], rtol=1e-14)
    np.testing.assert_allclose(E.conj_hess(sp, x), z[f"{name}_hess"], rtol=1e-14)
    # Berg: both sides stop the Newton solve at |h(y)| < 1e-12 (entropies.py:247-263)
    np.testing.assert_allclose(E.aprox(sp, 0.2, x), z[f"{name}_aprox"], rtol=1e-12, atol=1e-11)
    for key, mu in (("div", z[f"{name}_mu"]), ("div2", z[f"{name}_mu2"]), ("div_same", z[f"{name}_nu"])):
        ref = float(z[f"{name}_{key}"])
        got = E.divergence(sp, mu, z[f"{name}_nu"])
        if math.isinf(ref):
            assert math.isinf(got)
        else:
            assert got == pytest.approx(ref, rel=1e-13, abs=1e-15)
    assert isinstance(E.conj(sp, 0.5), float)
    if name == "berg":
        with pytest.raises(ValueError):
            E.conj(sp, 3.0)
        assert E.phi_prime_inf(sp) == 2.5
    else:
        assert E.phi_prime_inf(sp) == math.inf


def test_fw_single_steps():
    z = golden("entropy_api.npz")
    prob = P.UotProblem(P.DiscreteMeasure(z["fw_x"], z["fw_a"]), P.DiscreteMeasure(z["fw_y"], z["fw_b"]),
                        P.PowerDistance(2.0), P.KL(1.2), P.KL(0.8), eps=0.0)
    n, m = len(z["fw_x"]), len(z["fw_y"])
    cur = P.DualPair(np.zeros(n), np.zeros(m))
    ta, tb = P.updated_marginals(prob, cur)
    _, atom = P.solve_ot_1d(P.DiscreteMeasure(z["fw_x"], ta), P.DiscreteMeasure(z["fw_y"], tb),
                            P.PowerDistance(2.0))
    # ternary search on a flat maximum: resolves gamma to ~1e-6
    assert F.line_search_h0(prob, cur, atom) == pytest.approx(float(z["ls_gamma"]), abs=1e-6)
    # pairwise steps: the reference's ternary search stops ~1e-11 short of the
    # w_away endpoint and leaves dust atoms (weights ~1e-11) that ours drops,
    # and a dust atom can then be chosen as the away atom -- trajectories are
    # tie-sensitive by construction.  Steps 0-1 must match
    # the reference (iterate and non-dust weights); later steps keep the
    # invariants: convex weights and a non-decreasing dual value.
    store = F.AtomStore(np.zeros((1, n)), np.zeros((1, m)), np.array([1.0]))
    h_prev = -math.inf
    for it in range(4):
        store = F.pfw_step(prob, store)
        cur = store.current()
        assert abs(store.weights.sum() - 1.0) <= 1e-12 and (store.weights >= 0).all()
        h = F._h0_value(prob, cur.f, cur.g)
        assert h >= h_prev - 1e-12
        h_prev = h
        if it > 1:
            continue
        ref_w = z[f"pfw{it}_w"]
        ref_r = ref_w @ z[f"pfw{it}_r"]
        ref_s = ref_w @ z[f"pfw{it}_s"]
        scale = max(np.abs(ref_r).max(), np.abs(ref_s).max(), 1.0)
        assert np.abs(cur.f - ref_r).max() <= 1e-6 * scale, it
        assert np.abs(cur.g - ref_s).max() <= 1e-6 * scale, it
        np.testing.assert_allclose(np.sort(store.weights[store.weights > 1e-9]),
                                   np.sort(ref_w[ref_w > 1e-9]), atol=1e-6)


def test_fw_solve_reference_err_f_trace():
    """fw_solve(..., reference=pair) traces ||f_t + lambda*_t - ref.f||_inf
    (src/fw.py:217-219); harmonic steps so the trajectory is the reference's."""
    z = golden("entropy_api.npz")
    prob = P.UotProblem(P.DiscreteMeasure(z["fw_x"], z["fw_a"]), P.DiscreteMeasure(z["fw_y"], z["fw_b"]),
                        P.PowerDistance(2.0), P.KL(1.2), P.KL(0.8), eps=0.0)
    ref = P.DualPair(z["fw_ref_f"], z["fw_ref_g"])
    rep = P.fw_solve(prob, P.FwConfig("harmonic", 30, 1e-300), reference=ref)
    np.testing.assert_allclose(rep.trace["err_f"], z["fw_err_f"], rtol=1e-9, atol=1e-13)
