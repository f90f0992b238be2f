"""GPU parity of the non-KL dual functionals and Frank-Wolfe (Berg and mixed
KL/Berg penalties; csrc/fw1d_generic.cu, csrc/dense.cu) against the
reference (tests/golden/berg.npz): the bracketed-Newton translation
(src/duality.py:182-247, residual 1e-11), updated marginals, F / G / H,
the primal with the Berg divergence, fixed-iteration FW traces and the
reference's own fw_solve report on tests/test_fw.py:121-125's instance."""

import numpy as np
import pytest

import paper_2201_00730_b200 as P
from conftest import golden, rel_err
from paper_2201_00730_b200 import _device as D
from paper_2201_00730_b200 import duality as PD
from paper_2201_00730_b200 import fw as F

pytestmark = pytest.mark.gpu


def _ent(code, rho):
    return P.KL(float(rho)) if int(code) == 0 else P.Berg(float(rho))


def _dprob(z, k, eps=0.0):
    e = z[f"d{k}_ent"]
    return P.UotProblem(P.DiscreteMeasure(z[f"d{k}_x"], z[f"d{k}_a"]),
                        P.DiscreteMeasure(z[f"d{k}_y"], z[f"d{k}_b"]), P.PowerDistance(2.0),
                        _ent(e[0], e[1]), _ent(e[2], e[3]), eps=eps)


@pytest.mark.parametrize("k", range(4))
def test_translation_marginals_and_values(k):
    z = golden("berg.npz")
    prob = _dprob(z, k)
    d = P.DualPair(z[f"d{k}_f"], z[f"d{k}_g"])
    lam = P.lambda_star(prob, d)
    # both solves stop at |residual| < 1e-11 on a slope of O(mass / rho)
    assert lam == pytest.approx(float(z[f"d{k}_lam"]), abs=1e-10)
    ta, tb = P.updated_marginals(prob, d)
    np.testing.assert_allclose(ta, z[f"d{k}_ta"], rtol=1e-9, atol=1e-14)
    np.testing.assert_allclose(tb, z[f"d{k}_tb"], rtol=1e-9, atol=1e-14)
    assert ta.sum() == pytest.approx(tb.sum(), rel=1e-9)  # tests/test_duality.py:102-107
    dfs = P.DualPair(z[f"d{k}_fs"], z[f"d{k}_g"])
    assert PD.eval_F(prob, dfs) == pytest.approx(float(z[f"d{k}_F"]), rel=1e-12, abs=1e-14)
    assert PD.eval_G(prob, dfs, 0.07) == pytest.approx(float(z[f"d{k}_G"]), rel=1e-12, abs=1e-14)
    assert PD.eval_H(prob, dfs) == pytest.approx(float(z[f"d{k}_H"]), rel=1e-10, abs=1e-12)
    pe = _dprob(z, k, eps=0.3)
    assert PD.eval_F(pe, d) == pytest.approx(float(z[f"d{k}_Feps"]), rel=1e-12, abs=1e-14)
    plan = P.SparsePlan(z[f"d{k}_pi"], z[f"d{k}_pj"], z[f"d{k}_pm"])
    assert P.eval_primal(prob, plan) == pytest.approx(float(z[f"d{k}_primal"]), rel=1e-12)
    assert P.eval_primal(pe, plan) == pytest.approx(float(z[f"d{k}_primal_eps"]), rel=1e-12)


def test_newton_errors_and_balanced_rejection():
    a = P.DiscreteMeasure([0.0, 1.0], [0.5, 0.5])
    prob = P.UotProblem(a, a, P.PowerDistance(2.0), P.Berg(1.0), P.Berg(1.0), eps=0.0)
    with pytest.raises(P.NewtonError):  # -rho1 - min f >= rho2 + min g (duality.py:187-190)
        P.lambda_star(prob, P.DualPair(np.full(2, -2.0), np.full(2, -2.0)))
    pb = P.UotProblem(a, a, P.PowerDistance(2.0), P.Berg(1.0), P.Balanced(), eps=0.0)
    with pytest.raises(P.UnsupportedEntropyError):
        P.lambda_star(pb, P.DualPair.zeros(2, 2))
    with pytest.raises(P.UnsupportedEntropyError):
        P.fw_solve(pb)


def test_berg_divergence_infinities():
    """Berg(mu | nu) is +inf where mu vanishes on nu's support
    (src/entropies.py:132-137)."""
    a = P.DiscreteMeasure([0.0, 1.0], [0.5, 0.5])
    prob = P.UotProblem(a, a, P.PowerDistance(2.0), P.Berg(1.0), P.KL(1.0), eps=0.0)
    plan = P.SparsePlan(np.array([0]), np.array([0]), np.array([1.0]))
    assert P.eval_primal(prob, plan) == np.inf


@pytest.mark.parametrize("k", range(4))
def test_berg_fw_fixed_iterations(k):
    z = golden("berg.npz")
    e1c, r1, e2c, r2, iters, ls = z[f"w{k}_par"]
    ent = {0: "kl", 1: "berg"}
    step = "linesearch" if ls else "harmonic"
    r = F.fw_solve_batched(z[f"w{k}_x"], z[f"w{k}_y"], z[f"w{k}_a"], z[f"w{k}_b"], float(r1),
                           float(r2), 2.0, int(iters), step, ent1=ent[int(e1c)],
                           ent2=ent[int(e2c)])
    assert int(r.status[0].item()) == 0
    assert int(r.iterations[0].item()) == int(iters)
    h0, ref_h0 = D.to_np(r.h0[0]), z[f"w{k}_h0"]
    scale = np.abs(ref_h0).max()
    np.testing.assert_allclose(h0, ref_h0, rtol=1e-9, atol=1e-12 * scale)
    np.testing.assert_allclose(D.to_np(r.pd_gap[0]), z[f"w{k}_pd_gap"], rtol=0,
                               atol=4e-9 * scale)
    np.testing.assert_allclose(D.to_np(r.fw_gap[0]), z[f"w{k}_fw_gap"], rtol=0,
                               atol=4e-9 * scale)
    err = rel_err(D.to_np(r.f[0]), D.to_np(r.g[0]), z[f"w{k}_f"], z[f"w{k}_g"])
    assert err < (1e-9 if step == "harmonic" else 1e-6), err
    if err < 1e-12:
        c = int(r.count[0].item())
        np.testing.assert_array_equal(D.to_np(r.ei[0, :c]), z[f"w{k}_i"])
        np.testing.assert_array_equal(D.to_np(r.ej[0, :c]), z[f"w{k}_j"])


def test_berg_fw_solve_report():
    """tests/test_fw.py:121-125 on the reference's own run: early exit at the
    same iteration, certificate passes, final translated pair agrees."""
    z = golden("berg.npz")
    prob = P.UotProblem(P.DiscreteMeasure(z["e_x"], z["e_a"]), P.DiscreteMeasure(z["e_y"], z["e_b"]),
                        P.PowerDistance(2.0), P.Berg(1.0), P.Berg(1.0), eps=0.0)
    rep = P.fw_solve(prob, P.FwConfig("linesearch", 3000, 1e-7))
    assert rep.certificate.passed == bool(z["e_passed"])
    assert rep.iterations == int(z["e_iters"])
    np.testing.assert_allclose(rep.trace["h0"], z["e_h0"], rtol=1e-9, atol=1e-12)
    assert rel_err(rep.final.f, rep.final.g, z["e_f"], z["e_g"]) < 1e-6


def test_berg_line_search_and_batched_equals_single():
    z = golden("berg.npz")
    e1c, r1, e2c, r2, iters, ls = z["w0_par"]
    args = [z[f"w0_{s}"] for s in "xyab"]
    rs = F.fw_solve_batched(*args, float(r1), float(r2), 2.0, 10, "linesearch", ent1="berg",
                            ent2="berg")
    rb = F.fw_solve_batched(*(np.stack([v, v, v]) for v in args), float(r1), float(r2), 2.0, 10,
                            "linesearch", ent1="berg", ent2="berg")
    for q in range(3):
        assert np.array_equal(D.to_np(rb.f[q]), D.to_np(rs.f[0]))
        assert np.array_equal(D.to_np(rb.h0[q]), D.to_np(rs.h0[0]))
    # the public single-step line search agrees with the in-kernel one at t = 0
    prob = P.UotProblem(P.DiscreteMeasure(args[0], args[2]), P.DiscreteMeasure(args[1], args[3]),
                        P.PowerDistance(2.0), P.Berg(float(r1)), P.Berg(float(r2)), eps=0.0)
    d0 = P.DualPair.zeros(len(args[0]), len(args[1]))
    ta, tb = P.updated_marginals(prob, d0)
    _, atom = P.solve_ot_1d(P.DiscreteMeasure(args[0], ta), P.DiscreteMeasure(args[1], tb))
    gm = F.line_search_h0(prob, d0, atom)
    assert gm == pytest.approx(float(rs.step_size[0, 0].item()), abs=1e-9)


@pytest.mark.parametrize("k", range(3))
def test_berg_pairwise_report(k):
    """Pairwise FW with Berg / mixed penalties (src/fw.py:326-357) against the
    reference's own report: same early exit (+-1 at a 1e-10 gap), the H0 trace
    while one atom is active, final translated pair and certificate."""
    z = golden("berg_pfw.npz")
    c1, r1, c2, r2, iters = z[f"c{k}_par"]
    prob = P.UotProblem(P.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"]),
                        P.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"]), P.PowerDistance(2.0),
                        _ent(c1, r1), _ent(c2, r2), eps=0.0)
    rep = P.fw_solve(prob, P.FwConfig("pairwise", int(iters), 1e-10))
    ref_h0 = z[f"c{k}_h0"]
    assert abs(rep.iterations - len(ref_h0)) <= 1
    np.testing.assert_allclose(rep.trace["h0"][:2], ref_h0[:2], rtol=1e-9, atol=1e-13)
    assert rep.certificate.passed == bool(z[f"c{k}_passed"])
    assert rel_err(rep.final.f, rep.final.g, z[f"c{k}_f"], z[f"c{k}_g"]) < 1e-6


@pytest.mark.parametrize("method", ["fw-ls", "fw", "pfw"])
def test_cli_uot1d_berg(tmp_path, capsys, method):
    """uot1d --entropy berg through the CLI: exit code and certificate as the
    reference's CLI prints them on the same generated inputs."""
    import json

    from paper_2201_00730_b200 import cli

    z = golden("berg_pfw.npz")
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(["gen", "--n", "12", "--seed", "5", "--out", str(a)]) == 0
    assert cli.main(["gen", "--n", "10", "--seed", "6", "--out", str(b)]) == 0
    capsys.readouterr()
    rc = cli.main(["uot1d", str(a), str(b), "--entropy", "berg", "--method", method, "--gap-tol",
                   "1e-7", "--max-iters", "3000", "--out", str(tmp_path / "o.json")])
    assert rc == int(z[f"cli_{method}_rc"])
    got = json.loads(capsys.readouterr().out.splitlines()[0])
    want = json.loads(bytes(z[f"cli_{method}_cert"]).decode())
    assert got["passed"] == want["passed"]
    assert got["primal"] == pytest.approx(want["primal"], rel=1e-6)
    assert got["dual"] == pytest.approx(want["dual"], rel=1e-6)


def test_berg_fw_edges_and_ragged_early_exit():
    """Single atoms, zero-weight atoms, and a batch whose problems stop at
    different iterations (per-problem done flags, host check every 16)."""
    rng = np.random.default_rng(77)
    one = F.fw_solve_batched([0.2], [0.7], [1.0], [0.5], 1.0, 0.7, 2.0, 50, "linesearch",
                             gap_tol=1e-10, early_exit=True, ent1="berg", ent2="berg")
    assert int(one.status[0].item()) == 0 and int(one.count[0].item()) == 1
    B, n, m = 5, 30, 24
    x = np.sort(rng.uniform(0, 1, (B, n)), axis=1)
    y = np.sort(rng.uniform(0, 1, (B, m)), axis=1)
    a = rng.uniform(0.1, 1, (B, n))
    a[:, ::6] = 0.0
    b = rng.uniform(0.1, 1, (B, m)) * rng.uniform(0.3, 3.0, (B, 1))
    rb = F.fw_solve_batched(x, y, a, b, 0.8, 1.3, 2.0, 200, "harmonic", gap_tol=1e-4,
                            early_exit=True, ent1="kl", ent2="berg")
    its = D.to_np(rb.iterations)
    assert len(set(its.tolist())) > 1  # ragged stop
    for q in range(B):
        rs = F.fw_solve_batched(x[q], y[q], a[q], b[q], 0.8, 1.3, 2.0, 200, "harmonic",
                                gap_tol=1e-4, early_exit=True, ent1="kl", ent2="berg")
        assert int(rs.iterations[0].item()) == its[q]
        assert np.array_equal(D.to_np(rs.f[0]), D.to_np(rb.f[q]))
        assert D.to_np(rb.pd_gap[q, its[q] - 1]) < 1e-4
        assert np.all(D.to_np(rb.em[q, :int(rb.count[q].item())]) > 0)


def test_lambda_star_tolerance_arguments():
    """lambda_star(prob, d, tol, max_iters, initial) (src/duality.py:160):
    the stopping rule is the caller's; too few Newton steps raise."""
    z = golden("berg.npz")
    prob = _dprob(z, 0)
    d = P.DualPair(z["d0_f"], z["d0_g"])
    tight = P.lambda_star(prob, d)
    loose = P.lambda_star(prob, d, tol=1e-2)
    assert abs(loose - tight) < 0.1
    assert P.lambda_star(prob, d, initial=tight) == pytest.approx(tight, abs=1e-10)
    with pytest.raises(P.NewtonError):
        P.lambda_star(prob, d, tol=1e-300, max_iters=1)


@pytest.mark.parametrize("k", range(2))
def test_berg_fw_explicit_cost(k):
    """Explicit (negative-entry) Monge costs with Berg / mixed penalties on the
    generic FW path: the oracle reads C(i, j), the primal's transport cost
    too; h0 trace and final pair vs the reference's fixed-iteration loop."""
    z = golden("berg_pfw.npz")
    c1, r1, c2, r2, ls = z[f"x{k}_par"]
    ent = {0: "kl", 1: "berg"}
    step = "linesearch" if ls else "harmonic"
    r = F.fw_solve_batched(z[f"x{k}_x"], z[f"x{k}_y"], z[f"x{k}_a"], z[f"x{k}_b"], float(r1),
                           float(r2), 2.0, 30, step, f0=z[f"x{k}_f0"], g0=z[f"x{k}_g0"],
                           C=z[f"x{k}_C"], ent1=ent[int(c1)], ent2=ent[int(c2)])
    assert int(r.status[0].item()) == 0
    ref_h0 = z[f"x{k}_h0"]
    np.testing.assert_allclose(D.to_np(r.h0[0]), ref_h0, rtol=1e-9,
                               atol=1e-12 * np.abs(ref_h0).max())
    err = rel_err(D.to_np(r.f[0]), D.to_np(r.g[0]), z[f"x{k}_f"], z[f"x{k}_g"])
    assert err < (1e-9 if step == "harmonic" else 1e-6), err


@pytest.mark.parametrize("k", range(2))
def test_berg_fw_explicit_newton_error_like_reference(k):
    """With the unscaled negative cost the half-minima init can leave the Berg
    translation domain empty: fw_solve raises NewtonError exactly when the
    reference does (src/duality.py:187-190)."""
    z = golden("berg_pfw.npz")
    c1, r1, c2, r2, ls = z[f"x{k}_par"]
    prob = P.UotProblem(P.DiscreteMeasure(z[f"x{k}_x"], z[f"x{k}_a"]),
                        P.DiscreteMeasure(z[f"x{k}_y"], z[f"x{k}_b"]),
                        P.ExplicitMatrix(z[f"x{k}_Cbig"]), _ent(c1, r1), _ent(c2, r2), eps=0.0)
    cfg = P.FwConfig("linesearch" if ls else "harmonic", 5, 1e-12)
    if bool(z[f"x{k}_big_newton_error"]):
        with pytest.raises(P.NewtonError):
            P.fw_solve(prob, cfg)
    else:
        assert P.fw_solve(prob, cfg).iterations >= 1
