"""Parity at the full BASELINE sizes against fixtures the
fp64 oracle computed at those sizes (tests/golden/make_scale.py; the oracle
is pinned to the reference's own outputs in test_oracle_golden.py):

* cfg3: one problem N = M = 65536, d = 2, 200 H iterations (src/sinkhorn.py:
  137-163) in fp32 -- raw potentials, lambda*-translated potentials and the
  dual objective H (src/duality.py:256-290 with the eps term :124-132) within
  1e-4 * eps absolute.
* cfg4: problems 0 and 1 of the seeded B = 256 batch, N = M = 4096, d = 64,
  300 H iterations through the tcgen05 path -- same bar.
* cfg5: problems 0 and 1 of the seeded 64-problem batch, K = 16, N = 8192,
  200 barycenter FW iterations (src/barycenter.py:361-411): harmonic steps
  and the line search with the reference's gamma_t replayed -- every
  iteration's plan support bit-exact (hash + entry count), H_0 and the
  potentials to 1e-9 relative; the production Newton line search's measured
  deviation is asserted separately.
* cfg5 without the density floor: the K-marginal sweep against the oracle,
  every support mismatch reported with its breakpoint gap.

Inputs are regenerated from the seeded generators (synthetic.py)."""

import numpy as np
import pytest

import oracle as O
import paper_2201_00730_b200 as P
from conftest import golden
from paper_2201_00730_b200 import _device as D
from paper_2201_00730_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _dual_h(x, y, a, b, f, g, eps, rho):
    """eval_H of the pair, evaluated on the device in fp64 (uot_sinkhorn_verify:
    eps-term log-sum and both softmins, two on-the-fly passes)."""
    out = P.verify_batched(x[None], y[None], a[None], b[None], f[None], g[None], eps, rho, rho,
                           precision="fp64")
    o = D.to_np(out[0], readonly=False)
    ma, mb = float(a.sum()), float(b.sum())
    la, lb = -o[5] / rho, -o[6] / rho  # LSE_a(-f/rho), LSE_b(-g/rho)
    return (rho * ma + rho * mb - 2 * rho * np.exp(0.5 * la + 0.5 * lb)
            - eps * (np.exp(o[1]) - ma * mb))


def _check_sinkhorn_fp32(x, y, a, b, eps, rho, f, g, ref_f, ref_g, ref_dual, tag):
    tol = 1e-4 * eps
    f = f.astype(np.float64)
    g = g.astype(np.float64)
    raw = max(np.abs(f - ref_f).max(), np.abs(g - ref_g).max())
    lam = O.lambda_star_kl(a, b, f, g, rho, rho)
    lam_r = O.lambda_star_kl(a, b, ref_f, ref_g, rho, rho)
    tr = max(np.abs(f + lam - ref_f - lam_r).max(), np.abs(g - lam - ref_g + lam_r).max())
    dual = _dual_h(x, y, a, b, f, g, eps, rho)
    print(f"{tag}: raw {raw:.3e}  translated {tr:.3e}  dual {abs(dual - ref_dual):.3e}  "
          f"(tol {tol:.3e})")
    assert raw <= tol, (tag, "raw", raw, tol)
    assert tr <= tol, (tag, "translated", tr, tol)
    assert abs(dual - ref_dual) <= tol, (tag, "dual", dual, ref_dual)


def test_cfg3_full_size_200_iterations_fp32():
    z = golden("cfg3_full.npz")
    c = S.cfg3_inputs()
    assert abs(c.eps - float(z["eps"])) == 0.0
    for iters, fk, gk in ((1, "f1", "g1"), (200, "f", "g")):
        f, g, _, its = P.sinkhorn_batched(c.x[None], c.y[None], c.alpha[None], c.beta[None],
                                          c.eps, c.rho, c.rho, iters, precision="fp32")
        assert int(its[0].item()) == iters
        f, g = D.to_np(f[0]), D.to_np(g[0])
        if iters == 200:
            _check_sinkhorn_fp32(c.x, c.y, c.alpha, c.beta, c.eps, c.rho, f, g, z["f"], z["g"],
                                 float(z["dual"]), "cfg3 200 it")
        else:
            err = max(np.abs(f - z[fk]).max(), np.abs(g - z[gk]).max())
            print(f"cfg3 {iters} it: raw {err:.3e}")
            assert err <= 1e-4 * c.eps, (iters, err)


def test_cfg4_full_size_300_iterations_tcgen05():
    z = golden("cfg4_full.npz")
    probs = [int(p) for p in z["problems"]]
    x, y, a, b = S.cfg4_batch(start=0, count=max(probs) + 1)
    eps, rho = float(z["eps"]), float(z["rho"])
    f, g, _, its = P.sinkhorn_batched(x, y, a, b, eps, rho, rho, int(z["iters"]),
                                      precision="fp32")
    for p in probs:
        assert int(its[p].item()) == int(z["iters"])
        _check_sinkhorn_fp32(x[p], y[p], a[p], b[p], eps, rho, D.to_np(f[p]), D.to_np(g[p]),
                             z[f"p{p}_f"], z[f"p{p}_g"], float(z[f"p{p}_dual"]), f"cfg4 p{p}")


def _cfg5_check(r, z, probs, mode, pot_tol):
    for i, p in enumerate(probs):
        tag = f"p{p}_{mode}"
        hs, nz = D.to_np(r.supp_hash[i]), D.to_np(r.supp_nnz[i])
        bad = np.nonzero((hs != z[f"{tag}_supp_hash"]) | (nz != z[f"{tag}_nnz"]))[0]
        assert bad.size == 0, f"{tag}: support differs at iterations {bad[:10]}"
        np.testing.assert_allclose(D.to_np(r.h0[i]), z[f"{tag}_h0"], rtol=1e-9, atol=0)
        f = D.to_np(r.f[i])
        ref8 = z[f"{tag}_pots8"]
        scale = np.abs(ref8).max()
        err = np.abs(f[:, ::8] - ref8).max() / scale
        serr = np.abs(f.sum(axis=1) - z[f"{tag}_potsum"]).max() / (scale * f.shape[1])
        print(f"cfg5 {tag}: potentials {err:.2e}, sums {serr:.2e} (relative)")
        assert err <= pot_tol and serr <= pot_tol, (tag, err, serr)


@pytest.mark.parametrize("mode", ["h", "l"])
def test_cfg5_full_size_200_iterations(mode):
    z = golden("cfg5_full.npz")
    probs = [int(p) for p in z["problems"]]
    xs, ws = S.cfg5_batch(start=0, count=max(probs) + 1)
    w = np.full(16, 1 / 16)
    iters = int(z["iters"])
    step_in = None
    if mode == "l":  # the reference's gamma_t replayed (make_scale.py recorded them)
        step_in = np.stack([z[f"p{p}_l_gamma"] for p in probs])
    r = P.fw_barycenter_batched(xs[probs], ws[probs], w, 1.0, iters,
                                "harmonic" if mode == "h" else "linesearch", step_in=step_in,
                                trace_support=True)
    assert (D.to_np(r.status) == 0).all()
    _cfg5_check(r, z, probs, mode, 1e-9)


def test_cfg5_full_size_newton_line_search_deviation():
    """Production step rule (safeguarded Newton) vs the reference's ternary
    search at cfg5 scale: the objective trace agrees to 1e-9; the
    potentials carry the ternary search's gamma resolution."""
    z = golden("cfg5_full.npz")
    xs, ws = S.cfg5_batch(start=0, count=1)
    r = P.fw_barycenter_batched(xs, ws, np.full(16, 1 / 16), 1.0, int(z["iters"]), "linesearch")
    np.testing.assert_allclose(D.to_np(r.h0[0]), z["p0_l_h0"], rtol=1e-9, atol=0)
    f = D.to_np(r.f[0])
    ref8 = z["p0_l_pots8"]
    err = np.abs(f[:, ::8] - ref8).max() / np.abs(ref8).max()
    print(f"cfg5 Newton vs ternary: potentials {err:.2e} relative")
    assert err <= 1e-6


def test_cfg5_unfloored_sweep_mismatch_report():
    """solve_mot_1d at full cfg5 size on UNFLOORED mixture densities (atoms
    down to ~1e-33): the device merge and the oracle's sequential sweep may
    order breakpoints that coincide to within rounding differently.  Every
    mismatch is reported with its breakpoint gap; the bar is that each
    mismatch sits at a near-tie (gap <= 1e-12 of the mass) and moves no more
    mass than that."""
    xs, ws = S.cfg5_batch(start=0, count=2, floor=0.0)
    ws = ws / ws.sum(axis=2, keepdims=True)
    w = np.full(16, 1 / 16)
    _, idx, mass, count, status = P.solve_mot_1d_batched(xs, ws, w)
    assert (D.to_np(status) == 0).all()
    for p in range(2):
        c = int(count[p].item())
        di = D.to_np(idx[p, :c]).astype(np.int64)
        dm = D.to_np(mass[p, :c])
        oi, om, _ = O.solve_mot_1d(list(xs[p]), list(ws[p]), w)
        cums = [np.cumsum(ws[p, q]) for q in range(16)]
        rep = O.mot_mismatch_report(di, dm, oi, om, cums)
        print(f"cfg5 unfloored problem {p}: {rep}")
        assert rep["max_gap_rel"] <= 1e-12, rep
        assert rep["mass_moved"] <= 1e-12, rep
