"""Anderson-extrapolated Sinkhorn on the device (csrc/anderson.cu) against
the reference's own run() with AndersonConfig (tests/golden/anderson.npz)
and the oracle window restatement.  fp64: 1e-9 relative on the final pair."""

import numpy as np
import pytest

import oracle as O
import paper_2201_00730_b200 as P
from conftest import cases, golden, rel_err
from paper_2201_00730_b200 import _device as D

pytestmark = pytest.mark.gpu


def test_anderson_weights_known_answers():
    """rtol 1e-7 as in the reference's own test (tests/test_sinkhorn.py:248):
    identical columns make U'U + rI ill-conditioned (cond ~ 1e8)."""
    z = golden("anderson.npz")
    for k in range(int(z["nwin"])):
        c = P.anderson_weights(z[f"w{k}_U"], float(z[f"w{k}_r"]))
        np.testing.assert_allclose(c, z[f"w{k}_c"], rtol=1e-7, atol=1e-12)
    assert P.anderson_weights(np.array([[1.0], [2.0]]), 1e-7).tolist() == [1.0]
    with pytest.raises(np.linalg.LinAlgError):
        P.anderson_weights(np.zeros((3, 2)), 0.0)


def _problem(z, k):
    p, eps, r1, r2, iters, depth, reg, var, ent = z[f"c{k}_par"]
    E = P.KL if ent == 0 else P.Berg
    prob = P.UotProblem(P.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"]),
                        P.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"]), P.PowerDistance(p), E(r1),
                        E(r2), eps=eps)
    return prob, "fhg"[int(var)], int(depth), reg


def test_anderson_runs_match_reference():
    z = golden("anderson.npz")
    for k in cases(z):
        prob, var, depth, reg = _problem(z, k)
        steps = len(z[f"c{k}_delta"])
        init = P.DualPair(z[f"c{k}_f0"], z[f"c{k}_g0"])
        rep = P.run(prob, P.SinkhornConfig(var, steps, 1e-300, P.AndersonConfig(depth, reg)),
                    init=init)
        assert rep.iterations == steps, (k, rep.iterations, steps)
        err = rel_err(rep.final.f, rep.final.g, z[f"c{k}_f"], z[f"c{k}_g"])
        assert err < 1e-9, (k, var, err)
        scale = max(np.abs(z[f"c{k}_f"]).max(), 1.0)
        np.testing.assert_allclose(rep.trace["delta_f"], z[f"c{k}_delta"], rtol=1e-6,
                                   atol=1e-11 * scale)


def test_anderson_no_worse_at_budget():
    """The reference's acceptance criterion 9 (tests/test_sinkhorn.py:260-271)
    on its own problem (mixture_measure(20, 55/56), KL(5), eps=0.1)."""
    z = golden("anderson.npz")
    prob, _, _, _ = _problem(z, 0)
    ref = P.run(prob, P.SinkhornConfig("f", 400000, 1e-13)).final
    plain = P.run(prob, P.SinkhornConfig("f", 200, 1e-16), reference=ref)
    accel = P.run(prob, P.SinkhornConfig("f", 200, 1e-16, P.AndersonConfig(4, 1e-7)),
                  reference=ref)
    assert accel.trace["err_f"][-1] <= plain.trace["err_f"][-1]


def test_anderson_window_batched_vs_oracle(rng):
    """AndersonWindow with several independent windows on synthetic
    contractive sequences: restarts, evictions and the mixed vector match the
    oracle's window (sinkhorn.py:215-243) per problem."""
    B, L, depth, reg = 3, 777, 3, 1e-9
    A = [rng.normal(size=(L, L)) * (0.4 / np.sqrt(L)) for _ in range(B)]
    c = [rng.normal(size=L) for _ in range(B)]
    zs = [rng.normal(size=L) for _ in range(B)]
    wins = [O.AndersonState(depth, reg) for _ in range(B)]
    t = D.torch()
    win = P.AndersonWindow(B, L, depth, reg)
    zd = D.to_dev(np.stack(zs), t.float64)
    for it in range(12):
        zc = D.to_np(zd, readonly=False)
        tz = np.stack([np.tanh(A[b] @ zc[b]) + c[b] + (0.3 if it == 5 else 0.0) for b in range(B)])
        want = np.stack([wins[b].push_extrapolate(zc[b], tz[b]) for b in range(B)])
        out = t.empty_like(zd)
        delta, status = win.step(zd, D.to_dev(tz, t.float64), out, L // 2)
        assert (D.to_np(status) == 0).all()
        got = D.to_np(out, readonly=False)
        np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(D.to_np(delta), np.abs(want[:, :L // 2] - zc[:, :L // 2]).max(1),
                                   rtol=1e-10, atol=1e-13)
        zd = out
