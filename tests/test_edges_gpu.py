"""Edge cases on the device paths, against the CPU oracle: single-atom and
very unequal supports, ragged barycenter lists, zero-weight runs, the size
limits of each kernel (and the errors just beyond them)."""

import numpy as np
import pytest

import oracle as O
import paper_2201_00730_b200 as P
from conftest import rel_err
from paper_2201_00730_b200 import _device as D

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m", [(1, 1), (1, 37), (53, 1), (2, 700)])
@pytest.mark.parametrize("variant", ["h", "f"])
def test_sinkhorn_degenerate_shapes_fp64(n, m, variant):
    rng = np.random.default_rng(n * 1000 + m)
    x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
    a, b = rng.uniform(0.1, 1, n), rng.uniform(0.1, 1, m) * 1.3
    f, g, _, _ = P.sinkhorn_batched(x[None], y[None], a[None], b[None], 0.1, 0.7, 1.9, 30,
                                    variant=variant, cost="power", p=1.5, precision="fp64")
    fo, go, _ = O.sinkhorn_fixed(O.PointCost(x, y, p=1.5, power1d=True), a, b, 0.1, 0.7, 1.9,
                                 variant, 30)
    assert rel_err(D.to_np(f[0]), D.to_np(g[0]), fo, go) < 1e-9


def test_sinkhorn_zero_weight_runs_point_cloud():
    """Whole blocks of zero-weight atoms (masked out of every log-sum-exp,
    entropies.py:78-89) on both sides of a d = 3 point cloud."""
    rng = np.random.default_rng(8)
    n, m, d = 700, 650, 3
    x, y = rng.normal(size=(n, d)), rng.normal(size=(m, d))
    a, b = rng.uniform(0.1, 1, n), rng.uniform(0.1, 1, m)
    a[100:400] = 0.0
    b[:257] = 0.0
    b[600:] = 0.0
    f, g, _, _ = P.sinkhorn_batched(x[None], y[None], a[None], b[None], 0.5, 1.0, 1.0, 25,
                                    precision="fp64")
    fo, go, _ = O.sinkhorn_fixed(O.PointCost(x, y), a, b, 0.5, 1.0, 1.0, "h", 25)
    assert rel_err(D.to_np(f[0]), D.to_np(g[0]), fo, go) < 1e-9


@pytest.mark.parametrize("n,m", [(1, 9), (9, 1), (4096, 4096), (4096, 17)])
def test_ot1d_shapes_and_max_size(n, m):
    rng = np.random.default_rng(n + 7 * m)
    x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
    a = rng.exponential(1.0, n)
    if n > 4:
        a[: n // 5] = 0.0  # a leading zero-weight run
    b = rng.exponential(1.0, m)
    b *= a.sum() / b.sum()
    f, g, ei, ej, em, cnt, st = P.solve_ot_1d_batched(x, y, a, b, 2.0)
    assert int(st[0].item()) == 0
    ii, jj, mm, fo, go = O.solve_ot_1d(x, y, a, b, 2.0)
    c = int(cnt[0].item())
    np.testing.assert_array_equal(D.to_np(ei[0, :c]), ii)
    np.testing.assert_array_equal(D.to_np(ej[0, :c]), jj)
    np.testing.assert_allclose(D.to_np(em[0, :c]), mm, rtol=0, atol=1e-13 * a.sum())
    assert rel_err(D.to_np(f[0]), D.to_np(g[0]), fo, go) < 1e-12


def test_ot1d_beyond_max_size_raises():
    """n, m <= 4096 run resident on chip, up to 262144 on the large-problem
    kernels (tests/test_large_gpu.py); beyond that the call raises."""
    x = np.linspace(0, 1, 262145)
    w = np.full(262145, 1.0 / 262145)
    with pytest.raises(ValueError):
        P.solve_ot_1d_batched(x, x, w, w, 2.0)


@pytest.mark.parametrize("n,m", [(1, 1), (1, 300), (4096, 4096)])
def test_fw_harmonic_shapes_vs_oracle(n, m):
    """Harmonic steps make the trajectory independent of the line search,
    so the device run equals the oracle's to rounding (plan bit-exact)."""
    rng = np.random.default_rng(5 * n + m)
    x, y = np.sort(rng.uniform(0, 1, n)), np.sort(rng.uniform(0, 1, m))
    a, b = rng.exponential(1.0, n), rng.exponential(1.0, m) * 1.4
    iters = 12
    r = P.fw_solve_batched(x[None], y[None], a[None], b[None], 1.0, 1.0, 2.0, iters, "harmonic")
    ref = O.fw_fixed(x, y, a, b, 1.0, 1.0, iters, step="harmonic")
    assert rel_err(D.to_np(r.f[0]), D.to_np(r.g[0]), ref["f"], ref["g"]) < 1e-9
    np.testing.assert_allclose(D.to_np(r.h0[0]), ref["h0"], rtol=1e-9, atol=1e-12)


def test_mot_ragged_lists_vs_oracle():
    """Lists of different lengths (1 .. 700 atoms), zero weights inside."""
    rng = np.random.default_rng(21)
    lens = [1, 700, 33, 2, 129, 512]
    xs = [np.sort(rng.uniform(0, 1, L)) for L in lens]
    ws = []
    for L in lens:
        w = rng.uniform(0.1, 1.0, L)
        if L > 10:
            w[L // 3: L // 2] = 0.0
        ws.append(w / w.sum() * 1.7)
    om = rng.dirichlet(np.ones(len(lens)))
    plan, duals = P.solve_mot_1d([P.DiscreteMeasure(x, w) for x, w in zip(xs, ws)], om)
    idx, mass, pots = O.solve_mot_1d(xs, ws, om)
    np.testing.assert_array_equal(plan.indices, idx)
    np.testing.assert_allclose(plan.mass, mass, rtol=0, atol=1e-13 * 1.7)
    scale = max(1.0, max(np.abs(p).max() for p in pots))
    for q in range(len(lens)):
        assert np.abs(duals.potentials[q] - pots[q]).max() <= 1e-12 * scale


def test_mot_max_list_length_and_k2():
    """n = 16384 atoms per list (the 32-atoms-per-thread instantiation), K = 2."""
    rng = np.random.default_rng(4)
    n = 16384
    xs = [np.sort(rng.uniform(0, 1, n)) for _ in range(2)]
    ws = [rng.uniform(0.5, 1.5, n) for _ in range(2)]
    ws[1] *= ws[0].sum() / ws[1].sum()
    om = np.array([0.3, 0.7])
    plan, duals = P.solve_mot_1d([P.DiscreteMeasure(x, w) for x, w in zip(xs, ws)], om)
    idx, mass, pots = O.solve_mot_1d(xs, ws, om)
    np.testing.assert_array_equal(plan.indices, idx)
    scale = max(1.0, max(np.abs(p).max() for p in pots))
    for q in range(2):
        assert np.abs(duals.potentials[q] - pots[q]).max() <= 1e-12 * scale


def test_mot_limits_raise():
    one = P.DiscreteMeasure([0.5], [1.0])
    with pytest.raises(ValueError):
        P.solve_mot_1d([one] * 33, np.full(33, 1 / 33))  # K > 32 (two lists per CTA, 16-CTA clusters)
    P.solve_mot_1d([one] * 17, np.full(17, 1 / 17))  # 16 < K <= 32 runs
    big = P.DiscreteMeasure(np.linspace(0, 1, 16385), np.full(16385, 1 / 16385))
    P.solve_mot_1d([big, big], np.array([0.5, 0.5]))  # up to 131072 atoms per list (K <= 16)
    huge = P.DiscreteMeasure(np.linspace(0, 1, 131073), np.full(131073, 1 / 131073))
    with pytest.raises(ValueError):
        P.solve_mot_1d([huge, huge], np.array([0.5, 0.5]))


def test_barycenter_ragged_vs_oracle():
    """KL barycenter FW (harmonic steps) on ragged lists."""
    rng = np.random.default_rng(77)
    lens = [40, 7, 64]
    xs = [np.sort(rng.uniform(0, 1, L)) for L in lens]
    ws = [rng.uniform(0.1, 1.0, L) * s for L, s in zip(lens, (1.0, 0.6, 1.8))]
    om = np.array([0.2, 0.5, 0.3])
    prob = P.BarycenterProblem(tuple(P.DiscreteMeasure(x, w) for x, w in zip(xs, ws)), om, 1.5)
    rep, _ = P.fw_barycenter(prob, P.FwConfig("harmonic", 15, 1e-300))
    ref = O.fw_barycenter_fixed(xs, ws, om, 1.5, 15, step="harmonic")
    k = len(rep.trace["h0"])
    assert k >= 10
    np.testing.assert_allclose(rep.trace["h0"], ref["h0"][:k], rtol=1e-9, atol=1e-12)
