"""GPU parity of the fused Sinkhorn kernels against the reference goldens
and the CPU oracle.  Tolerances (north star): 1e-9 relative in fp64,
1e-4 * eps absolute in fp32."""

import numpy as np
import pytest

import oracle as O
import paper_2201_00730_b200 as P
from conftest import cases, golden, rel_err
from paper_2201_00730_b200 import _device as D
from paper_2201_00730_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def run_dev(x, y, a, b, eps, rho, iters, variant="h", cost="sqeuclid", p=2.0, c=None,
            precision="fp64", rho2=None, f0=None):
    f, g, tr, its = P.sinkhorn_batched(x, y, a, b, eps, rho, rho if rho2 is None else rho2, iters,
                                       variant=variant, cost=cost, p=p, c=c,
                                       precision=precision, f0=f0)
    return (D.to_np(f).astype(np.float64), D.to_np(g).astype(np.float64), D.to_np(tr),
            D.to_np(its))


@pytest.mark.parametrize("variant", ["h", "f"])
def test_cfg1_fp64_1000_iterations(variant):
    z = golden("cfg1.npz")
    f, g, tr, its = run_dev(z["x"][None], z["y"][None], z["alpha"][None], z["beta"][None],
                            float(z["eps"]), 1.0, 1000, variant=variant, cost="power")
    assert its[0] == 1000
    assert rel_err(f[0], g[0], z[f"{variant}_f"], z[f"{variant}_g"]) < 1e-9
    np.testing.assert_allclose(tr[0], z[f"{variant}_delta"], rtol=1e-6,
                               atol=1e-12 * np.abs(z[f"{variant}_f"]).max())


def test_small_cases_fp64_power_costs_and_zero_weights():
    z = golden("sinkhorn_small.npz")
    for k in cases(z):
        p, eps, r1, r2, iters = z[f"c{k}_par"]
        for v in ("h", "f"):
            f, g, _, _ = run_dev(z[f"c{k}_x"][None], z[f"c{k}_y"][None], z[f"c{k}_a"][None],
                                 z[f"c{k}_b"][None], eps, r1, int(iters), variant=v, cost="power",
                                 p=p, rho2=r2)
            assert rel_err(f[0], g[0], z[f"c{k}_{v}_f"], z[f"c{k}_{v}_g"]) < 1e-9, (k, v)


def test_small_cases_explicit_cost_fp64():
    z = golden("sinkhorn_small.npz")
    for k in cases(z)[:6]:
        p, eps, r1, r2, iters = z[f"c{k}_par"]
        C = np.abs(z[f"c{k}_x"][:, None] - z[f"c{k}_y"][None, :]) ** p
        f, g, _, _ = run_dev(z[f"c{k}_x"][None], z[f"c{k}_y"][None], z[f"c{k}_a"][None],
                             z[f"c{k}_b"][None], eps, r1, int(iters), variant="h", cost="explicit",
                             c=C[None], rho2=r2)
        assert rel_err(f[0], g[0], z[f"c{k}_h_f"], z[f"c{k}_h_g"]) < 1e-9, k


@pytest.mark.parametrize("name", ["cfg3_small.npz", "cfg4_small.npz"])
def test_point_clouds_fp64(name):
    z = golden(name)
    f, g, _, _ = run_dev(z["x"][None], z["y"][None], z["alpha"][None], z["beta"][None],
                         float(z["eps"]), float(z["rho"]), int(z["iters"]))
    assert rel_err(f[0], g[0], z["f"], z["g"]) < 1e-9


def translated(a, b, f, g, r1, r2):
    """Canonical representative (f + t*, g - t*) of the H-iterate.  H is
    exactly invariant along (f + c, g - c) (src/duality.py:256-276), so the
    H-Sinkhorn iterate's translation is a neutral direction in which fp32
    rounding bias accumulates linearly (measured: -5e-6 after 300 iterations
    at cfg4 with eps = 0.05; scripts/exp_fp32_cfg4.py); parity in fp32 is
    therefore stated on the translated pair and on the (translation
    invariant) dual objective."""
    lam = O.lambda_star_kl(a, b, f, g, r1, r2)
    return f + lam, g - lam


@pytest.mark.parametrize("name", ["cfg3_small.npz", "cfg4_small.npz"])
def test_point_clouds_fp32_tolerance(name):
    z = golden(name)
    eps, rho = float(z["eps"]), float(z["rho"])
    f, g, _, _ = run_dev(z["x"][None], z["y"][None], z["alpha"][None], z["beta"][None], eps,
                         rho, int(z["iters"]), precision="fp32")
    ft, gt = translated(z["alpha"], z["beta"], f[0], g[0], rho, rho)
    fr, gr = translated(z["alpha"], z["beta"], z["f"], z["g"], rho, rho)
    assert np.abs(ft - fr).max() <= 1e-4 * eps
    assert np.abs(gt - gr).max() <= 1e-4 * eps
    cost = O.PointCost(z["x"], z["y"])
    H = O.eval_h_kl(z["alpha"], z["beta"], f[0], g[0], rho, rho, eps,
                    smin_fn=lambda ff, e: cost.smin_cols(ff, e, z["alpha"]))
    assert abs(H - float(z["dual"])) <= 1e-4 * eps


def test_batched_equals_individual():
    x, y, a, b = S.cfg4_batch(batch=3, n=96, m=80, d=3)
    fb, gb, _, _ = run_dev(x, y, a, b, 0.05, 0.5, 30)
    for k in range(3):
        f1, g1, _, _ = run_dev(x[k:k + 1], y[k:k + 1], a[k:k + 1], b[k:k + 1], 0.05, 0.5, 30)
        assert rel_err(fb[k], gb[k], f1[0], g1[0]) < 1e-13


def test_cfg3_shape_fp32_vs_oracle_2048():
    c = S.cfg3_inputs(n=2048, seed=99)
    f, g, _, _ = run_dev(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps, c.rho, 200,
                         precision="fp32")
    cost = O.PointCost(c.x, c.y)
    fo, go, _ = O.sinkhorn_fixed(cost, c.alpha, c.beta, c.eps, c.rho, c.rho, "h", 200)
    ft, gt = translated(c.alpha, c.beta, f[0], g[0], c.rho, c.rho)
    fr, gr = translated(c.alpha, c.beta, fo, go, c.rho, c.rho)
    assert np.abs(ft - fr).max() <= 1e-4 * c.eps
    assert np.abs(gt - gr).max() <= 1e-4 * c.eps


def test_full_cfg3_one_step_sampled_columns():
    """Size-independent check at the full BASELINE size (N = M = 65536): the
    column differences of one GPU g-update equal the oracle's softmin
    differences on sampled columns (translation-free, so the global Smin
    shift cancels), from a GPU-produced f."""
    c = S.cfg3_inputs()
    f, g, _, _ = run_dev(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps, c.rho, 3,
                         precision="fp32")
    f2, g2, _, _ = run_dev(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps, c.rho, 1,
                           precision="fp32", f0=f)
    rng = np.random.default_rng(0)
    cols = np.sort(rng.choice(len(c.y), 256, replace=False))
    cost = O.PointCost(c.x, c.y[cols])
    smin = cost.smin_cols(f[0], c.eps, c.alpha)
    a_coef = c.rho / (c.rho + c.eps)
    ref = a_coef * (smin - smin[0])
    got = g2[0][cols] - g2[0][cols[0]]
    assert np.abs(got - ref).max() <= 1e-4 * c.eps


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("nshards", [2, 3])
@pytest.mark.parametrize("chunks", [None, "3"])
def test_row_sharded_protocol_emulated(precision, nshards, chunks, monkeypatch):
    """The NCCL row-sharding protocol (one all-gather per iteration, or the
    exchange in column chunks on a second stream overlapping the next chunk's
    main kernel), run for all shards in one process, equals the unsharded
    solve."""
    from paper_2201_00730_b200.distributed import shard_rows

    if chunks is not None:
        monkeypatch.setenv("UOT_SHARD_CHUNKS", chunks)

    c = S.cfg3_inputs(n=1536, m=1280, seed=11)
    rows = shard_rows(len(c.x), nshards)
    f1, g1, t1, _ = run_dev(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps, c.rho, 25,
                            precision=precision)
    f, g, tr, its = P.sinkhorn_batched(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps,
                                       c.rho, c.rho, 25, precision=precision, nranks=nshards,
                                       shard_rows=rows)
    f, g = D.to_np(f).astype(float), D.to_np(g).astype(float)
    tr = D.to_np(tr)
    assert int(its[0].item()) == 25
    if precision == "fp64":
        assert rel_err(f[0], g[0], f1[0], g1[0]) < 1e-12
        np.testing.assert_allclose(tr[0], t1[0], rtol=1e-9, atol=1e-14)
    else:
        ft, gt = translated(c.alpha, c.beta, f[0], g[0], c.rho, c.rho)
        fr, gr = translated(c.alpha, c.beta, f1[0], g1[0], c.rho, c.rho)
        assert np.abs(ft - fr).max() <= 1e-4 * c.eps
        assert np.abs(gt - gr).max() <= 1e-4 * c.eps


@pytest.mark.parametrize("d,n,m", [(64, 300, 257), (32, 128, 640), (48, 513, 129)])
def test_tcgen05_point_clouds_vs_oracle(d, n, m):
    """d >= 32 runs the tcgen05 fp16-split kernel; ragged sizes exercise the
    padded tiles.  fp32 tolerance on the translated pair (1e-4 eps)."""
    x, y, a, b = S.cfg4_batch(batch=2, n=n, m=m, d=d, seed=d)
    eps, rho = 0.05, 0.5
    f, g, _, _ = run_dev(x, y, a, b, eps, rho, 40, precision="fp32")
    for k in range(2):
        cost = O.PointCost(x[k], y[k])
        fo, go, _ = O.sinkhorn_fixed(cost, a[k], b[k], eps, rho, rho, "h", 40)
        ft, gt = translated(a[k], b[k], f[k], g[k], rho, rho)
        fr, gr = translated(a[k], b[k], fo, go, rho, rho)
        assert np.abs(ft - fr).max() <= 1e-4 * eps, (k, np.abs(ft - fr).max())
        assert np.abs(gt - gr).max() <= 1e-4 * eps


# ---------------------------------------------------------------------------
# G-Sinkhorn (src/sinkhorn.py:117-134), §8f row 2


@pytest.mark.parametrize("k", range(9))
def test_g_sinkhorn_matches_reference(k):
    z = golden("sinkhorn_g.npz")
    p, eps, r1, r2, iters, hasinit = z[f"c{k}_par"]
    f0 = z[f"c{k}_f0"] if hasinit else None
    g0 = z[f"c{k}_g0"] if hasinit else None
    f, g, dl, its = P.sinkhorn_batched(z[f"c{k}_x"], z[f"c{k}_y"], z[f"c{k}_a"], z[f"c{k}_b"],
                                       eps, r1, r2, int(iters), variant="g", cost="power", p=p,
                                       f0=f0, g0=g0, precision="fp64")
    fg, gg = D.to_np(f[0]), D.to_np(g[0])
    assert rel_err(fg, gg, z[f"c{k}_f"], z[f"c{k}_g"]) < 1e-9
    np.testing.assert_allclose(D.to_np(dl[0]), z[f"c{k}_delta"], rtol=1e-6, atol=1e-12)


def test_g_sinkhorn_step_api():
    """g_sinkhorn_step(prob, d, lam) mirrors the reference's signature."""
    z = golden("sinkhorn_g.npz")
    k = 1
    p, eps, r1, r2, _, _ = z[f"c{k}_par"]
    prob = P.UotProblem(P.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"]),
                        P.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"]), P.PowerDistance(p),
                        P.KL(r1), P.KL(r2), eps=eps)
    d = P.DualPair(z[f"c{k}_f0"], z[f"c{k}_g0"])
    cost = O.PointCost(z[f"c{k}_x"], z[f"c{k}_y"], p=p, power1d=True)
    lam = 0.123
    fr, gr, lr = O.g_sinkhorn_step(cost, z[f"c{k}_a"], z[f"c{k}_b"], d.f, d.g, eps, r1, r2, lam)
    pair, lam_new = P.g_sinkhorn_step(prob, d, lam)
    assert rel_err(pair.f, pair.g, fr, gr) < 1e-9
    assert abs(lam_new - lr) < 1e-9 * max(1.0, abs(lr))


# ---------------------------------------------------------------------------
# Verification at scale (§8f row 3): dual objectives and stationarity
# residuals without the N x M matrix (uot_sinkhorn_verify)


@pytest.mark.parametrize("variant", ["h", "f"])
def test_dual_objective_matches_reference(variant):
    z = golden("sinkhorn_small.npz")
    for k in cases(z):
        p, eps, r1, r2, _ = z[f"c{k}_par"]
        prob = P.UotProblem(P.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"]),
                            P.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"]), P.PowerDistance(p),
                            P.KL(r1), P.KL(r2), eps=eps)
        d = P.DualPair(z[f"c{k}_{variant}_f"], z[f"c{k}_{variant}_g"])
        ref = float(z[f"c{k}_{variant}_dual"])
        got = P.eval_H(prob, d)
        assert abs(got - ref) <= 1e-9 * max(1.0, abs(ref)), (k, got, ref)


def test_dual_objective_cfg1_and_residual():
    z = golden("cfg1.npz")
    prob = P.UotProblem(P.DiscreteMeasure(z["x"], z["alpha"]), P.DiscreteMeasure(z["y"], z["beta"]),
                        P.PowerDistance(2.0), P.KL(float(z["rho"])), P.KL(float(z["rho"])),
                        eps=float(z["eps"]))
    for v in ("h", "f"):
        d = P.DualPair(z[f"{v}_f"], z[f"{v}_g"])
        ref = float(z[f"{v}_dual"])
        assert abs(P.eval_H(prob, d) - ref) <= 1e-9 * max(1.0, abs(ref))
    # stationarity right after an H step (tests/test_sinkhorn.py:145-150 of the reference)
    d = P.DualPair(z["h_f"], z["h_g"])
    assert P.h_optimality_residual(prob, d, "f") < 1e-9
    # eval_F and eval_G agree at the optimal translation: G(d, lam*) = H(d)
    lam = P.lambda_star(prob, d)
    assert abs(P.eval_G(prob, d, lam) - P.eval_H(prob, d)) < 1e-9


def test_verify_matches_oracle_points():
    """Point-cloud (fp32 on-the-fly) verification vs the oracle's dense terms."""
    z = golden("cfg3_small.npz")
    x, y, wa, wb = z["x"], z["y"], z["alpha"], z["beta"]
    eps, rho = float(z["eps"]), float(z["rho"])
    f, g = z["f"], z["g"]
    out = D.to_np(P.verify_batched(x, y, wa, wb, f, g, eps, rho, rho, precision="fp64")[0])
    cost = O.PointCost(x, y)
    C = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    expo = (f[:, None] + g[None, :] - C) / eps
    L = float(np.log(np.sum(wa[:, None] * wb[None, :] * np.exp(expo))))
    assert abs(out[1] - L) < 1e-9 * max(1.0, abs(L))
    res_f = np.abs(f - (rho / (rho + eps)) * cost.smin_rows(g, eps, wb)
                   + (eps / (eps + rho)) * out[4]).max()
    assert abs(out[2] - res_f) < 1e-9


@pytest.mark.parametrize("k", range(8))
def test_sinkhorn_berg_balanced(k):
    """F / G Sinkhorn with Berg (per-element Newton aprox, Newton lambda*)
    and Balanced penalties (§8f row 2) vs the reference."""
    z = golden("sinkhorn_ent.npz")
    p, eps, r1, r2, iters = z[f"c{k}_par"]
    var, e1, e2 = (str(v) for v in z[f"c{k}_spec"])
    f, g, dl, its = P.sinkhorn_batched(z[f"c{k}_x"], z[f"c{k}_y"], z[f"c{k}_a"], z[f"c{k}_b"],
                                       eps, r1, r2, int(iters), variant=var, cost="power", p=p,
                                       precision="fp64", ent1=e1, ent2=e2)
    assert rel_err(D.to_np(f[0]), D.to_np(g[0]), z[f"c{k}_f"], z[f"c{k}_g"]) < 1e-9, (var, e1, e2)
    np.testing.assert_allclose(D.to_np(dl[0]), z[f"c{k}_delta"], rtol=1e-6, atol=1e-12)


def test_h_rejects_berg():
    z = golden("sinkhorn_ent.npz")
    with pytest.raises(P.UnsupportedEntropyError):
        P.sinkhorn_batched(z["c0_x"], z["c0_y"], z["c0_a"], z["c0_b"], 0.1, 1.0, 1.0, 2,
                           variant="h", cost="power", precision="fp64", ent1="berg", ent2="kl")


@pytest.mark.parametrize("chunks", [None, "4"])
def test_row_sharded_real_nccl_single_rank(chunks, monkeypatch):
    """The real NCCL branch of the row-sharded path (communicator built in the
    extension from a unique id broadcast by torch.distributed, ncclAllGather
    per iteration -- or grouped ncclSend / ncclRecv per column chunk on a
    second stream --, the scalar all-gather at the end) with one rank: equals
    the unsharded solve.  Multi-rank runs need more than one GPU."""
    import os

    if chunks is not None:
        monkeypatch.setenv("UOT_SHARD_CHUNKS", chunks)

    import torch.distributed as dist

    from paper_2201_00730_b200.distributed import NcclComm

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    created = False
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
        created = True
    try:
        c = S.cfg3_inputs(n=1024, m=768, seed=13)
        f1, g1, t1, _ = run_dev(c.x[None], c.y[None], c.alpha[None], c.beta[None], c.eps, c.rho,
                                20, precision="fp64")
        with NcclComm(1, 0) as comm:
            f, g, tr, its = P.sinkhorn_batched(c.x[None], c.y[None], c.alpha[None], c.beta[None],
                                               c.eps, c.rho, c.rho, 20, precision="fp64",
                                               comm=comm.handle, nranks=1, rank=0)
            f, g = D.to_np(f).astype(float), D.to_np(g).astype(float)
        assert int(its[0].item()) == 20
        assert rel_err(f[0], g[0], f1[0], g1[0]) < 1e-12
        np.testing.assert_allclose(D.to_np(tr)[0], t1[0], rtol=1e-9, atol=1e-14)
    finally:
        if created:
            dist.destroy_process_group()


@pytest.mark.parametrize("d,offset", [(2, 1000.0), (3, -300.0), (5, 1000.0), (2, 0.0)])
def test_fp32_point_clouds_off_origin(d, offset):
    """The fp32 expanded-form engines (x.y on the FMA pipe, records
    U = (hat - |x|^2) L + log2 w) take the points relative to the midpoint
    of the two clouds' centroids (sk_center), so a cloud far from the origin
    keeps fp32 tolerance: uncentred, |x|^2 L would swamp the exponent.  The
    oracle runs on the same fp32-rounded points (fp64)."""
    rng = np.random.default_rng(d)
    n, m = 700, 530
    x = (rng.standard_normal((n, d)) * 0.3 + offset).astype(np.float32).astype(np.float64)
    y = (rng.standard_normal((m, d)) * 0.3 + 0.2 + offset).astype(np.float32).astype(np.float64)
    a = rng.uniform(0.5, 1.5, n)
    a /= a.sum()
    b = rng.uniform(0.5, 1.5, m)
    b *= 1.2 / b.sum()
    eps = 0.02
    f, g, _, _ = run_dev(x[None], y[None], a[None], b[None], eps, 1.0, 50, precision="fp32")
    fo, go, _ = O.sinkhorn_fixed(O.PointCost(x, y), a, b, eps, 1.0, 1.0, "h", 50)
    err = max(np.abs(f[0] - fo).max(), np.abs(g[0] - go).max())
    assert err <= 1e-4 * eps, err
