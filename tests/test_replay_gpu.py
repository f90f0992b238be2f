"""Reference-replay parity: the device FW, pairwise FW and
barycenter FW consume the reference's own step sizes gamma_t (and, for
pairwise, its away positions) -- tests/golden/replay.npz, recorded by
tests/golden/make_golden.py::gen_replay from src/fw.py:176-232, :275-310 and
src/barycenter.py:361-411 -- and record the hash of every iteration's oracle
plan support.  With the step rule taken out of the comparison, the rest of the
pipeline (tilt, lambda*, oracle, H_0, update) must match the reference at
EVERY iteration: supports bit-exact (hash and entry count), H_0 and the final
potentials to 1e-12 relative.  The production step rule (Newton) is compared
separately in test_fw_gpu.py / test_barycenter_gpu.py with its measured
deviation."""

import numpy as np
import pytest

import paper_2201_00730_b200 as P
from conftest import cases, golden, rel_err
from paper_2201_00730_b200 import _device as D

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _check_trace(r, zr, tag, iters):
    hs = D.to_np(r.supp_hash[0])
    nz = D.to_np(r.supp_nnz[0])
    bad = np.nonzero((hs != zr[f"{tag}_hash"]) | (nz != zr[f"{tag}_nnz"]))[0]
    assert bad.size == 0, f"{tag}: support differs at iterations {bad[:10]} of {iters}"
    h0 = D.to_np(r.h0[0])
    ref = zr[f"{tag}_h0"]
    assert np.abs(h0 - ref).max() <= TOL * max(1.0, np.abs(ref).max()), tag


@pytest.mark.parametrize("k", list(range(9)))
def test_fw_replay_every_iteration(k):
    z, zr = golden("fw.npz"), golden("replay.npz")
    assert k in cases(z)
    r1, r2, p, iters, ls = z[f"c{k}_par"]
    iters = int(iters)
    gam = zr[f"fw{k}_gamma"]
    r = P.fw_solve_batched(z[f"c{k}_x"], z[f"c{k}_y"], z[f"c{k}_a"], z[f"c{k}_b"], r1, r2, p,
                           iters, "linesearch" if ls else "harmonic", step_in=gam[None],
                           trace_support=True)
    assert int(r.status[0].item()) == 0
    _check_trace(r, zr, f"fw{k}", iters)
    f, g = D.to_np(r.f[0]), D.to_np(r.g[0])
    assert rel_err(f, g, z[f"c{k}_f"], z[f"c{k}_g"]) <= TOL, k
    c = int(r.count[0].item())  # the last plan, entry by entry
    np.testing.assert_array_equal(D.to_np(r.ei[0, :c]), z[f"c{k}_i"])
    np.testing.assert_array_equal(D.to_np(r.ej[0, :c]), z[f"c{k}_j"])


@pytest.mark.parametrize("k", list(range(6)))
def test_pairwise_replay_every_iteration(k):
    z, zr = golden("pfw.npz"), golden("replay.npz")
    assert k in cases(z)
    r1, r2, p, iters = z[f"c{k}_par"]
    iters = int(iters)
    r = P.fw_solve_batched(z[f"c{k}_x"], z[f"c{k}_y"], z[f"c{k}_a"], z[f"c{k}_b"], r1, r2, p,
                           iters, "pairwise", step_in=zr[f"pfw{k}_gamma"][None],
                           away_in=zr[f"pfw{k}_away"][None].astype(np.int32),
                           trace_support=True)
    assert int(r.status[0].item()) == 0
    _check_trace(r, zr, f"pfw{k}", iters)
    np.testing.assert_array_equal(D.to_np(r.natoms[0]), z[f"c{k}_natoms"])
    f, g = D.to_np(r.f[0]), D.to_np(r.g[0])
    assert rel_err(f, g, z[f"c{k}_f"], z[f"c{k}_g"]) <= TOL, k


@pytest.mark.parametrize("k", list(range(5)))
def test_barycenter_replay_every_iteration(k):
    from paper_2201_00730_b200.barycenter import _pack

    z, zr = golden("barycenter.npz"), golden("replay.npz")
    assert k in cases(z)
    kk = int(z[f"c{k}_k"])
    inputs = [P.DiscreteMeasure(z[f"c{k}_x{q}"], z[f"c{k}_a{q}"]) for q in range(kk)]
    rho, iters, ls = z[f"c{k}_par"]
    iters = int(iters)
    x, a, _, lens = _pack(inputs)
    r = P.fw_barycenter_batched(x, a, z[f"c{k}_w"], float(rho), iters,
                                "linesearch" if ls else "harmonic", lens=lens,
                                step_in=zr[f"bary{k}_gamma"][None], trace_support=True)
    assert int(r.status[0].item()) == 0
    _check_trace(r, zr, f"bary{k}", iters)
    f = D.to_np(r.f[0])
    scale = max(np.abs(z[f"c{k}_f{q}"]).max() for q in range(kk))
    err = max(np.abs(f[q, :lens[q]] - z[f"c{k}_f{q}"]).max() for q in range(kk))
    assert err <= TOL * scale, (k, err / scale)
    c = int(r.count[0].item())
    np.testing.assert_array_equal(D.to_np(r.idx[0, :c]).astype(np.int64), z[f"c{k}_idx"])
