"""File formats and the CLI's ``gen`` command, byte for byte against the
reference's own writers (tests/golden/formats.npz).  CPU only: these are
host-side formats; nothing here launches a kernel."""

import contextlib
import io
import json

import numpy as np
import pytest

import paper_2201_00730_b200 as P
from conftest import golden
from paper_2201_00730_b200 import cli
from paper_2201_00730_b200 import formats as F
from paper_2201_00730_b200.sinkhorn import SolverReport


def _text(fn, *args):
    buf = io.StringIO()
    fn(*args, buf)
    return buf.getvalue()


def test_gen_stdout_matches_reference():
    z = golden("formats.npz")
    k = 0
    while f"gen{k}_args" in z:
        kind, n, seed = (str(v) for v in z[f"gen{k}_args"])
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert cli.main(["gen", "--kind", kind, "--n", n, "--seed", seed]) == 0
        assert buf.getvalue() == str(z[f"gen{k}_text"]), (kind, n, seed)
        k += 1
    assert k == 4


def test_gen_file_deterministic_with_sidecar(tmp_path):
    p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
    assert cli.main(["gen", "--n", "40", "--seed", "9", "--out", str(p1)]) == 0
    assert cli.main(["gen", "--n", "40", "--seed", "9", "--out", str(p2)]) == 0
    assert p1.read_bytes() == p2.read_bytes()
    assert json.loads((tmp_path / "a.csv.meta.json").read_text())["command"] == "gen"
    assert cli.main(["gen", "--n", "0"]) == 1
    assert cli.main(["nope"]) == 1


def test_measure_formats_round_trip():
    z = golden("formats.npz")
    a = P.DiscreteMeasure(z["ma_x"], z["ma_w"])
    assert F.measure_to_csv_text(a, ["one", "two three"]) == str(z["ma_csv"])
    assert _text(F.write_measure_json, a) == str(z["ma_json"])
    back = F.read_measure_csv(io.StringIO(str(z["ma_csv"])))
    np.testing.assert_array_equal(back.points, a.points)
    np.testing.assert_array_equal(back.weights, a.weights)
    back = F.read_measure_json(io.StringIO(str(z["ma_json"])))
    np.testing.assert_array_equal(back.weights, a.weights)
    with pytest.raises(ValueError):
        F.read_measure_csv(io.StringIO("a,b\n1,2\n"))
    with pytest.raises(ValueError):
        F.read_measure_csv(io.StringIO("x,w\n1\n"))


def test_plan_formats():
    z = golden("formats.npz")
    plan = P.SparsePlan(z["plan_i"], z["plan_j"], z["plan_m"])
    assert _text(F.write_plan_csv, plan) == str(z["plan_csv"])
    back = F.read_plan_csv(io.StringIO(str(z["plan_csv"])))
    np.testing.assert_array_equal(back.mass, plan.mass)
    mp = P.MultiPlan(z["mp_idx"], z["mp_mass"])
    assert _text(F.write_multiplan_csv, mp) == str(z["mp_csv"])
    back = F.read_multiplan_csv(io.StringIO(str(z["mp_csv"])))
    np.testing.assert_array_equal(back.indices, mp.indices)
    with pytest.raises(ValueError):
        F.read_plan_csv(io.StringIO("i,j\n0,0\n"))


def test_trace_formats():
    z = golden("formats.npz")
    pair = P.DualPair.zeros(1, 1)
    tr = {"delta_f": z["tr_delta"], "wall_ns": z["tr_wall"]}
    rep = SolverReport(final=pair, iterations=3, converged=True, trace=tr)
    assert _text(F.write_trace_csv, rep) == str(z["trace_csv"])
    assert _text(P.write_trace_csv, rep) == str(z["trace_csv"])
    rep2 = SolverReport(final=pair, iterations=3, converged=True,
                        trace=dict(tr, err_f=z["tr_errf"], err_g=z["tr_errg"]))
    assert _text(F.write_trace_csv, rep2) == str(z["trace_ref_csv"])
    rep3 = SolverReport(final=pair, iterations=2, converged=True,
                        trace={"h0": z["gap_h0"], "fw_gap": z["gap_fw"], "pd_gap": z["gap_pd"],
                               "wall_ns": z["gap_wall"]})
    assert _text(F.write_gap_csv, rep3) == str(z["gap_csv"])


def test_estimate_rate():
    e = 0.5 ** np.arange(10)
    assert P.estimate_rate(e) == pytest.approx(0.5, rel=1e-12)
    assert P.estimate_rate(np.ones(6)) == 1.0
    with pytest.raises(ValueError):
        P.estimate_rate(np.array([1.0, 1e-14, 1e-15]))


def test_certificate_assembly():
    """assemble_certificate (src/certify.py:55-66): pass / fail / weak-duality breach."""
    c = P.assemble_certificate(1.0, 1.0 - 1e-10, 0.0, 1e-8)
    assert c.passed and not c.weak_duality_breach
    assert not P.assemble_certificate(1.0, 0.9, 0.0, 1e-8).passed
    b = P.assemble_certificate(1.0, 1.0 + 1e-6, 0.0, 1e-3)
    assert b.weak_duality_breach and not b.passed
    with pytest.raises(ValueError):
        P.assemble_certificate(float("nan"), 0.0, 0.0, 1e-8)
