"""The uotkit-compatible CLI (paper_2201_00730_b200/cli.py) end to end on
the device: outputs, exit codes and certificates as the reference's CLI
tests check them (reference tests/test_cli.py)."""

import io
import json

import numpy as np
import pytest

import paper_2201_00730_b200 as P
from paper_2201_00730_b200 import cli
from paper_2201_00730_b200 import formats as F

pytestmark = pytest.mark.gpu


def _gen(path, n, seed):
    assert cli.main(["gen", "--n", str(n), "--seed", str(seed), "--out", str(path)]) == 0


def _atoms(path, pts, wts):
    F.write_measure_csv(P.DiscreteMeasure(pts, wts), str(path))


def test_sinkhorn_trace_and_exit_codes(tmp_path, capsys):
    one = tmp_path / "one.csv"
    _atoms(one, [0.5], [1.0])
    out = tmp_path / "t.csv"
    assert cli.main(["sinkhorn", str(one), str(one), "--eps", "1.0", "--out", str(out)]) == 0
    rows = out.read_text().splitlines()
    assert rows[0] == "iter,delta_f,err_f,err_g,wall_ns" and len(rows) - 1 <= 2
    assert (tmp_path / "t.csv.meta.json").exists()
    assert cli.main(["sinkhorn", str(one), str(one), "--variant", "h", "--entropy", "berg",
                     "--eps", "1"]) == 1
    assert "h-sinkhorn requires kl" in capsys.readouterr().err
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    _gen(a, 10, 3)
    _gen(b, 10, 4)
    assert cli.main(["sinkhorn", str(a), str(b), "--eps", "0.05", "--rho1", "5", "--max-iters",
                     "3", "--out", str(tmp_path / "x.csv")]) == 2
    assert cli.main(["sinkhorn", "nope.csv", "nope.csv", "--eps", "1"]) == 1


def test_sinkhorn_rate_in_theory_band(tmp_path):
    """kappa of the F trace within [0.7, 1] x (1 + eps/rho)^-2 (+0.02)."""
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    _gen(a, 20, 21)
    _gen(b, 20, 22)
    out = tmp_path / "trace.csv"
    eps, rho = 0.1, 1.0
    assert cli.main(["sinkhorn", str(a), str(b), "--eps", str(eps), "--rho1", str(rho), "--tol",
                     "1e-11", "--out", str(out)]) == 0
    deltas = np.array([float(r.split(",")[1]) for r in out.read_text().splitlines()[1:]])
    kappa = P.estimate_rate(deltas[deltas > 1e-9])
    theory = (1 + eps / rho) ** -2
    assert 0.7 * theory <= kappa <= theory + 0.02


def test_sinkhorn_anderson_and_reference_columns(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    _gen(a, 20, 55)
    _gen(b, 20, 56)
    ref = tmp_path / "ref.json"
    prob = P.UotProblem(F.read_measure_csv(str(a)), F.read_measure_csv(str(b)),
                        P.PowerDistance(2.0), P.KL(5.0), P.KL(5.0), eps=0.1)
    fin = P.run(prob, P.SinkhornConfig("f", 100000, 1e-13)).final
    ref.write_text(json.dumps({"f": fin.f.tolist(), "g": fin.g.tolist()}))
    out = tmp_path / "t.csv"
    assert cli.main(["sinkhorn", str(a), str(b), "--eps", "0.1", "--rho1", "5", "--anderson",
                     "--max-iters", "60", "--tol", "1e-16", "--ref", str(ref),
                     "--out", str(out)]) == 2
    rows = out.read_text().splitlines()[1:]
    assert len(rows) == 60 and all(r.split(",")[2] != "" for r in rows)


def test_rates_rows(tmp_path, capsys):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    _gen(a, 15, 41)
    _gen(b, 15, 42)
    assert cli.main(["rates", str(a), str(b), "--eps", "0.05", "--rho-grid", "0.5,1.0",
                     "--jobs", "2"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "rho,kappa_f,kappa_g,kappa_h"
    assert [float(r.split(",")[0]) for r in lines[1:]] == [0.5, 1.0]
    for row in lines[1:]:
        _, kf, kg, kh = (float(c) for c in row.split(","))
        assert kh <= kf


def test_uot1d_methods(tmp_path, capsys):
    f = tmp_path / "a.csv"
    _gen(f, 12, 51)
    assert cli.main(["uot1d", str(f), str(f), "--rho1", "1", "--gap-tol", "1e-9"]) == 0
    cert = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert cert["passed"] and cert["gap"] < 1e-9
    a, b = tmp_path / "a2.csv", tmp_path / "b2.csv"
    _gen(a, 25, 61)
    _gen(b, 25, 62)
    for method in ("fw-ls", "pfw"):
        out = tmp_path / f"{method}.csv"
        assert cli.main(["uot1d", str(a), str(b), "--method", method, "--gap-tol", "1e-7",
                         "--out", str(out)]) == 0
        rows = out.read_text().splitlines()
        assert rows[0] == "iter,h0,fw_gap,pd_gap,wall_ns"
        assert sum(int(r.split(",")[-1]) for r in rows[1:]) > 0
    a, b = tmp_path / "a3.csv", tmp_path / "b3.csv"
    _gen(a, 30, 71)
    _gen(b, 30, 72)
    assert cli.main(["uot1d", str(a), str(b), "--method", "fw", "--gap-tol", "1e-12",
                     "--max-iters", "3"]) == 2


def test_barycenter_commands(tmp_path, capsys):
    f = tmp_path / "a.csv"
    _gen(f, 10, 81)
    out = tmp_path / "bar.csv"
    assert cli.main(["barycenter", str(f), str(f), "--rho", "1.0", "--gap-tol", "1e-9",
                     "--out", str(out)]) == 0
    assert json.loads(capsys.readouterr().out.strip().splitlines()[-1])["passed"]
    bar, orig = F.read_measure_csv(str(out)), F.read_measure_csv(str(f))
    np.testing.assert_allclose(bar.points, orig.points)
    np.testing.assert_allclose(bar.weights, orig.weights, atol=1e-12)
    fa, fb = tmp_path / "d0.csv", tmp_path / "d1.csv"
    _atoms(fa, [0.0], [1.0])
    _atoms(fb, [1.0], [1.0])
    assert cli.main(["barycenter", str(fa), str(fb), "--weights", "0.25,0.75", "--rho",
                     "2.0"]) == 0
    text = capsys.readouterr().out
    assert F.read_measure_csv(io.StringIO(text[: text.rindex("{")])).points.tolist() == [0.75]
    a, b = tmp_path / "a9.csv", tmp_path / "b9.csv"
    _gen(a, 9, 91)
    _gen(b, 9, 92)
    plan_out = tmp_path / "plan.csv"
    assert cli.main(["barycenter", str(a), str(b), "--balanced", "--plan-out", str(plan_out),
                     "--out", str(tmp_path / "bb.csv")]) == 0
    assert plan_out.read_text().splitlines()[0] == "i1,i2,mass"
    assert cli.main(["barycenter", str(fa), str(fa), "--weights", "0.9,0.9", "--rho", "1"]) == 1


@pytest.mark.parametrize("shift,code", [(0.0, 0), (0.1, 2)])
def test_certify(tmp_path, capsys, shift, code):
    a = P.DiscreteMeasure([0.0, 1.0], [0.7, 0.3])
    b = P.DiscreteMeasure([0.0, 1.0], [0.4, 0.6])
    F.write_measure_csv(a, str(tmp_path / "a.csv"))
    F.write_measure_csv(b, str(tmp_path / "b.csv"))
    plan, d = P.solve_ot_1d(a, b, P.PowerDistance(2.0))
    F.write_plan_csv(plan, str(tmp_path / "plan.csv"))
    (tmp_path / "duals.json").write_text(json.dumps({"f": (d.f + shift).tolist(),
                                                     "g": d.g.tolist()}))
    assert cli.main(["certify", str(tmp_path / "a.csv"), str(tmp_path / "b.csv"), "--plan",
                     str(tmp_path / "plan.csv"), "--duals", str(tmp_path / "duals.json")]) == code
    assert json.loads(capsys.readouterr().out.strip())["passed"] == (code == 0)
