"""File formats of the reference, byte-compatible.

Measures: CSV with header ``x,w`` (optional leading ``# comment`` lines,
``repr`` floats, ``\\n`` line ends; src/measures.py:185-254) or JSON
``{"points": [...], "weights": [...]}``.  Plans: ``i,j,mass``
(src/ot1d.py:188-215) and ``i1,...,iK,mass`` (src/barycenter.py:446-475).
Traces: ``iter,delta_f,err_f,err_g,wall_ns`` (src/sinkhorn.py:349-373) and
``iter,h0,fw_gap,pd_gap,wall_ns`` (src/fw.py:360-381).

Readers skip ``#`` lines and blank rows and validate the header; measures are
sorted / validated by ``DiscreteMeasure``.  Writers accept a path or a text
buffer, like the reference.
"""

from __future__ import annotations

import contextlib
import csv
import io
import json

import numpy as np

from .measures import DiscreteMeasure


def _num(v):
    return repr(float(v))


@contextlib.contextmanager
def _text_out(target):
    if isinstance(target, (str, bytes)):
        with open(target, "w", encoding="utf-8", newline="") as fh:
            yield fh
    else:
        yield target


@contextlib.contextmanager
def _text_in(source):
    if isinstance(source, (str, bytes)):
        with open(source, "r", encoding="utf-8", newline="") as fh:
            yield fh
    else:
        yield source


def _emit(target, header, rows, comments=()):
    with _text_out(target) as out:
        for line in comments:
            out.write(f"# {line}\n")
        out.write(",".join(header) + "\n")
        for row in rows:
            out.write(",".join(row) + "\n")


def _rows(source):
    """Non-comment, non-empty CSV rows of a text source."""
    with _text_in(source) as src:
        data = [ln for ln in src if not ln.startswith("#")]
    return [r for r in csv.reader(data) if r]


# -- measures ----------------------------------------------------------------


def write_measure_csv(measure, path_or_buf, header_comments=()):
    _emit(path_or_buf, ("x", "w"),
          ((_num(x), _num(w)) for x, w in zip(measure.points, measure.weights)), header_comments)


def read_measure_csv(path_or_buf):
    rows = _rows(path_or_buf)
    if not rows or [c.strip() for c in rows[0]] != ["x", "w"]:
        raise ValueError("measure CSV must start with header 'x,w'")
    try:
        pts = [float(r[0]) for r in rows[1:]]
        wts = [float(r[1]) for r in rows[1:]]
    except (IndexError, ValueError) as exc:
        raise ValueError(f"malformed measure CSV row: {exc}") from exc
    return DiscreteMeasure(pts, wts)


def measure_to_csv_text(measure, header_comments=()):
    buf = io.StringIO()
    write_measure_csv(measure, buf, header_comments)
    return buf.getvalue()


def write_measure_json(measure, path_or_buf):
    doc = {"points": [float(v) for v in measure.points],
           "weights": [float(v) for v in measure.weights]}
    if isinstance(path_or_buf, (str, bytes)):
        with open(path_or_buf, "w", encoding="utf-8") as fh:
            json.dump(doc, fh)
    else:
        json.dump(doc, path_or_buf)


def read_measure_json(path_or_buf):
    if isinstance(path_or_buf, (str, bytes)):
        with open(path_or_buf, "r", encoding="utf-8") as fh:
            doc = json.load(fh)
    else:
        doc = json.load(path_or_buf)
    return DiscreteMeasure(doc["points"], doc["weights"])


def load_measure(path):
    """CLI rule (src/cli.py:61-64): ``.json`` -> JSON, anything else -> CSV."""
    return read_measure_json(path) if path.endswith(".json") else read_measure_csv(path)


# -- plans -------------------------------------------------------------------


def write_plan_csv(plan, path_or_buf):
    _emit(path_or_buf, ("i", "j", "mass"),
          ((str(int(i)), str(int(j)), _num(w))
           for i, j, w in zip(plan.source_idx, plan.target_idx, plan.mass)))


def read_plan_csv(path_or_buf):
    from .ot1d import SparsePlan

    rows = _rows(path_or_buf)
    if not rows or [c.strip() for c in rows[0]] != ["i", "j", "mass"]:
        raise ValueError("plan CSV must start with header 'i,j,mass'")
    body = rows[1:]
    return SparsePlan(np.array([int(r[0]) for r in body]), np.array([int(r[1]) for r in body]),
                      np.array([float(r[2]) for r in body]))


def write_multiplan_csv(plan, path_or_buf):
    head = tuple(f"i{k + 1}" for k in range(plan.k)) + ("mass",)
    _emit(path_or_buf, head,
          (tuple(str(int(i)) for i in idx) + (_num(m),) for idx, m in zip(plan.indices, plan.mass)))


def read_multiplan_csv(path_or_buf):
    from .barycenter import MultiPlan

    rows = _rows(path_or_buf)
    if not rows or not rows[0] or rows[0][-1].strip() != "mass":
        raise ValueError("multimarginal plan CSV must end with a 'mass' column")
    k = len(rows[0]) - 1
    body = rows[1:]
    return MultiPlan(np.array([[int(c) for c in r[:k]] for r in body], dtype=np.int64).reshape(-1, k),
                     np.array([float(r[k]) for r in body]))


# -- traces ------------------------------------------------------------------


def write_trace_csv(report, path_or_buf):
    """Sinkhorn trace; the err columns stay empty without a reference."""
    tr = report.trace
    ef, eg = tr.get("err_f"), tr.get("err_g")

    def row(t):
        return (str(t + 1), _num(tr["delta_f"][t]), "" if ef is None else _num(ef[t]),
                "" if eg is None else _num(eg[t]), str(int(tr["wall_ns"][t])))

    _emit(path_or_buf, ("iter", "delta_f", "err_f", "err_g", "wall_ns"),
          (row(t) for t in range(report.iterations)))


def write_gap_csv(report, path_or_buf):
    """Frank-Wolfe trace (h0, fw_gap, pd_gap per iteration)."""
    tr = report.trace
    _emit(path_or_buf, ("iter", "h0", "fw_gap", "pd_gap", "wall_ns"),
          ((str(t + 1), _num(tr["h0"][t]), _num(tr["fw_gap"][t]), _num(tr["pd_gap"][t]),
            str(int(tr["wall_ns"][t]))) for t in range(report.iterations)))
