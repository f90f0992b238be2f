"""run(..., reference=) error traces for penalties off the KL closed form
(src/sinkhorn.py:246-315) vs the reference (tests/golden/sk_trace.npz): F
with Berg / Balanced marginals (untranslated iterates) and G with a Berg
marginal (translated by the Newton lambda*, csrc/fw1d_generic.cu)."""

import numpy as np
import pytest

import paper_2201_00730_b200 as P
from conftest import golden

pytestmark = pytest.mark.gpu


def _ent(code, rho):
    return [P.KL, P.Berg, None][int(code)](float(rho)) if int(code) < 2 else P.Balanced()


@pytest.mark.parametrize("k", range(4))
def test_error_traces_match_reference(k):
    z = golden("sk_trace.npz")
    var, c1, r1, c2, r2 = z[f"c{k}_par"]
    variant = "f" if int(var) == 0 else "g"
    prob = P.UotProblem(P.DiscreteMeasure(z[f"c{k}_x"], z[f"c{k}_a"]),
                        P.DiscreteMeasure(z[f"c{k}_y"], z[f"c{k}_b"]), P.PowerDistance(2.0),
                        _ent(c1, r1), _ent(c2, r2), eps=0.2)
    ref = P.DualPair(z[f"c{k}_ref_f"], z[f"c{k}_ref_g"])
    rep = P.run(prob, P.SinkhornConfig(variant, 25, 1e-15), reference=ref)
    # the stopping test sits at delta ~ 1e-15 (rounding): compare the common prefix
    want = z[f"c{k}_err_f"]
    L = min(len(want), rep.iterations)
    assert abs(len(want) - rep.iterations) <= 3
    for key in ("delta_f", "err_f", "err_g"):
        np.testing.assert_allclose(rep.trace[key][:L], z[f"c{k}_{key}"][:L], rtol=1e-8, atol=1e-11,
                                   err_msg=key)
