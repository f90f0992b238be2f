from paper_2201_00730_b200.duality import *  # noqa
import numpy as _np
from paper_2201_00730_b200.entropies import KL as _KL, Berg as _Berg


def _neg_conj_neg_sum(spec, weights, pot):
    w = _np.asarray(weights, dtype=_np.float64)
    pot = _np.asarray(pot, dtype=_np.float64)
    with _np.errstate(all="ignore"):
        if isinstance(spec, _KL):
            vals = spec.rho * (1.0 - _np.exp(-pot / spec.rho))
        elif isinstance(spec, _Berg):
            vals = _np.where(pot > -spec.rho, spec.rho * _np.log1p(pot / spec.rho), -_np.inf)
        else:
            vals = pot
        return float(_np.dot(w, _np.where(w > 0, vals, 0.0)))
