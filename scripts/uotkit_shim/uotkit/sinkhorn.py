from paper_2201_00730_b200.sinkhorn import *  # noqa
import numpy as _np
from paper_2201_00730_b200.entropies import logdotexp as _lde


def _smin_cols(C, pot, eps, weights):
    C = _np.asarray(C, dtype=_np.float64)
    return -eps * _np.asarray(_lde((_np.asarray(pot)[:, None] - C) / eps, weights, axis=0))


def _smin_rows(C, pot, eps, weights):
    C = _np.asarray(C, dtype=_np.float64)
    return -eps * _np.asarray(_lde((_np.asarray(pot)[None, :] - C) / eps, weights, axis=1))
