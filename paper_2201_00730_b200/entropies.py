"""Marginal penalty specifications (src/entropies.py:40-64).

The B200 kernels implement the KL family, which is what every BASELINE
config uses; Balanced and Berg are accepted as types so that the reference's
validation order is preserved, and the solvers raise
UnsupportedEntropyError for them ("Out of scope").
"""

from __future__ import annotations

import math
from dataclasses import dataclass


def _check_rho(rho):
    if not (isinstance(rho, (int, float)) and math.isfinite(rho) and rho > 0):
        raise ValueError("rho must be positive and finite")


@dataclass(frozen=True)
class KL:
    """KL marginal penalty rho * KL(. | nu), rho > 0."""

    rho: float = 1.0

    def __post_init__(self):
        _check_rho(self.rho)


@dataclass(frozen=True)
class Berg:
    """Berg marginal penalty rho * (sum log(nu/mu) ...): F and G Sinkhorn steps
    run it on the device (aprox by per-element Newton, lambda* by Newton)."""

    rho: float = 1.0

    def __post_init__(self):
        _check_rho(self.rho)


@dataclass(frozen=True)
class Balanced:
    """Hard marginal constraint (aprox = identity): F Sinkhorn steps only."""


def ent_code(spec):
    """UOT_ENT_* code of an entropy spec (include/uot_b200.h)."""
    from .exceptions import UnsupportedEntropyError

    if isinstance(spec, KL):
        return 0
    if isinstance(spec, Berg):
        return 1
    if isinstance(spec, Balanced):
        return 2
    raise UnsupportedEntropyError(f"unknown entropy {spec!r}")


def ent_rho(spec):
    return float(getattr(spec, "rho", 1.0))


def require_kl(*specs, what="this solver"):
    from .exceptions import UnsupportedEntropyError

    for s in specs:
        if not isinstance(s, KL):
            raise UnsupportedEntropyError(f"{what} runs KL penalties on the B200 path, got {s!r}")
