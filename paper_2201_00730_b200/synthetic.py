"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference publishes no dataset for these paths; every
config is synthetic.  The reference's own generator (`src/synthetic.py:12-49`)
draws two-bump mixtures for its CLI and is not used by any config, so the
generators below follow the BASELINE.json text literally.  Choices the text
leaves open are pinned here and recorded in DESIGN.md §"Synthetic inputs":

* cfg1 "Gaussian" = the normalised pdf (SURVEY.md §8d ambiguity note).
* cfg3 mixture component weights are equal; eps = 1e-2 * max_ij |x_i - y_j|^2
  computed exactly in fp64 (the maximum is attained on convex-hull vertices).
* cfg5 mixtures: means U[0.1, 0.9], std U[0.02, 0.1], weights Dirichlet(1);
  a relative floor of 1e-3 * max(pdf) is added before the mass rescale so the
  cumulative masses carry no sub-ulp atoms (SURVEY.md §0 finding 8).

Seeds: ``numpy.random.default_rng(SeedSequence(base).spawn(B)[b])``, one stream
per problem, as SURVEY.md §8d prescribes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "cfg1_inputs",
    "cfg2_batch",
    "cfg3_inputs",
    "cfg4_batch",
    "cfg5_batch",
    "max_sq_distance",
    "gaussian_pdf",
    "mixture_measure",
    "uniform_measure",
]


def gaussian_pdf(x, mean, std):
    return np.exp(-0.5 * ((x - mean) / std) ** 2) / (std * np.sqrt(2.0 * np.pi))


@dataclass(frozen=True)
class Cfg1:
    x: np.ndarray
    y: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray
    eps: float = 1e-2
    rho: float = 1.0
    iters: int = 1000


def cfg1_inputs(n=256):
    """cfg1: N=M=256 on linspace(0,1); two-bump alpha (mass 1), one-bump beta (mass 1.5)."""
    x = np.linspace(0.0, 1.0, n)
    a = 0.5 * gaussian_pdf(x, 0.2, 0.05) + 0.5 * gaussian_pdf(x, 0.4, 0.05) + 1e-3
    a *= 1.0 / a.sum()
    b = gaussian_pdf(x, 0.7, 0.1) + 1e-3
    b *= 1.5 / b.sum()
    return Cfg1(x=x, y=x.copy(), alpha=a, beta=b)


def _children(seed, count):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(count)]


def _exp_weights(rng, n):
    w = rng.exponential(1.0, n)
    return w * (rng.uniform(0.5, 2.0) / w.sum())


def cfg2_batch(batch=4096, n=1024, m=1024, seed=2022, start=0, count=None):
    """cfg2: B sorted-uniform 1-D problems with Exp(1) weights, masses U[0.5, 2].

    Returns arrays (x, y, a, b) of shapes (count, n) / (count, m) for problems
    ``start .. start+count-1`` of the seeded batch (problem b always gets the
    same stream regardless of the slice requested).
    """
    count = batch - start if count is None else count
    rngs = _children(seed, batch)[start:start + count]
    x = np.empty((count, n))
    y = np.empty((count, m))
    a = np.empty((count, n))
    b = np.empty((count, m))
    for k, rng in enumerate(rngs):
        x[k] = np.sort(rng.uniform(0.0, 1.0, n))
        y[k] = np.sort(rng.uniform(0.0, 1.0, m))
        a[k] = _exp_weights(rng, n)
        b[k] = _exp_weights(rng, m)
    return x, y, a, b


def _mixture_points(rng, n, d, comps, std):
    means = rng.uniform(-1.0, 1.0, (comps, d))
    lab = rng.integers(0, comps, n)
    return means[lab] + std * rng.standard_normal((n, d))


def max_sq_distance(x, y):
    """Exact max_ij |x_i - y_j|^2 in fp64 (attained on hull vertices for d = 2)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape[1] == 2 and len(x) > 16 and len(y) > 16:
        from scipy.spatial import ConvexHull

        x = x[ConvexHull(x).vertices]
        y = y[ConvexHull(y).vertices]
    best = 0.0
    for s in range(0, len(x), 4096):
        blk = x[s:s + 4096]
        d2 = (blk[:, None, :] - y[None, :, :]) ** 2
        best = max(best, float(d2.sum(axis=2).max()))
    return best


@dataclass(frozen=True)
class Cfg3:
    x: np.ndarray
    y: np.ndarray
    alpha: np.ndarray
    beta: np.ndarray
    eps: float
    rho: float = 1.0
    iters: int = 200


def cfg3_inputs(n=65536, m=None, seed=2023, comps=8, std=0.1):
    """cfg3: two independently seeded 8-component 2-D Gaussian mixtures."""
    m = n if m is None else m
    rx, ry = _children(seed, 2)
    x = _mixture_points(rx, n, 2, comps, std)
    y = _mixture_points(ry, m, 2, comps, std)
    alpha = np.full(n, 1.0 / n)
    beta = np.full(m, 1.3 / m)
    eps = 1e-2 * max_sq_distance(x, y)
    return Cfg3(x=x, y=y, alpha=alpha, beta=beta, eps=eps)


def cfg4_batch(batch=256, n=4096, m=4096, d=64, seed=2024, start=0, count=None):
    """cfg4: unit-sphere standard-normal features, Exp(1) weights with masses U[0.5, 2]."""
    count = batch - start if count is None else count
    rngs = _children(seed, batch)[start:start + count]
    x = np.empty((count, n, d))
    y = np.empty((count, m, d))
    a = np.empty((count, n))
    b = np.empty((count, m))
    for k, rng in enumerate(rngs):
        xx = rng.standard_normal((n, d))
        yy = rng.standard_normal((m, d))
        x[k] = xx / np.linalg.norm(xx, axis=1, keepdims=True)
        y[k] = yy / np.linalg.norm(yy, axis=1, keepdims=True)
        a[k] = _exp_weights(rng, n)
        b[k] = _exp_weights(rng, m)
    return x, y, a, b


CFG4_EPS = 0.05
CFG4_RHO = 0.5


def cfg5_batch(batch=64, k=16, n=8192, seed=2025, start=0, count=None, floor=1e-3):
    """cfg5: K sorted-uniform supports per problem, 3-component mixture densities.

    Returns (x, w) of shape (count, k, n).  Barycentric weights are 1/K and
    rho = 1 (KL), per BASELINE.json config 5.
    """
    count = batch - start if count is None else count
    rngs = _children(seed, batch)[start:start + count]
    x = np.empty((count, k, n))
    w = np.empty((count, k, n))
    for p, rng in enumerate(rngs):
        for q in range(k):
            pts = np.sort(rng.uniform(0.0, 1.0, n))
            means = rng.uniform(0.1, 0.9, 3)
            stds = rng.uniform(0.02, 0.1, 3)
            mix = rng.dirichlet(np.ones(3))
            dens = sum(mix[c] * gaussian_pdf(pts, means[c], stds[c]) for c in range(3))
            dens = dens + floor * dens.max()
            x[p, q] = pts
            w[p, q] = dens * (rng.uniform(0.5, 2.0) / dens.sum())
    return x, w


# -- CLI generators (src/synthetic.py:12-49), same draws per seed ------------


def mixture_measure(n, seed, sigma=0.03, mu1_range=(0.1, 0.4), mu2_range=(0.6, 0.9),
                    amp_range=(0.1, 0.8)):
    """Two-bump empirical mixture with equal atom weights 1/n: centres from
    the two ranges, amplitudes from ``amp_range``, each sample assigned to
    the first bump with probability a/(a+b).  Returns (measure, params)."""
    from .measures import DiscreteMeasure

    if n < 1:
        raise ValueError("need at least one sample")
    rng = np.random.default_rng(seed)
    centre1, centre2 = float(rng.uniform(*mu1_range)), float(rng.uniform(*mu2_range))
    amp1, amp2 = float(rng.uniform(*amp_range)), float(rng.uniform(*amp_range))
    first = rng.random(n) < amp1 / (amp1 + amp2)
    z = rng.normal(0.0, 1.0, n)
    pts = np.where(first, centre1 + sigma * z, centre2 + sigma * z)
    return (DiscreteMeasure(pts, np.full(n, 1.0 / n)),
            {"sigma": sigma, "mu1": centre1, "mu2": centre2, "a": amp1, "b": amp2})


def uniform_measure(n, seed, lo=0.0, hi=1.0):
    """n atoms drawn uniformly on [lo, hi], weights 1/n."""
    from .measures import DiscreteMeasure

    if n < 1:
        raise ValueError("need at least one sample")
    pts = np.random.default_rng(seed).uniform(lo, hi, n)
    return DiscreteMeasure(pts, np.full(n, 1.0 / n)), {"lo": lo, "hi": hi}
