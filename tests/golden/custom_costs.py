"""Custom tuple costs for the costfn parity cases (test infrastructure:
imported by make_golden.py::gen_mot_custom and tests/test_mot_custom_gpu.py,
so the reference and the B200 path evaluate the same callables)."""

import numpy as np


def pairwise_pow15(points):
    """sum_{k<l} |x_k - x_l|^1.5."""
    p = np.asarray(points, dtype=np.float64)
    d = np.abs(p[:, None] - p[None, :])
    return float(np.sum(np.triu(d, 1) ** 1.5))


def spread(points):
    """max_k x_k - min_k x_k."""
    p = np.asarray(points, dtype=np.float64)
    return float(p.max() - p.min())


def plain_barycentric(w):
    """The barycentric cost as an anonymous callable (no .weights attribute,
    so the B200 path treats it as a custom cost)."""
    w = np.asarray(w, dtype=np.float64)

    def cost(points):
        p = np.asarray(points, dtype=np.float64)
        b = float(np.dot(w, p))
        return float(np.dot(w, (p - b) ** 2))

    return cost


COSTS = {"pow15": lambda w: pairwise_pow15, "spread": lambda w: spread,
         "bary": plain_barycentric}
