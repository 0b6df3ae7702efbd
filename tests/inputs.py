"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests
and bench.py.  No arithmetic of the method lives here: only numpy random
draws with the shapes / ranges of the paper's workload (DESIGN.md "Input
recipe")."""
import numpy as np


def raw_params(seed, k, scale=1.0):
    """Unconstrained generator outputs [k, 6] ~ N(0, scale^2)."""
    return np.random.default_rng(seed).normal(scale=scale, size=(k, 6))


def coefficients(seed, k):
    """Valid quantile coefficients [k, 6] (c1, c2 > 0) spanning the
    histogram window [0, 4): c0 in [0, 2), c1, c2 in (0, 1]."""
    rng = np.random.default_rng(seed)
    c = np.empty((k, 2, 3))
    c[:, :, 0] = rng.uniform(0.0, 2.0, size=(k, 2))
    c[:, :, 1] = rng.uniform(0.01, 1.0, size=(k, 2))
    c[:, :, 2] = rng.uniform(0.01, 1.0, size=(k, 2))
    return c.reshape(k, 6)


def gradient_like(seed, shape, scale=1e-3):
    return np.random.default_rng(seed).normal(scale=scale, size=shape)


def sample_indices(seed, n, count):
    return np.sort(np.random.default_rng(seed).choice(n, size=min(count, n), replace=False))
