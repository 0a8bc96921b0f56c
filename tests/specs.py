"""Problem specs shared by the tests (restated from the reference problem.py:31-106;
pure numpy, usable by both the oracle and the product)."""

import numpy as np


def _parts(x, y):
    return x * (x - 1.0), y * (y - 1.0), np.exp(-x * x - y * y)


def bump_u(x, y):
    P, Q, E = _parts(x, y)
    return P * Q * E


def tanh_K(x, y):
    return np.tanh(x + y) + 1.0


def bump_f(x, y):
    P, Q, E = _parts(x, y)
    Px = (2.0 * x - 1.0) - 2.0 * x * P
    Qy = (2.0 * y - 1.0) - 2.0 * y * Q
    Pxx = (2.0 + 4.0 * x - 6.0 * x * x) - 2.0 * x * Px
    Qyy = (2.0 + 4.0 * y - 6.0 * y * y) - 2.0 * y * Qy
    t = np.tanh(x + y)
    return -((1.0 - t * t) * (Px * Q * E + P * Qy * E) + (t + 1.0) * (Pxx * Q * E + Qyy * P * E))


def zero(x, y):
    return np.zeros_like(np.asarray(x, float))


def one(x, y):
    return np.ones_like(np.asarray(x, float))


def manufactured(spec_cls, tau=1.0):
    """problem.py:80-89 (tanh coefficient, bump solution) as spec_cls(K, f, g, tau)."""
    return spec_cls(tanh_K, bump_f, bump_u, tau)


def constant(spec_cls, value=0.0, kappa=1.0, tau=1.0):
    return spec_cls(lambda x, y: np.full_like(np.asarray(x, float), kappa), zero,
                    lambda x, y: np.full_like(np.asarray(x, float), value), tau)


def hetero_K(n, seed=2, lo=1e-2, hi=1e2):
    rng = np.random.default_rng(seed)
    return np.exp(rng.uniform(np.log(lo), np.log(hi), (n, n)))
