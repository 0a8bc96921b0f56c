"""Problem data (reference: problem.py:9-106) and the BASELINE config inputs.

ProblemSpec matches the reference dataclass, so reference specs work too.
`nodal_source` / `piecewise_coefficient` build the configs' "per element DOF"
source and per-element K."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .discretization import eval_matrix, gll_rule


@dataclass(frozen=True)
class ProblemSpec:
    coefficient: Callable
    source: Callable
    dirichlet: Callable
    tau: float = 1.0
    exact_u: Optional[Callable] = field(default=None)
    exact_flux: Optional[Callable] = field(default=None)

    def __post_init__(self):
        if not self.tau > 0:
            raise ValueError(f"stabilization tau must be positive, got {self.tau}")


def _full(v):
    return lambda x, y: np.full_like(np.asarray(x, dtype=float), v)


def constant_problem(value=0.0, kappa=1.0, tau=1.0):
    """problem.py:92-106."""
    return ProblemSpec(_full(float(kappa)), _full(0.0), _full(float(value)), tau, _full(float(value)),
                       lambda x, y: (_full(0.0)(x, y), _full(0.0)(x, y)))


def nodal_source(f_nodal, n, p):
    """f = sum_I f[e, I] phi_I on element e of an n x n unit-square mesh (I = a + b (p+1))."""
    basis = gll_rule(p)
    f_nodal = np.asarray(f_nodal, float)

    def src(x, y):
        x = np.asarray(x, float)
        y = np.asarray(y, float)
        i = np.clip(np.floor(x * n).astype(np.int64), 0, n - 1)
        j = np.clip(np.floor(y * n).astype(np.int64), 0, n - 1)
        Ex = eval_matrix(basis, (2.0 * (x * n - i) - 1.0).ravel())
        Ey = eval_matrix(basis, (2.0 * (y * n - j) - 1.0).ravel())
        v = f_nodal[(j * n + i).ravel()].reshape(-1, p + 1, p + 1)
        return np.einsum("qb,qa,qba->q", Ey, Ex, v).reshape(x.shape)

    return src


def piecewise_coefficient(Kgrid):
    """K = Kgrid[floor(y ny), floor(x nx)] on the unit square (element e = j nx + i)."""
    Kgrid = np.asarray(Kgrid, float)
    ny, nx = Kgrid.shape

    def coef(x, y):
        i = np.clip(np.floor(np.asarray(x, float) * nx).astype(np.int64), 0, nx - 1)
        j = np.clip(np.floor(np.asarray(y, float) * ny).astype(np.int64), 0, ny - 1)
        return Kgrid[j, i]

    return coef


def piecewise_anisotropic(Kxx, Kyy):
    """Diagonal anisotropic K = diag(Kxx, Kyy) per element (BASELINE configs[4]); the
    coefficient returns the pair, which TraceSystem treats as one flux mass per component
    (the reference's scalar coefficient cannot represent this)."""
    fx, fy = piecewise_coefficient(Kxx), piecewise_coefficient(Kyy)
    return lambda x, y: (fx(x, y), fy(x, y))


def config1_problem(n=64, p=2, seed=0):
    """BASELINE configs[0]: K = 1, g_D = 0, tau = 1, nodal f ~ U[-1, 1] (seed 0)."""
    f = np.random.default_rng(seed).uniform(-1.0, 1.0, (n * n, (p + 1) ** 2))
    return ProblemSpec(_full(1.0), nodal_source(f, n, p), _full(0.0), 1.0)
