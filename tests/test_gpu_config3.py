"""configs[2]'s solver at reduced size against the oracle: the configs[2] coefficient law
(piecewise-constant isotropic K, log-uniform in [1e-2, 1e2], seed 2; b ~ U[-1, 1] from the same
generator), p = 8, the reference's own smoother (baseline FSAI, multigrid.py:47-173, set up on
the device) inside MG-preconditioned CG (trace.py:142-163, multigrid.py:457-463).

Same PCG iteration count, per-iteration residual ratios within 1e-5, both at <= 1e-10.
"""

import numpy as np
import pytest

import specs
from oracle import hdg_oracle as O

pytestmark = pytest.mark.gpu


def config3_law(n, p):
    rng = np.random.default_rng(2)
    Kg = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), (n, n)))
    b = rng.uniform(-1.0, 1.0, 2 * n * (n - 1) * (p + 1))
    return Kg, b


@pytest.mark.parametrize("n", [32, 64])
def test_config3_law_fsai_pcg_matches_oracle(P, n):
    p = 8
    Kg, b = config3_law(n, p)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother="baseline")
    assert all(isinstance(lev.smoother, P.mg.StructuredFSAI) for lev in levels[:-1])
    x, it = levels[0].system.solve_cg(tol=1e-10, precond=P.mg.mg_preconditioner(levels), b=b)
    h = np.asarray(levels[0].system.cg_residuals)
    lo = O.build_levels(O.Grid(n, n), p, O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0),
                        smoother="baseline")
    ho = []
    xo, ito = lo[0].system.solve_cg(b=b, tol=1e-10, precond=O.mg_preconditioner(lo), hist=ho)
    ho = np.asarray(ho)
    assert it == ito
    assert len(h) == len(ho) == it + 1
    rho, rho_o = h[1:] / h[:-1], ho[1:] / ho[:-1]
    assert np.abs(rho - rho_o).max() <= 1e-5 * rho_o.max()
    bn = np.linalg.norm(b)
    assert h[-1] <= 1e-10 * bn and ho[-1] <= 1e-10 * bn
    assert np.abs(h[-1] - ho[-1]) <= 1e-10 * bn
    assert np.abs(x - xo).max() <= 1e-9 * np.abs(xo).max()
    # lambda_max of every level's FSAI (seed-1234 power iteration) as the oracle's
    lam = np.array([lev.smoother.lam_max for lev in levels[:-1]])
    lam_o = np.array([lev.smoother.lam_max for lev in lo[:-1]])
    assert np.abs(lam - lam_o).max() <= 1e-9 * lam_o.max()
