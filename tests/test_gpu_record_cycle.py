"""GPU parity of the record-layout multigrid cycle (hdg_soa_cycle.cuh; hdgb200.h:
hdg_mg_set_records) against the CPU oracle's cycle (oracle/hdg_oracle.py: cycle, restating
multigrid.py:393-406) and against the reference-layout device cycle."""

import numpy as np
import pytest

import specs
from oracle import hdg_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def _hier(P, nx, ny, p):
    levels = P.mg.build_hierarchy(P.mesh(nx, ny), p, specs.constant(P.pb.ProblemSpec), smoother="blockjacobi",
                                  omega=0.8)
    lo = O.build_levels(O.Grid(nx, ny), p, specs.constant(O.Spec), smoother="blockjacobi")
    return levels, lo


@pytest.mark.parametrize("nx,ny,p", [(16, 16, 1), (32, 32, 2), (40, 24, 3), (64, 64, 4), (36, 44, 5), (24, 24, 8),
                                     (66, 8, 2), (8, 70, 4), (2, 2, 3), (4, 2, 2), (16, 16, 10), (20, 12, 12)])
def test_record_vcycle_matches_oracle(P, nx, ny, p):
    levels, lo = _hier(P, nx, ny, p)
    rng = np.random.default_rng(nx * 100 + p)
    b = rng.uniform(-1, 1, levels[0].ndof)
    P.mg.set_records(levels, 2)
    x = P.mg.v_cycle(levels, b)
    m = p if len(levels) > p else 0                        # the whole p-ladder of the fine mesh, if h-linked
    assert P.mg.record_levels(levels) == m
    xo = O.v_cycle(lo, b)
    assert rel(x, xo) < TOL
    x0 = rng.standard_normal(levels[0].ndof)
    assert rel(P.mg.v_cycle(levels, b, x0), O.v_cycle(lo, b, x0)) < TOL
    # unfused p-prolongation and the reference-layout cycle give the same iterate to rounding
    P.mg.set_records(levels, 3)
    assert rel(P.mg.v_cycle(levels, b), x) < 1e-13
    P.mg.set_records(levels, 0)
    assert P.mg.record_levels(levels) == m                 # unchanged until the next cycle
    xr = P.mg.v_cycle(levels, b)
    assert P.mg.record_levels(levels) == 0
    assert rel(x, xr) < 1e-13
    P.mg.set_records(levels, 1)


@pytest.mark.parametrize("nu1,nu2,visits", [(1, 1, 1), (0, 2, 1), (2, 0, 1), (3, 3, 1), (2, 2, 2), (1, 2, 2)])
def test_record_cycle_sweep_counts_and_w(P, nu1, nu2, visits):
    levels, lo = _hier(P, 32, 32, 3)
    b = np.random.default_rng(7).uniform(-1, 1, levels[0].ndof)
    P.mg.set_records(levels, 2)
    run = P.mg.v_cycle if visits == 1 else P.mg.w_cycle
    x = run(levels, b, None, nu1, nu2)
    assert P.mg.record_levels(levels) == 3
    xo = O.cycle(lo, 0, b, np.zeros_like(b), nu1, nu2, visits)
    assert rel(x, xo) < TOL
    P.mg.set_records(levels, 1)


def test_record_cycle_config1_solve(P, golden):
    """configs[0] through the record cycle: the reference's 92 cycles and rho = 0.80898."""
    g = golden("config1.npz")
    levels = P.mg.build_hierarchy(P.mesh(64, 64), 2, P.pb.config1_problem(), smoother=None)[:6]
    P.mg.attach_smoothers(levels, "blockjacobi", 0.8)
    P.mg.set_records(levels, 2)
    b = levels[0].rhs
    x1 = P.mg.v_cycle(levels, b)
    assert P.mg.record_levels(levels) == 2
    assert rel(x1, g["x1"]) < TOL
    x, mon = P.mg.solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    assert len(mon.residuals) - 1 == 92
    assert abs(mon.asymptotic_rate() - 0.80898) < 1e-5
    assert rel(x, g["x"]) < 1e-10
    x, it = levels[0].system.solve_cg(tol=1e-10, precond=P.mg.mg_preconditioner(levels), b=b)
    P.mg.set_records(levels, 0)
    x2, it2 = levels[0].system.solve_cg(tol=1e-10, precond=P.mg.mg_preconditioner(levels), b=b)
    assert it == it2 and rel(x, x2) < 1e-9
    P.mg.set_records(levels, 1)


def test_record_cycle_skips_unqualified_hierarchies(P):
    """Stored (heterogeneous K) levels and FSAI-smoothed levels stay on the reference layout."""
    Kg = specs.hetero_K(16, seed=5)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(16, 16), 2, spec, smoother="blockjacobi", omega=0.8)
    P.mg.set_records(levels, 2)
    b = np.random.default_rng(3).uniform(-1, 1, levels[0].ndof)
    P.mg.v_cycle(levels, b)
    assert P.mg.record_levels(levels) == 0
    levels = P.mg.build_hierarchy(P.mesh(16, 16), 2, specs.constant(P.pb.ProblemSpec), smoother="baseline")
    P.mg.set_records(levels, 2)
    P.mg.v_cycle(levels, np.random.default_rng(3).uniform(-1, 1, levels[0].ndof))
    assert P.mg.record_levels(levels) == 0


def test_record_cycle_full_size_configs1(P):
    """configs[1]'s hierarchy (1024^2, p = 4, K = I): automatic record cycle, same iterate as the
    reference-layout cycle (itself pinned to the oracle at small sizes) and a contracting residual."""
    levels = P.mg.build_hierarchy(P.mesh(1024, 1024), 4, P.pb.constant_problem(0.0, 1.0), smoother="blockjacobi",
                                  omega=0.8)
    import torch
    b = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, levels[0].ndof)).cuda()
    x = P.mg.v_cycle(levels, b)
    assert P.mg.record_levels(levels) == 7                 # the p-ladder and the 512^2, 256^2, 128^2 levels (>= 50k dofs)
    P.mg.set_records(levels, 0)
    xr = P.mg.v_cycle(levels, b)
    assert P.mg.record_levels(levels) == 0
    err = float((x - xr).abs().max() / xr.abs().max())
    assert err < 1e-12
    r = b - levels[0].system.matvec_free(x)
    assert float(r.norm() / b.norm()) < 0.5


@pytest.mark.parametrize("nx,ny,p,nu1,nu2,visits", [(64, 64, 4, 2, 2, 1), (40, 24, 3, 0, 1, 1), (32, 32, 2, 1, 0, 2),
                                                   (16, 16, 1, 0, 2, 1)])
def test_cycle_on_resident_records(P, nx, ny, p, nu1, nu2, visits):
    """hdg_mg_cycle_records: b and x stay facet records; x0 is not mutated, x may alias x0."""
    levels, lo = _hier(P, nx, ny, p)
    P.mg.set_records(levels, 2)
    sysf = levels[0].system
    rng = np.random.default_rng(11)
    b, x0 = rng.uniform(-1, 1, sysf.ndof), rng.standard_normal(sysf.ndof)
    P.mg.v_cycle(levels, b)                                   # sets the record levels up
    bp, x0p = sysf.facet_planes(b), sysf.facet_planes(x0)
    x = P.mg.cycle_records(levels, bp, None, nu1, nu2, visits).numpy()
    assert rel(x, O.cycle(lo, 0, b, np.zeros_like(b), nu1, nu2, visits)) < TOL
    xo = O.cycle(lo, 0, b, x0.copy(), nu1, nu2, visits)
    x2 = P.mg.cycle_records(levels, bp, x0p, nu1, nu2, visits)
    assert rel(x2.numpy(), xo) < TOL
    np.testing.assert_array_equal(x0p.numpy(), x0)            # x0 untouched
    P.mg.cycle_records(levels, bp, x0p, nu1, nu2, visits, out=x0p)   # in place
    assert rel(x0p.numpy(), xo) < TOL
    np.testing.assert_array_equal(bp.numpy(), b)
    P.mg.set_records(levels, 1)


@pytest.mark.parametrize("nx,ny,p,visits", [(64, 64, 2, 1), (32, 32, 1, 1), (96, 40, 3, 1), (64, 32, 4, 2)])
def test_record_cycle_with_h_levels_on_records(P, nx, ny, p, visits):
    """Mode 4: the h-coarsened p = 1 levels keep their vectors as records too (record-to-record
    h-transfers, hdg_soa_cycle.cuh: soa_h_restrict_kernel / soa_h_prolong_kernel with CREC)."""
    levels, lo = _hier(P, nx, ny, p)
    rng = np.random.default_rng(5 * nx + p)
    b, x0 = rng.uniform(-1, 1, levels[0].ndof), rng.standard_normal(levels[0].ndof)
    P.mg.set_records(levels, 4)
    run = P.mg.v_cycle if visits == 1 else P.mg.w_cycle
    x = run(levels, b)
    assert P.mg.record_levels(levels) > p                  # at least one h-level beyond the p-ladder
    assert rel(x, O.cycle(lo, 0, b, np.zeros_like(b), 2, 2, visits)) < TOL
    assert rel(run(levels, b, x0), O.cycle(lo, 0, b, x0.copy(), 2, 2, visits)) < TOL
    P.mg.set_records(levels, 1)
