"""The reference's own hot-path test behaviours (pkg/tests/test_trace.py, test_multigrid.py),
restated against the drop-in: same properties, sizes and criteria, each citing the reference
test it mirrors.  The reference package is not importable on the GPU box, so direct solves use
scipy on the drop-in's assembled operator (trace.py:98-131)."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import specs

pytestmark = pytest.mark.gpu


def spec_m(P):
    return specs.manufactured(P.pb.ProblemSpec)


def direct(system, b=None):
    A = system.assemble_csr()
    rhs = system.rhs if b is None else b
    return spla.spsolve(A.tocsc(), rhs) if A.shape[0] else np.zeros(0)


@pytest.fixture(scope="module")
def small(P):
    return P.tr.TraceSystem(P.mesh(4, 4), 2, spec_m(P))


@pytest.fixture(scope="module")
def h8p3(P):
    return P.mg.build_hierarchy(P.mesh(8, 8), 3, spec_m(P), smoother="baseline")


# ------------------------------------------------------------------- test_trace.py


def test_dof_counts(P):                                                    # test_trace.py:16
    s = P.tr.TraceSystem(P.mesh(2, 2), 1, spec_m(P))
    assert s.n_blocks == 4 and s.ndof == 8
    assert P.tr.TraceSystem(P.mesh(1, 1), 1, spec_m(P)).ndof == 0


def test_matvec_zero(small):                                               # test_trace.py:33
    np.testing.assert_array_equal(small.matvec_free(np.zeros(small.ndof)), 0.0)


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_matvec_free_matches_csr(P, n, p):                                 # test_trace.py:40
    s = P.tr.TraceSystem(P.mesh(n, n), p, spec_m(P))
    A = s.assemble_csr()
    rng = np.random.default_rng(n * 100 + p)
    for _ in range(20):
        x = rng.standard_normal(s.ndof)
        ref = A @ x
        assert np.abs(s.matvec_free(x) - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_matvec_deterministic(small):                                      # test_trace.py:51
    x = np.random.default_rng(0).standard_normal(small.ndof)
    np.testing.assert_array_equal(small.matvec_free(x), small.matvec_free(x))


def test_operator_symmetry(small):                                         # test_trace.py:59
    rng = np.random.default_rng(1)
    for _ in range(5):
        x, y = rng.standard_normal(small.ndof), rng.standard_normal(small.ndof)
        a, b = small.matvec_free(x) @ y, x @ small.matvec_free(y)
        assert abs(a - b) <= 1e-11 * max(1.0, abs(a))


@pytest.mark.parametrize("p", [1, 2, 3])
def test_operator_positive_definite(P, p):                                 # test_trace.py:70
    s = P.tr.TraceSystem(P.mesh(4, 4), p, spec_m(P))
    assert np.linalg.eigvalsh(s.assemble_csr().toarray()).min() > 0


def test_unit_vector_stencil(small):                                       # test_trace.py:76
    n1 = small.p + 1
    rng = np.random.default_rng(5)
    for block in rng.integers(0, small.n_blocks, size=4):
        x = np.zeros(small.ndof)
        x[block * n1] = 1.0
        y = small.matvec_free(x)
        assert np.count_nonzero(np.abs(y.reshape(-1, n1)).max(axis=1) > 0) <= 7


def test_nnz_per_row_bound(P):                                             # test_trace.py:88
    A = P.tr.TraceSystem(P.mesh(4, 4), 2, spec_m(P)).assemble_csr()
    assert np.diff(A.indptr).max() <= 7 * 3


def test_rhs_zero_for_zero_data(P):                                        # test_trace.py:95
    s = P.tr.TraceSystem(P.mesh(3, 3), 2, P.pb.constant_problem(0.0, 1.0))
    np.testing.assert_array_equal(s.rhs, 0.0)


def test_constant_solution_trace(P):                                       # test_trace.py:100
    s = P.tr.TraceSystem(P.mesh(3, 3), 2, P.pb.constant_problem(4.0, 2.0))
    np.testing.assert_allclose(direct(s), 4.0, atol=1e-12)


def test_cg_matches_direct(small):                                         # test_trace.py:115
    ref = direct(small)
    got, iters = small.solve_cg(tol=1e-13)
    assert iters < 5000
    assert np.abs(got - ref).max() < 1e-9 * np.abs(ref).max()


def test_gather_element_layout(small):                                     # test_trace.py:131
    x = np.random.default_rng(9).standard_normal(small.ndof)
    n1, nx, ny = small.p + 1, small.mesh.n_x, small.mesh.n_y
    e = 5
    i, j = e % nx, e // nx
    nh = nx * (ny - 1)
    sides = [(j - 1) * nx + i if j > 0 else -1,                  # bottom h(i, j)
             nh + i * ny + j if i < nx - 1 else -1,              # right  v(i+1, j)
             j * nx + i if j < ny - 1 else -1,                   # top    h(i, j+1)
             nh + (i - 1) * ny + j if i > 0 else -1]             # left   v(i, j)
    lam_e = small.gather_element(x, e)
    for s, blk in enumerate(sides):
        expect = np.zeros(n1) if blk < 0 else x[blk * n1:(blk + 1) * n1]
        np.testing.assert_array_equal(lam_e[s * n1:(s + 1) * n1], expect)


def test_counter_formulas(P, small):                                       # test_trace.py:144
    rows, nnz = small.ndof, small.assemble_csr().nnz
    csr = P.tr.flop_memop_count(small, "csr")
    assert csr["flops"] == 2 * nnz - rows
    assert csr["bytes"] == 8 * nnz + 4 * (nnz + rows + 1) + 8 * 2 * rows
    n1 = small.p + 1
    assert P.tr.flop_memop_count(small, "free")["flops"] == small.n_blocks * (2 * 2 * n1 * 4 * n1 - n1)
    with pytest.raises(ValueError):
        P.tr.flop_memop_count(small, "blocked")


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_free_mode_ai_beats_csr(P, p):                                     # test_trace.py:168
    s = P.tr.TraceSystem(P.mesh(8, 8), p, spec_m(P))
    assert P.tr.flop_memop_count(s, "free")["ai"] > P.tr.flop_memop_count(s, "csr")["ai"]


def test_constant_vector_annihilated_away_from_boundary(P):                # test_trace.py:174
    n, p = 6, 2
    s = P.tr.TraceSystem(P.mesh(n, n), p, P.pb.constant_problem(0.0, 1.0))
    y = s.matvec_free(np.ones(s.ndof)).reshape(-1, p + 1)
    nh = n * (n - 1)

    def interior_elem(i, j):       # all four sides of element (i, j) are interior facets
        return 1 <= i <= n - 2 and 1 <= j <= n - 2
    checked = 0
    for blk in range(s.n_blocks):
        if blk < nh:
            j, i = blk // n + 1, blk % n          # h(i, j): owners (i, j-1), (i, j)
            owners = [(i, j - 1), (i, j)]
        else:
            u = blk - nh
            i, j = u // n + 1, u % n              # v(i, j): owners (i-1, j), (i, j)
            owners = [(i - 1, j), (i, j)]
        if all(interior_elem(*o) for o in owners):
            assert np.abs(y[blk]).max() < 1e-12
            checked += 1
    assert checked > 0


# ---------------------------------------------------------------- test_multigrid.py


def test_level_schedule_p4(P):                                             # test_multigrid.py:40
    levels = P.mg.build_hierarchy(P.mesh(16, 16), 4, spec_m(P), smoother=None)
    assert [(l.mesh.n_x, l.p, l.kind) for l in levels] == [
        (16, 4, "p-level"), (16, 3, "p-level"), (16, 2, "p-level"), (16, 1, "p-level"),
        (8, 1, "h-level"), (4, 1, "h-level"), (2, 1, "coarsest")]


def test_level_count_p8(P):                                                # test_multigrid.py:49
    assert len(P.mg.build_hierarchy(P.mesh(16, 16), 8, spec_m(P), smoother=None)) == 11


def test_single_level_direct(P):                                           # test_multigrid.py:54
    levels = P.mg.build_hierarchy(P.mesh(2, 2), 1, spec_m(P), smoother="baseline")
    assert len(levels) == 1 and levels[0].kind == "coarsest"
    x, _ = P.mg.solve_mg(levels)
    np.testing.assert_allclose(x, direct(levels[0].system), atol=1e-12)


def test_coarse_cap_and_odd_mesh(P):                                       # test_multigrid.py:62, :67
    with pytest.raises(P.mg.HierarchyError):
        P.mg.build_hierarchy(P.mesh(6, 6), 2, spec_m(P), coarse_cap=10, smoother=None)
    levels = P.mg.build_hierarchy(P.mesh(6, 6), 2, spec_m(P), smoother=None)
    assert [(l.mesh.n_x, l.p) for l in levels] == [(6, 2), (6, 1), (3, 1)]


def test_p_transfer_constants_and_embedding(P):                            # test_multigrid.py:76, :84
    m = P.mesh(4, 4)
    fine, coarse = P.tr.TraceSystem(m, 3, spec_m(P)), P.tr.TraceSystem(m, 2, spec_m(P))
    Pp = P.mg.p_prolongation(fine, coarse)
    np.testing.assert_allclose(Pp @ np.ones(coarse.ndof), 1.0, atol=1e-13)

    def f(x, y):
        return x * x - 2 * x * y + 0.5 * y * y
    np.testing.assert_allclose(Pp @ P.tr.exact_trace(coarse, f), P.tr.exact_trace(fine, f), atol=1e-13)


def test_restriction_is_adjoint_of_prolongation(P):                        # test_multigrid.py:139
    from paper_1705_09907_b200.mesh import coarsen
    m = P.mesh(4, 4)
    fine, coarse = P.tr.TraceSystem(m, 1, spec_m(P)), P.tr.TraceSystem(coarsen(m), 1, spec_m(P))
    Ph = P.mg.h_prolongation(fine, coarse, spec_m(P))
    rng = np.random.default_rng(11)
    x, y = rng.standard_normal(coarse.ndof), rng.standard_normal(fine.ndof)
    a, b = (Ph @ x) @ y, x @ (Ph.T @ y)
    assert abs(a - b) < 1e-12 * max(1.0, abs(b))


def test_fsai_reference_properties(P):                                     # test_multigrid.py:153-201
    from paper_1705_09907_b200.fsai import fsai_build, NotSPDError
    s = P.tr.TraceSystem(P.mesh(4, 4), 2, spec_m(P))
    A = s.assemble_csr()
    sm = fsai_build(A, 1)
    assert abs(sm.complexity - 1.0) < 1e-12
    assert np.all(sm.G.diagonal() > 0)
    M, Ad = (sm.Gt @ sm.G).toarray(), A.toarray()
    E = np.eye(Ad.shape[0])
    for w in sm.sweep_weights(2):
        E = (np.eye(Ad.shape[0]) - w * M @ Ad) @ E
    assert np.abs(np.linalg.eigvals(E)).max() < 1.0
    big = P.tr.TraceSystem(P.mesh(16, 16), 4, spec_m(P))
    assert 2.0 <= fsai_build(big.assemble_csr(), 2).complexity <= 3.0
    with pytest.raises(NotSPDError):
        fsai_build(sp.csr_matrix(np.array([[1.0, 2.0], [2.0, 1.0]])), 1)


def test_v_cycle_zero_input_and_converges_to_direct(h8p3, P):             # test_multigrid.py:206, :212
    np.testing.assert_array_equal(P.mg.v_cycle(h8p3, np.zeros(h8p3[0].ndof)), 0.0)
    x, mon = P.mg.solve_mg(h8p3, cycle="v")
    ref = direct(h8p3[0].system)
    assert np.abs(x - ref).max() < 1e-9 * np.abs(ref).max()
    assert not mon.diverged()


@pytest.mark.parametrize("p", [2, 3])
def test_v_cycle_rate_bound_small(P, p):                                   # test_multigrid.py:220
    levels = P.mg.build_hierarchy(P.mesh(8, 8), p, spec_m(P), smoother="baseline")
    _, mon = P.mg.solve_mg(levels, cycle="v", nu1=2, nu2=2)
    assert mon.asymptotic_rate() <= 0.25


def test_v_cycle_residuals_monotone(P):                                    # test_multigrid.py:226
    levels = P.mg.build_hierarchy(P.mesh(4, 4), 2, spec_m(P), smoother="baseline")
    _, mon = P.mg.solve_mg(levels, cycle="v")
    assert all(r <= 1.0 + 1e-12 for r in mon.rho[1:])


def test_w_cycle_properties(h8p3, P):                                      # test_multigrid.py:233-252
    one = P.mg.build_hierarchy(P.mesh(2, 2), 1, spec_m(P), smoother="baseline")
    np.testing.assert_allclose(P.mg.w_cycle(one, one[0].rhs), direct(one[0].system), atol=1e-12)
    _, mv = P.mg.solve_mg(h8p3, cycle="v")
    _, mw = P.mg.solve_mg(h8p3, cycle="w")
    assert mw.asymptotic_rate() <= mv.asymptotic_rate() + 0.02
    fine = h8p3[0]
    b = fine.matvec(np.random.default_rng(21).standard_normal(fine.ndof))
    _, mon = P.mg.solve_mg(h8p3, b=b, cycle="w", max_cycles=10)
    assert all(r2 <= r1 for r1, r2 in zip(mon.residuals, mon.residuals[1:]))


def test_aggressive_rate_and_h_independence(P):                            # test_multigrid.py:267, :273
    levels = P.mg.build_hierarchy(P.mesh(8, 8), 3, spec_m(P), smoother="aggressive")
    _, mon = P.mg.solve_mg(levels, cycle="v", tol=1e-13)
    assert mon.asymptotic_rate() <= 0.05
    _, m8 = P.mg.solve_mg(P.mg.build_hierarchy(P.mesh(8, 8), 4, spec_m(P), smoother="baseline"))
    _, m16 = P.mg.solve_mg(P.mg.build_hierarchy(P.mesh(16, 16), 4, spec_m(P), smoother="baseline"))
    assert abs(m8.asymptotic_rate() - m16.asymptotic_rate()) <= 0.05


def test_fmg_single_level(P):                                              # test_multigrid.py:279
    levels = P.mg.build_hierarchy(P.mesh(2, 2), 1, spec_m(P), smoother="baseline")
    np.testing.assert_allclose(P.mg.fmg(levels), direct(levels[0].system), atol=1e-12)


def test_mg_preconditioned_cg(P):                                          # test_multigrid.py:293
    levels = P.mg.build_hierarchy(P.mesh(8, 8), 2, spec_m(P), smoother="baseline")
    s = levels[0].system
    x, iters = s.solve_cg(tol=1e-12, precond=P.mg.mg_preconditioner(levels))
    ref = direct(s)
    assert iters < 20
    assert np.abs(x - ref).max() < 1e-9 * np.abs(ref).max()


def test_attach_smoothers_modes(h8p3, P):                                  # test_multigrid.py:302
    levels = P.mg.attach_smoothers(h8p3, "baseline")
    assert levels[0].smoother.aggressiveness == 1
    with pytest.raises(ValueError):
        P.mg.attach_smoothers(levels, "extreme")
