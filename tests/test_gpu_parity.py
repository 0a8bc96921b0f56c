"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle and the
reference golden vectors.  Criterion: max|y_gpu - y_ref| <= 1e-12 ||y_ref||_inf
(stricter than the reference's own max(1, ||ref||) floor, test_trace.py:48, also checked)."""

import numpy as np
import pytest

import specs
from oracle import hdg_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)




# ------------------------------------------------------------------------------ matvec


@pytest.mark.parametrize("n,p", [(2, 1), (4, 2), (4, 3), (8, 1), (8, 2), (8, 5), (3, 2)])
def test_matvec_manufactured_golden(P, golden, n, p):
    """Stored-block path (tanh K varies per element) against reference outputs."""
    g = golden("small_systems.npz")
    s = P.tr.TraceSystem(P.mesh(n, n), p, specs.manufactured(P.pb.ProblemSpec))
    assert not s.operator.shared
    key = f"n{n}p{p}"
    y = s.matvec_free(g[key + "_x"])
    ref = g[key + "_y"]
    assert rel(y, ref) < TOL
    assert np.abs(y - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())   # test_trace.py:48


@pytest.mark.parametrize("p", list(range(1, 13)))
@pytest.mark.parametrize("shape", [(37, 21), (64, 64)])
def test_matvec_shared_all_orders(P, p, shape):
    """Shared-block path (K = I), every order the kernels are built for, ragged tiles."""
    nx, ny = shape
    s = P.tr.TraceSystem(P.mesh(nx, ny), p, specs.constant(P.pb.ProblemSpec))
    assert s.operator.shared
    S = s.operator.S_cls[0]
    o = O.OracleTrace(O.Grid(nx, ny), p, None, _blocks=np.broadcast_to(S, (nx * ny,) + S.shape).copy())
    o.schur *= o.gmask[:, None, :]
    x = np.random.default_rng(1000 * p + nx).uniform(-1, 1, s.ndof)
    assert rel(s.matvec_free(x), o.matvec(x)) < TOL


@pytest.mark.parametrize("p", [1, 2, 4, 8, 12])
def test_matvec_stored_equals_shared(P, p):
    """Same operator held both ways (stored stream vs constant bank)."""
    m = P.mesh(40, 33)
    s = P.tr.TraceSystem(m, p, specs.constant(P.pb.ProblemSpec))
    E = 40 * 33
    st = P.tr.TraceSystem.from_blocks(m, p, np.repeat(s.operator.S_cls, E, axis=0), np.arange(E))
    assert not st.operator.shared
    x = np.random.default_rng(p).standard_normal(s.ndof)
    assert rel(st.matvec_free(x), s.matvec_free(x)) < TOL


@pytest.mark.parametrize("p", [2, 4, 7])
def test_matvec_shared_asymmetric_block_falls_back(P, p):
    """A single-class block that is NOT invariant under the facet mirrors (the mirror-reduced
    constant-bank kernel would be wrong for it) is streamed as stored facets instead."""
    nx, ny = 23, 17
    s = P.tr.TraceSystem(P.mesh(nx, ny), p, specs.constant(P.pb.ProblemSpec))
    S = s.operator.S_cls[0].copy()
    rng = np.random.default_rng(p)
    Pm = rng.uniform(-0.05, 0.05, S.shape) * np.abs(S).max()
    S = S + Pm + Pm.T                          # still symmetric, no longer mirror-invariant
    m = P.mesh(nx, ny)
    a = P.tr.TraceSystem.from_blocks(m, p, S[None], np.zeros(nx * ny, np.int64))
    assert a.operator.shared
    o = O.OracleTrace(O.Grid(nx, ny), p, None, _blocks=np.broadcast_to(S, (nx * ny,) + S.shape).copy())
    o.schur *= o.gmask[:, None, :]
    x = rng.uniform(-1, 1, a.ndof)
    assert rel(a.matvec_free(x), o.matvec(x)) < TOL


@pytest.mark.parametrize("n,p", [(16, 2), (24, 4), (16, 8)])
def test_matvec_heterogeneous_vs_oracle(P, n, p):
    Kg = specs.hetero_K(n, seed=n + p)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    s = P.tr.TraceSystem(P.mesh(n, n), p, spec)
    o = O.OracleTrace(O.Grid(n, n), p, O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0))
    x = np.random.default_rng(7).uniform(-1, 1, s.ndof)
    assert rel(s.matvec_free(x), o.matvec(x)) < TOL


def test_matvec_edge_cases(P):
    s11 = P.tr.TraceSystem(P.mesh(1, 1), 2, specs.constant(P.pb.ProblemSpec))
    assert s11.ndof == 0 and s11.matvec_free(np.zeros(0)).size == 0      # trace.py:90-91
    s = P.tr.TraceSystem(P.mesh(4, 4), 2, specs.manufactured(P.pb.ProblemSpec))
    np.testing.assert_array_equal(s.matvec_free(np.zeros(s.ndof)), 0.0)   # test_trace.py:33-35
    with pytest.raises(ValueError):
        s.matvec_free(np.zeros(s.ndof + 1))
    x = np.random.default_rng(0).standard_normal(s.ndof)
    np.testing.assert_array_equal(s.matvec_free(x), s.matvec_free(x))     # determinism (:51-56)


def test_matvec_torch_zero_copy(P):
    import torch
    s = P.tr.TraceSystem(P.mesh(32, 32), 3, specs.constant(P.pb.ProblemSpec))
    x = torch.rand(s.ndof, dtype=torch.float64, device="cuda")
    y = s.matvec_free(x)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    assert rel(y.cpu().numpy(), s.matvec_free(x.cpu().numpy())) == 0.0


def test_config2_properties_full_size(P):
    """BASELINE configs[1] size (1024^2, p=4, K=I): symmetry, linearity, determinism and a
    sampled-row check against the oracle block."""
    import torch
    n, p = 1024, 4
    s = P.tr.TraceSystem(P.mesh(n, n), p, specs.constant(P.pb.ProblemSpec))
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(s.ndof, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    yv = torch.rand(s.ndof, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    Ax, Ay = s.matvec_free(x), s.matvec_free(yv)
    lhs, rhs_ = float(Ax @ yv), float(x @ Ay)
    assert abs(lhs - rhs_) <= 1e-11 * max(1.0, abs(lhs))                 # test_trace.py:59-66
    A2 = s.matvec_free(2.0 * x + yv)
    assert float((A2 - (2.0 * Ax + Ay)).abs().max()) <= 1e-12 * float(A2.abs().max())
    assert torch.equal(Ax, s.matvec_free(x))


def test_config2_full_size_vs_oracle_both_kernels(P):
    """configs[1] at full size (1024^2, p=4, K=I, x ~ U[-1,1] seed 1) against the ORACLE's own
    injected system (its element block from its own local condensation; gather / einsum /
    two-owner sum of trace.py:87-94): the reference-layout kernel (matvec_free on a vector) and
    the facet-record kernel (the bench's), both at 1e-12 relative."""
    n, p = 1024, 4
    osys = O.injected_shared_system(n, p)
    x = np.random.default_rng(1).uniform(-1.0, 1.0, osys.ndof)
    ref = osys.matvec(x)
    del osys
    s = P.tr.TraceSystem(P.mesh(n, n), p, specs.constant(P.pb.ProblemSpec))
    y_ref_layout = s.matvec_free(x)
    y_records = s.matvec_free(s.facet_planes(x)).numpy()
    assert rel(y_ref_layout, ref) < TOL
    assert rel(y_records, ref) < TOL


# ------------------------------------------------------------------------------ transfers


@pytest.mark.parametrize("tag,n,p", [("m8p3", 8, 3), ("m4p2", 4, 2)])
def test_transfers_match_golden(P, golden, tag, n, p):
    g = golden("hierarchies.npz")
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, specs.manufactured(P.pb.ProblemSpec), smoother=None)
    for k, lev in enumerate(levels):
        assert rel(lev.matvec(g[f"{tag}_L{k}_v"]), g[f"{tag}_L{k}_Av"]) < TOL
        if lev.prolong is not None:
            assert rel(lev.prolong @ g[f"{tag}_L{k}_Pv_in"], g[f"{tag}_L{k}_Pv"]) < TOL
            assert rel(lev.prolong.T @ g[f"{tag}_L{k}_v"], g[f"{tag}_L{k}_PTv"]) < TOL


def test_h_transfer_heterogeneous_vs_oracle(P):
    n = 16
    Kg = specs.hetero_K(n, seed=5)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(n, n), 2, spec, smoother=None)
    lo = O.build_levels(O.Grid(n, n), 2, O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0))
    rng = np.random.default_rng(3)
    for lev, ol in zip(levels, lo):
        v = rng.standard_normal(lev.ndof)
        assert rel(lev.matvec(v), ol.operator @ v) < TOL
        if lev.prolong is not None:
            vc = rng.standard_normal(lev.prolong.shape[1])
            assert rel(lev.prolong @ vc, ol.prolong @ vc) < TOL
            assert rel(lev.prolong.T @ v, ol.prolong.T @ v) < TOL


# ------------------------------------------------------------------------------- cycles


def history_close(got, ref):
    got, ref = np.asarray(got), np.asarray(ref)
    assert got.shape == ref.shape, (got.shape, ref.shape)       # identical iteration counts
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-10 * ref[0])


@pytest.mark.parametrize("tag,n,p", [("m8p3", 8, 3), ("m4p2", 4, 2)])
def test_vcycle_and_solve_match_golden(P, golden, tag, n, p):
    g = golden("hierarchies.npz")
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, specs.manufactured(P.pb.ProblemSpec),
                                  smoother="blockjacobi", omega=0.8)
    b = levels[0].rhs
    assert rel(P.mg.v_cycle(levels, b), g[f"{tag}_bj_x1"]) < TOL
    _, mon = P.mg.solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    history_close(mon.residuals, g[f"{tag}_bj_res"])
    _, monw = P.mg.solve_mg(levels, b=b, cycle="w", tol=1e-10, max_cycles=400)
    history_close(monw.residuals, g[f"{tag}_bjw_res"])


def test_kI_vcycle_matches_golden(P, golden):
    g = golden("hierarchies.npz")
    levels = P.mg.build_hierarchy(P.mesh(16, 16), 4, specs.constant(P.pb.ProblemSpec), smoother="blockjacobi")
    b = g["kI16p4_b"]
    assert rel(P.mg.v_cycle(levels, b), g["kI16p4_bj_x1"]) < TOL
    _, mon = P.mg.solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    history_close(mon.residuals, g["kI16p4_bj_res"])


def test_heterogeneous_vcycle_and_pcg_match_golden(P, golden):
    g = golden("hierarchies.npz")
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(g["het8p2_K"]), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(8, 8), 2, spec, smoother="blockjacobi")
    b = g["het8p2_b"]
    assert rel(levels[0].system.matvec_free(b), g["het8p2_y"]) < TOL
    assert rel(P.mg.v_cycle(levels, b), g["het8p2_bj_x1"]) < TOL
    _, mon = P.mg.solve_mg(levels, b=b, tol=1e-10, max_cycles=2000)
    history_close(mon.residuals, g["het8p2_bj_res"])
    x, it = levels[0].system.solve_cg(tol=1e-10, precond=P.mg.mg_preconditioner(levels), b=b)
    assert it == int(g["het8p2_pcg_iters"][0])
    assert rel(x, g["het8p2_pcg_x"]) < 1e-9


def test_config1_golden(P, golden):
    """BASELINE configs[0] end to end: rhs, one matvec, one V(2,2) BJ(0.8) cycle on
    levels[:6] (down to 4x4): rel. residual 0.267064; full solve 92 cycles, rho 0.80898."""
    g = golden("config1.npz")
    levels = P.mg.build_hierarchy(P.mesh(64, 64), 2, P.pb.config1_problem(), smoother=None)[:6]
    P.mg.attach_smoothers(levels, "blockjacobi", 0.8)
    fine = levels[0]
    b = fine.rhs
    assert rel(b, g["b"]) < TOL
    assert rel(fine.matvec(b), g["Ab"]) < TOL
    x1 = P.mg.v_cycle(levels, b)
    assert rel(x1, g["x1"]) < TOL
    r1 = np.linalg.norm(b - fine.matvec(x1)) / np.linalg.norm(b)
    assert abs(r1 - 0.267064) < 5e-7
    x, mon = P.mg.solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    history_close(mon.residuals, g["res"])
    assert len(mon.residuals) - 1 == 92
    assert abs(mon.asymptotic_rate() - 0.80898) < 1e-5
    assert rel(x, g["x"]) < 1e-10


def test_vcycle_graph_replay_and_zero_input(P):
    levels = P.mg.build_hierarchy(P.mesh(32, 32), 3, specs.constant(P.pb.ProblemSpec), smoother="blockjacobi")
    b = np.random.default_rng(4).uniform(-1, 1, levels[0].ndof)
    x1 = P.mg.v_cycle(levels, b)
    x2 = P.mg.v_cycle(levels, b)
    np.testing.assert_array_equal(x1, x2)
    np.testing.assert_array_equal(P.mg.v_cycle(levels, np.zeros_like(b)), 0.0)   # test_multigrid.py:206-209
    lo = O.build_levels(O.Grid(32, 32), 3, specs.constant(O.Spec), smoother="blockjacobi")
    assert rel(x1, O.v_cycle(lo, b)) < TOL
    x0 = np.random.default_rng(5).standard_normal(levels[0].ndof)
    x0c = x0.copy()
    assert rel(P.mg.v_cycle(levels, b, x0), O.v_cycle(lo, b, x0)) < TOL
    np.testing.assert_array_equal(x0, x0c)                                       # x0 not mutated


# ------------------------------------------------------------------------------- FSAI


@pytest.mark.parametrize("tag,n,p", [("m8p3", 8, 3), ("m4p2", 4, 2)])
def test_fsai_solve_matches_golden(P, golden, tag, n, p):
    """Reference default smoother (FSAI baseline, multigrid.py:47-173) on the device:
    identical lambda_max, iteration count and residual history."""
    g = golden("hierarchies.npz")
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, specs.manufactured(P.pb.ProblemSpec), smoother="baseline")
    lam = [lev.smoother.lam_max for lev in levels[:-1]]
    assert rel(lam, g[f"{tag}_fsai_lam"]) < 1e-10
    x, mon = P.mg.solve_mg(levels)
    history_close(mon.residuals, g[f"{tag}_fsai_res"])
    assert rel(x, g[f"{tag}_fsai_x"]) < 1e-10


def test_fsai_smoother_api(P):
    levels = P.mg.build_hierarchy(P.mesh(8, 8), 2, specs.manufactured(P.pb.ProblemSpec), smoother="baseline")
    lo = O.build_levels(O.Grid(8, 8), 2, specs.manufactured(O.Spec), smoother="baseline")
    rng = np.random.default_rng(8)
    for lev, ol in zip(levels[:-1], lo[:-1]):
        r = rng.standard_normal(lev.ndof)
        assert rel(lev.smoother.apply_inverse(r), ol.smoother.apply_inverse(r)) < TOL
        b = rng.standard_normal(lev.ndof)
        x0 = rng.standard_normal(lev.ndof)
        got = lev.smoother.smooth(lev.matvec, b, x0, 3)
        ref = ol.smoother.smooth(ol.matvec, b, x0, 3)
        assert rel(got, ref) < TOL
    b = levels[0].rhs
    assert rel(P.mg.v_cycle(levels, b), O.v_cycle(lo, b)) < TOL


def test_aggressive_fsai_converges_fast(P):
    """test_multigrid.py:267-270: aggressive FSAI V-cycle rate <= 0.05."""
    levels = P.mg.build_hierarchy(P.mesh(8, 8), 3, specs.manufactured(P.pb.ProblemSpec), smoother="aggressive")
    _, mon = P.mg.solve_mg(levels, tol=1e-13)
    assert mon.asymptotic_rate() <= 0.05
    lo = O.build_levels(O.Grid(8, 8), 3, specs.manufactured(O.Spec), smoother="aggressive")
    _, mo = O.solve_mg(lo, tol=1e-13)
    assert len(mon.residuals) == len(mo.residuals)


# ------------------------------------------------------- GPU batched condensation (8f #1)


@pytest.mark.parametrize("n,p", [(16, 2), (12, 4), (8, 8)])
def test_gpu_condensation_matches_oracle(P, n, p, monkeypatch):
    """Heterogeneous piecewise-constant K condensed on the device (flux eliminated first,
    nb x nb solves) against the oracle's full local LU (local.py:204-237)."""
    monkeypatch.setattr(P.tr.TraceSystem, "GPU_CLASSES", 0)
    Kg = specs.hetero_K(n, seed=11)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.bump_f, specs.bump_u, 1.0)
    s = P.tr.TraceSystem(P.mesh(n, n), p, spec)
    assert s.piecewise is not None
    o = O.OracleTrace(O.Grid(n, n), p, O.Spec(O.piecewise_coefficient(Kg), specs.bump_f, specs.bump_u, 1.0))
    assert rel(s.schur, o.schur) < 1e-11
    assert rel(s.rhs, o.rhs) < 1e-11
    x = np.random.default_rng(2).uniform(-1, 1, s.ndof)
    assert rel(s.matvec_free(x), o.matvec(x)) < 1e-11


def test_gpu_condensed_hierarchy_solve(P, monkeypatch):
    """MG-PCG on a GPU-condensed heterogeneous hierarchy equals the oracle's iteration count."""
    monkeypatch.setattr(P.tr.TraceSystem, "GPU_CLASSES", 0)
    g = golden_het = None
    n, p = 16, 2
    Kg = specs.hetero_K(n, seed=2)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother="blockjacobi")
    lo = O.build_levels(O.Grid(n, n), p, O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0),
                        smoother="blockjacobi")
    b = np.random.default_rng(9).uniform(-1, 1, levels[0].ndof)
    x, it = levels[0].system.solve_cg(tol=1e-10, precond=P.mg.mg_preconditioner(levels), b=b)
    xo, ito = lo[0].system.solve_cg(b=b, tol=1e-10, precond=O.mg_preconditioner(lo))
    assert it == ito
    assert rel(x, xo) < 1e-9


def test_chebyshev_blockjacobi_matches_oracle(P):
    """Chebyshev-weighted block-Jacobi (robust smoother for high-contrast K): lambda_max, one
    V-cycle and the MG-PCG iteration count agree with the oracle restatement."""
    n, p = 16, 2
    Kg = specs.hetero_K(n, seed=4)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother="bj-chebyshev")
    lo = O.build_levels(O.Grid(n, n), p, O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0),
                        smoother="bj-chebyshev")
    for lev, ol in zip(levels[:-1], lo[:-1]):
        assert abs(lev.smoother.lam_max - ol.smoother.lam_max) < 1e-10 * ol.smoother.lam_max
    b = np.random.default_rng(6).uniform(-1, 1, levels[0].ndof)
    assert rel(P.mg.v_cycle(levels, b), O.v_cycle(lo, b)) < TOL
    x, it = levels[0].system.solve_cg(tol=1e-10, precond=P.mg.mg_preconditioner(levels), b=b)
    xo, ito = lo[0].system.solve_cg(b=b, tol=1e-10, precond=O.mg_preconditioner(lo))
    assert it == ito and it < 100
    assert rel(x, xo) < 1e-9


def test_w_cycle_fmg_and_single_level(P):
    """test_multigrid.py:233-290 analogues against the oracle."""
    spec = specs.manufactured(P.pb.ProblemSpec)
    one = P.mg.build_hierarchy(P.mesh(2, 2), 1, spec, smoother="blockjacobi")
    assert len(one) == 1 and one[0].kind == "coarsest"
    ref = O.OracleTrace(O.Grid(2, 2), 1, specs.manufactured(O.Spec)).solve_direct()
    np.testing.assert_allclose(P.mg.w_cycle(one, one[0].rhs), ref, atol=1e-12)
    np.testing.assert_allclose(P.mg.fmg(one), ref, atol=1e-12)
    x, mon = P.mg.solve_mg(one)
    np.testing.assert_allclose(x, ref, atol=1e-12)
    levels = P.mg.build_hierarchy(P.mesh(8, 8), 3, spec, smoother="baseline")
    lo = O.build_levels(O.Grid(8, 8), 3, specs.manufactured(O.Spec), smoother="baseline")
    b = levels[0].rhs
    assert rel(P.mg.w_cycle(levels, b), O.cycle(lo, 0, b, np.zeros_like(b), 2, 2, 2)) < TOL
    assert rel(P.mg.fmg(levels), O.fmg(lo)) < 1e-11


def test_rectangular_vcycle_and_plain_cg(P):
    spec = specs.manufactured(P.pb.ProblemSpec)
    levels = P.mg.build_hierarchy(P.mesh(12, 8), 2, spec, smoother="blockjacobi")
    lo = O.build_levels(O.Grid(12, 8), 2, specs.manufactured(O.Spec), smoother="blockjacobi")
    b = levels[0].rhs
    assert rel(P.mg.v_cycle(levels, b), O.v_cycle(lo, b)) < TOL
    x, it = levels[0].system.solve_cg(tol=1e-12)                      # trace.py:142-163
    xo, ito = lo[0].system.solve_cg(tol=1e-12)
    assert it == ito
    assert rel(x, xo) < 1e-9


def test_anisotropic_gpu_condensation_and_vcycle(P, monkeypatch):
    """configs[4]-style anisotropic diagonal K condensed on the device; matvec and one V-cycle
    against the oracle restatement (F9)."""
    monkeypatch.setattr(P.tr.TraceSystem, "GPU_CLASSES", 0)
    n, p = 16, 4
    rng = np.random.default_rng(3)
    Kx, Ky = np.exp(rng.uniform(np.log(0.1), np.log(10.0), (2, n, n)))
    spec = P.pb.ProblemSpec(P.pb.piecewise_anisotropic(Kx, Ky), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother="blockjacobi")
    assert levels[0].system.piecewise is not None
    lo = O.build_levels(O.Grid(n, n), p, O.Spec(O.piecewise_anisotropic(Kx, Ky), specs.zero, specs.zero, 1.0),
                        smoother="blockjacobi")
    b = rng.uniform(-1, 1, levels[0].ndof)
    assert rel(levels[0].matvec(b), lo[0].matvec(b)) < 1e-11
    assert rel(P.mg.v_cycle(levels, b), O.v_cycle(lo, b)) < 1e-11


def test_reconstruct_all_matches_oracle(P):
    """trace.py:171-178 (volume recovery after the solve) on the device."""
    for spec_o, spec_p in [(specs.manufactured(O.Spec), specs.manufactured(P.pb.ProblemSpec)),
                           (specs.constant(O.Spec, 0.0, 1.0), specs.constant(P.pb.ProblemSpec, 0.0, 1.0))]:
        s = P.tr.TraceSystem(P.mesh(6, 5), 2, spec_p)
        o = O.OracleTrace(O.Grid(6, 5), 2, spec_o)
        lam = np.random.default_rng(1).standard_normal(s.ndof)
        q, u = s.reconstruct_all(lam)
        qo, uo = O.reconstruct_all(o, lam)
        assert rel(q, qo) < 1e-11 and rel(u, uo) < 1e-11
        assert rel(s.postprocess_all(q, u), O.postprocess_all(o, qo, uo)) < 1e-11


@pytest.mark.parametrize("tag,kind,n,p", [("m4p2", "m", 4, 2), ("m5p3", "m", 5, 3), ("m6p1", "m", 6, 1),
                                          ("kI4p4", "kI", 4, 4)])
def test_reconstruct_postprocess_match_golden(P, golden, tag, kind, n, p):
    """reconstruct_all / postprocess_all against the unmodified reference (trace.py:171-185)."""
    import torch
    g = golden("postprocess.npz")
    spec = specs.manufactured(P.pb.ProblemSpec) if kind == "m" else specs.constant(P.pb.ProblemSpec, 0.0, 1.0)
    s = P.tr.TraceSystem(P.mesh(n, n), p, spec)
    q, u = s.reconstruct_all(g[f"{tag}_lam"])
    assert rel(q, g[f"{tag}_q"]) < TOL and rel(u, g[f"{tag}_u"]) < TOL
    assert rel(s.postprocess_all(g[f"{tag}_q"], g[f"{tag}_u"]), g[f"{tag}_ustar"]) < TOL
    qt, ut = s.reconstruct_all(torch.as_tensor(g[f"{tag}_lam"], device="cuda"))   # tensor in -> tensors out
    assert qt.is_cuda and rel(qt.cpu().numpy(), g[f"{tag}_q"]) < TOL
    assert s.postprocess_all(qt, ut).is_cuda


@pytest.mark.parametrize("aniso", [False, True])
def test_reconstruct_postprocess_gpu_condensed(P, aniso):
    """Element-wise constant media with more distinct elements than GPU_CLASSES take the
    flux-first device elimination (PiecewiseCondenser.reconstruct); checked against the oracle."""
    n, p = 66, 1
    rng = np.random.default_rng(21)
    if aniso:
        Kx, Ky = np.exp(rng.uniform(-2, 2, (2, n, n)))
        spec_p = P.pb.ProblemSpec(P.pb.piecewise_anisotropic(Kx, Ky), specs.bump_f, specs.zero, 1.0)
        spec_o = O.Spec(O.piecewise_anisotropic(Kx, Ky), specs.bump_f, specs.zero, 1.0)
    else:
        Kg = specs.hetero_K(n, seed=21)
        spec_p = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.bump_f, specs.bump_u, 1.0)
        spec_o = O.Spec(O.piecewise_coefficient(Kg), specs.bump_f, specs.bump_u, 1.0)
    s = P.tr.TraceSystem(P.mesh(n, n), p, spec_p)
    assert s.piecewise is not None
    o = O.OracleTrace(O.Grid(n, n), p, spec_o)
    lam = rng.standard_normal(s.ndof)
    q, u = s.reconstruct_all(lam)
    qo, uo = O.reconstruct_all(o, lam)
    assert rel(q, qo) < 1e-11 and rel(u, uo) < 1e-11
    assert rel(s.postprocess_all(q, u), O.postprocess_all(o, qo, uo)) < 1e-11


@pytest.mark.parametrize("case", ["cfg1", "hetero_w", "p1_rect"])
def test_fused_coarse_tail_matches_launch_path(P, case):
    """The trailing small p = 1 levels run as one cooperative kernel: same cycle as the
    per-launch path (to rounding) and as the oracle (1e-12)."""
    if case == "cfg1":
        levels = P.mg.build_hierarchy(P.mesh(64, 64), 2, P.pb.config1_problem(), smoother=None)[:6]
        P.mg.attach_smoothers(levels, "blockjacobi", 0.8)
        grid, ospec = O.config1_system(64, 2)
        olevels = O.build_levels(grid, 2, ospec, smoother="blockjacobi")[:6]
        visits = 1
    elif case == "hetero_w":
        Kg = specs.hetero_K(16, seed=5)
        spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
        levels = P.mg.build_hierarchy(P.mesh(16, 16), 2, spec, smoother="blockjacobi", omega=0.8)
        olevels = O.build_levels(O.Grid(16, 16), 2, O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0),
                                 smoother="blockjacobi")
        visits = 2
    else:
        spec, ospec = specs.manufactured(P.pb.ProblemSpec), specs.manufactured(O.Spec)
        levels = P.mg.build_hierarchy(P.mesh(32, 16), 1, spec, smoother="blockjacobi", omega=0.8)
        olevels = O.build_levels(O.Grid(32, 16), 1, ospec, smoother="blockjacobi")
        visits = 1
    b = np.random.default_rng(3).uniform(-1, 1, levels[0].ndof)
    run = P.mg.v_cycle if visits == 1 else P.mg.w_cycle
    P.mg.set_fused_tail(levels, True)
    xf = run(levels, b)
    xf2 = run(levels, b, xf)                 # second cycle from a nonzero guess (replayed graph)
    P.mg.set_fused_tail(levels, False)
    xl = run(levels, b)
    xl2 = run(levels, b, xl)
    P.mg.set_fused_tail(levels, True)
    assert rel(xf, xl) < 1e-13 and rel(xf2, xl2) < 1e-13
    xo = O.cycle(olevels, 0, b, np.zeros_like(b), 2, 2, visits)
    assert rel(xf, xo) < TOL


@pytest.mark.parametrize("power", [1, 2])
def test_fsai_rows_on_device_match_host(P, power):
    """fsai_build's per-row SPD solves on the GPU (hdg_fsai_rows, Cholesky) against the host
    restatement (LU, multigrid.py:133-152) on a K = I p=3 level and a heterogeneous p=2 level."""
    from paper_1705_09907_b200.fsai import fsai_build
    for spec, n, p in [(specs.constant(P.pb.ProblemSpec), 16, 3),
                       (P.pb.ProblemSpec(P.pb.piecewise_coefficient(specs.hetero_K(12, seed=3)), specs.zero,
                                         specs.zero, 1.0), 12, 2)]:
        lev = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother=None)[0]
        A = lev.operator.tocsr()
        gd = fsai_build(A, power, device=True)
        gh = fsai_build(A, power, device=False)
        assert (gd.G.indptr == gh.G.indptr).all() and (gd.G.indices == gh.G.indices).all()
        assert rel(gd.G.data, gh.G.data) < 1e-12
        assert abs(gd.lam_max - gh.lam_max) <= 1e-12 * gh.lam_max


@pytest.mark.parametrize("aniso", [False, True])
def test_heterogeneous_full_size_properties(P, aniso):
    """configs[2]'s coefficient law (log-uniform K in [1e-2, 1e2], seed 2) and configs[4]'s
    anisotropic diagonal law (Kxx, Kyy log-uniform in [1e-1, 1e1], seed 3) at 1024^2, p=4
    (1M elements condensed on the GPU, stored facet streams): sampled element blocks against the
    oracle's full local LU (SURVEY 8c recipe 7), then size-independent properties of the
    operator: symmetry, linearity, determinism (test_trace.py:51-66)."""
    import torch
    n, p = 1024, 4
    if aniso:
        rng3 = np.random.default_rng(3)
        Kx, Ky = np.exp(rng3.uniform(np.log(0.1), np.log(10.0), (2, n, n)))
        spec = P.pb.ProblemSpec(P.pb.piecewise_anisotropic(Kx, Ky), specs.zero, specs.zero, 1.0)
        ospec = O.Spec(O.piecewise_anisotropic(Kx, Ky), specs.zero, specs.zero, 1.0)
    else:
        Kg = specs.hetero_K(n, seed=2)
        spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
        ospec = O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    s = P.tr.TraceSystem(P.mesh(n, n), p, spec)
    assert s.piecewise is not None and not s.operator.shared
    core = O.ElementCore(O.Grid(n, n), p)
    rng = np.random.default_rng(7)
    elems = rng.choice(np.arange(n + 1, n * n - n - 1), 48, replace=False)
    elems = elems[(elems % n != 0) & (elems % n != n - 1)]          # interior: no Dirichlet sides
    S = s.operator.S_cls
    got = (S[torch.as_tensor(elems, device=S.device)] if isinstance(S, torch.Tensor) else S[elems])
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got)
    for k, e in enumerate(elems):
        assert rel(got[k], O.Local(core, int(e), ospec).schur) < 1e-11
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(s.ndof, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    y = torch.rand(s.ndof, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    Ax, Ay = s.matvec_free(x), s.matvec_free(y)
    lhs, rhs_ = float(Ax @ y), float(x @ Ay)
    assert abs(lhs - rhs_) <= 1e-11 * max(1.0, abs(lhs))
    A2 = s.matvec_free(2.0 * x - 3.0 * y)
    assert float((A2 - (2.0 * Ax - 3.0 * Ay)).abs().max()) <= 1e-12 * float(A2.abs().max())
    assert torch.equal(Ax, s.matvec_free(x))


@pytest.mark.parametrize("nx,ny,p", [(31, 9, 2), (32, 7, 1), (33, 12, 4), (64, 5, 3), (65, 3, 1), (1, 6, 2), (6, 1, 2)])
def test_half_stored_stream_mesh_widths(P, nx, ny, p):
    """Stored (per-element) operator with each coupling block kept by one facet and read
    transposed by its partner: mesh widths around the 32-lane interleave (slot (j, i+1) reads),
    thin meshes, against the oracle; plus a block-Jacobi sweep (D^-1 from the owned diagonal)."""
    rng = np.random.default_rng(nx * 100 + ny)
    Kg = np.exp(rng.uniform(-2.0, 2.0, (ny, nx)))
    def coef(x, y):
        i = np.clip(np.floor(np.asarray(x) * nx).astype(np.int64), 0, nx - 1)
        j = np.clip(np.floor(np.asarray(y) * ny).astype(np.int64), 0, ny - 1)
        return Kg[j, i]
    m = P.mesh(nx, ny)
    spec = P.pb.ProblemSpec(coef, specs.zero, specs.zero, 1.0)
    s = P.tr.TraceSystem(m, p, spec)
    if s.ndof == 0:
        return
    assert not s.operator.shared
    o = O.OracleTrace(O.Grid(nx, ny), p, O.Spec(coef, specs.zero, specs.zero, 1.0))
    x = rng.uniform(-1, 1, s.ndof)
    assert rel(s.matvec_free(x), o.matvec(x)) < TOL
    bj = P.mg.BlockJacobiSmoother(s.operator, 0.8)
    b = rng.uniform(-1, 1, s.ndof)
    got = bj.smooth(s.matvec_free, b, x, 1)
    n1 = p + 1
    ref = x.copy()
    r = b - o.matvec(x)
    Ad = s.operator.tocsr().toarray() if s.ndof <= 3000 else None
    if Ad is not None:
        for blk in range(s.ndof // n1):
            sl = slice(blk * n1, (blk + 1) * n1)
            ref[sl] = x[sl] + 0.8 * np.linalg.solve(Ad[sl, sl], r[sl])
        assert rel(got, ref) < 1e-11


def test_fsai_on_large_condensed_hierarchy_keeps_blocks(P, monkeypatch):
    """Large device-condensed levels drop their element blocks after the hierarchy is built.
    The baseline FSAI is set up on the device from each level's blocks while the hierarchy is
    built (so the blocks can go), the aggressive one builds from the level CSR and keeps them;
    attaching FSAI afterwards to a hierarchy whose blocks were released raises HierarchyError.
    Both match the oracle."""
    monkeypatch.setattr(P.tr.TraceSystem, "GPU_CLASSES", 0)
    monkeypatch.setattr(P.mg, "RELEASE_NDOF", 0)
    n, p = 16, 2
    Kg = specs.hetero_K(n, seed=2)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    bare = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother=None)
    assert bare[0].block_op.S_cls is None
    with pytest.raises(P.mg.HierarchyError):
        P.mg.attach_smoothers(bare, "baseline")
    P.mg.attach_smoothers(bare, "blockjacobi")            # block-Jacobi only needs the facet stream
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother="baseline")
    assert levels[0].block_op.S_cls is None
    assert all(isinstance(lev.smoother, P.mg.StructuredFSAI) for lev in levels[:-1])
    agg = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother="aggressive")
    assert agg[0].block_op.S_cls is not None
    lo = O.build_levels(O.Grid(n, n), p, O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0),
                        smoother="baseline")
    b = np.random.default_rng(9).uniform(-1, 1, levels[0].ndof)
    x, it = levels[0].system.solve_cg(tol=1e-10, precond=P.mg.mg_preconditioner(levels), b=b)
    xo, ito = lo[0].system.solve_cg(b=b, tol=1e-10, precond=O.mg_preconditioner(lo))
    assert it == ito
    assert rel(x, xo) < 1e-9


def test_reattached_smoother_recaptures_cycle_graphs(P):
    """Cycle graphs are cached per (b, x0, x, nu1, nu2, visits); attaching another smoother to
    the same levels (attach_smoothers, multigrid.py:345-352) must not replay the old one."""
    n, p = 16, 2
    Kg = specs.hetero_K(n, seed=4)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    b = np.random.default_rng(3).uniform(-1, 1, 2 * n * (n - 1) * (p + 1))
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother="blockjacobi")
    import torch
    bd = torch.from_numpy(b).cuda()   # same device b every call: the cached graphs are hit
    x_bj = P.mg.v_cycle(levels, bd).cpu().numpy()
    for mode in ("bj-chebyshev", "baseline", "blockjacobi"):
        P.mg.attach_smoothers(levels, mode)
        x = P.mg.v_cycle(levels, bd).cpu().numpy()
        fresh = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother=mode)
        xf = P.mg.v_cycle(fresh, bd).cpu().numpy()
        assert rel(x, xf) < 1e-13, mode
        if mode != "blockjacobi":
            assert rel(x, x_bj) > 1e-6, mode
    assert rel(x, x_bj) < 1e-13
    # fixed buffers through the C ABI: a replay hits the cache, a re-attached smoother forces a
    # fresh capture (hdg_mg_graph_captures counts instantiations)
    mg = P.mg._native_mg(levels)
    xo = torch.zeros_like(bd)
    st = torch.cuda.current_stream().cuda_stream
    cyc = lambda: P.lib_check(P.lib.hdg_mg_cycle(mg.handle, bd.data_ptr(), None, xo.data_ptr(), 2, 2, 1, 1, st))
    cyc()
    c0 = P.lib.hdg_mg_graph_captures(mg.handle)
    cyc()
    assert P.lib.hdg_mg_graph_captures(mg.handle) == c0
    P.mg.attach_smoothers(levels, "bj-chebyshev")
    cyc()
    assert P.lib.hdg_mg_graph_captures(mg.handle) == c0 + 1


def test_cycle_graph_cache_is_bounded(P):
    """Graphs are keyed by buffer pointers; callers whose buffers move must not grow the cache
    without bound (LRU of 8): 12 distinct output buffers -> 12 captures, replays of the last
    ones hit the cache, and every result equals the first."""
    import torch
    n, p = 8, 2
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, P.pb.constant_problem(0.0, 1.0), smoother="blockjacobi")
    mg = P.mg._native_mg(levels)
    bd = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, levels[0].ndof)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    outs = [torch.zeros_like(bd) for _ in range(12)]
    c0 = P.lib.hdg_mg_graph_captures(mg.handle)
    for o in outs:
        P.lib_check(P.lib.hdg_mg_cycle(mg.handle, bd.data_ptr(), None, o.data_ptr(), 2, 2, 1, 1, st))
    assert P.lib.hdg_mg_graph_captures(mg.handle) == c0 + 12
    for o in outs[-8:]:
        P.lib_check(P.lib.hdg_mg_cycle(mg.handle, bd.data_ptr(), None, o.data_ptr(), 2, 2, 1, 1, st))
    assert P.lib.hdg_mg_graph_captures(mg.handle) == c0 + 12
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_native_pcg_matches_python_loop(P, golden):
    """hdg_pcg (the whole trace.py:142-163 loop natively, one graph per iteration, one D2H)
    against the host-driven loop of the same device kernels: same iteration count, same iterate
    to rounding, with the MG preconditioner (multigrid.py:457-463), without one, and from x0."""
    g = golden("hierarchies.npz")
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(g["het8p2_K"]), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(8, 8), 2, spec, smoother="blockjacobi")
    sysg = levels[0].system
    b = g["het8p2_b"]
    pc = P.mg.mg_preconditioner(levels)
    x_nat, it_nat = sysg.solve_cg(tol=1e-10, precond=pc, b=b)
    x_py, it_py = sysg.solve_cg(tol=1e-10, precond=lambda r: pc(r), b=b)
    assert it_nat == it_py == int(g["het8p2_pcg_iters"][0])
    assert rel(x_nat, x_py) < 1e-13
    hist = sysg.cg_residuals
    assert len(hist) == it_nat + 1 and hist[-1] <= 1e-10 * np.linalg.norm(b) < hist[-2]
    x_nat, it_nat = sysg.solve_cg(tol=1e-9, b=b, maxiter=3000)
    x_py, it_py = sysg.solve_cg(tol=1e-9, b=b, maxiter=3000, matvec=sysg.operator.apply)
    assert it_nat == it_py and rel(x_nat, x_py) < 1e-12
    x0 = np.random.default_rng(2).standard_normal(sysg.ndof)
    x_nat, it_nat = sysg.solve_cg(tol=1e-10, precond=pc, b=b, x0=x0)
    x_py, it_py = sysg.solve_cg(tol=1e-10, precond=lambda r: pc(r), b=b, x0=x0)
    assert it_nat == it_py and rel(x_nat, x_py) < 1e-12
    _, it0 = sysg.solve_cg(tol=1e-10, precond=pc, b=b, maxiter=0)
    assert it0 == 0


def test_blockjacobi_complexity_matches_oracle(P):
    """BlockJacobiSmoother.complexity = n_blocks n1^2 / nnz(A) per level, counted like the
    oracle's CSR; the structural count used above 1M dofs agrees on K = I."""
    n, p = 16, 3
    lv = P.mg.build_hierarchy(P.mesh(n, n), p, specs.constant(P.pb.ProblemSpec), smoother="blockjacobi")
    lo = O.build_levels(O.Grid(n, n), p, specs.constant(O.Spec), smoother="blockjacobi")
    for a, b in zip(lv[:-1], lo[:-1]):
        assert abs(a.smoother.complexity - b.smoother.complexity) < 1e-12
        lay = a.block_op.layout
        assert P.mg.structural_nnz(lay.nx, lay.ny, lay.n1) == a.block_op.tocsr().nnz


@pytest.mark.parametrize("case", ["kI", "het", "aniso"])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_structured_fsai_matches_host_fsai(P, case, p):
    """The facet-structured device FSAI (one Cholesky per facet, hdg_fsai.cuh) reproduces the
    host restatement of fsai_build (per-row solves on lower(A), multigrid.py:123-159): same
    pattern, same values to rounding, same lambda_max (seed-1234 power iteration), and the same
    smoothing sweeps."""
    from paper_1705_09907_b200.fsai import StructuredFSAI, fsai_build
    n = 6 if p == 8 else 8
    if case == "kI":
        spec = specs.constant(P.pb.ProblemSpec)
    elif case == "het":
        spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(specs.hetero_K(n, seed=7)), specs.zero, specs.zero, 1.0)
    else:
        kx, ky = specs.hetero_K(n, seed=8), specs.hetero_K(n, seed=9)
        spec = P.pb.ProblemSpec(P.pb.piecewise_anisotropic(kx, ky), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother=None)
    for lev in levels[:-1]:
        A = lev.operator.tocsr()
        ref = fsai_build(A, 1, 1.0, device=False)
        sm = StructuredFSAI(lev.block_op, 1.0)
        G, Gr = sm.G, ref.G
        assert G.nnz == Gr.nnz
        assert (abs(G - Gr)).max() <= 1e-11 * abs(Gr).max()
        assert abs(sm.lam_max - ref.lam_max) <= 1e-10 * ref.lam_max
        assert abs(sm.complexity - ref.complexity) < 1e-12
        b = np.random.default_rng(1).uniform(-1, 1, lev.ndof)
        x0 = np.random.default_rng(2).uniform(-1, 1, lev.ndof)
        x = sm.smooth(None, b, x0, 3)
        xr = x0.copy()
        for w in ref.sweep_weights(3):
            xr = xr + w * (ref.Gt @ (ref.G @ (b - A @ xr)))
        assert rel(x, xr) < 1e-11


def test_structured_fsai_released_blocks_hierarchy(P, monkeypatch):
    """build_hierarchy(smoother="baseline") on a device-condensed heterogeneous hierarchy whose
    large levels release their element blocks: every level gets its device FSAI before the
    release, and the V-cycle / MG-PCG agree with the oracle's FSAI hierarchy."""
    import paper_1705_09907_b200.multigrid as mgm
    monkeypatch.setattr(mgm, "RELEASE_NDOF", 100)
    monkeypatch.setattr(P.tr.TraceSystem, "GPU_CLASSES", 0)
    n, p = 16, 3
    Kg = specs.hetero_K(n, seed=11)
    spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother="baseline")
    assert all(isinstance(lev.smoother, mgm.StructuredFSAI) for lev in levels[:-1])
    lo = O.build_levels(O.Grid(n, n), p, O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0),
                        smoother="baseline")
    b = np.random.default_rng(3).uniform(-1, 1, levels[0].ndof)
    assert rel(P.mg.v_cycle(levels, b), O.v_cycle(lo, b)) < 1e-10
    assert levels[0].block_op.S_cls is None                       # released after its FSAI was built
    x, it = levels[0].system.solve_cg(tol=1e-10, precond=P.mg.mg_preconditioner(levels), b=b)
    xo, ito = lo[0].system.solve_cg(b=b, tol=1e-10, precond=O.mg_preconditioner(lo))
    assert it == ito
    assert rel(x, xo) < 1e-9
