"""Hand-written setup / post-solve kernels (csrc/hdg_setup.cu; include/hdgb200.h) against their
numpy definitions on seeded random inputs, and against the oracle's local condensation."""

import numpy as np
import pytest

import specs
from oracle import hdg_oracle as O

pytestmark = pytest.mark.gpu


def cu(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


@pytest.mark.parametrize("E,I,J", [(1, 1, 1), (7, 3, 5), (130, 65, 33), (1000, 81, 100), (64, 1, 170)])
def test_gemm_nt_options(P, E, I, J):
    from paper_1705_09907_b200.discretization import gemm_nt
    rng = np.random.default_rng(E + I + J)
    A, B, C0 = rng.standard_normal((E, J)), rng.standard_normal((I, J)), rng.standard_normal((E, I))
    rs, cs, ad = rng.uniform(0.5, 2, E), rng.standard_normal(J), rng.uniform(0.5, 2, (E, J))
    assert rel(gemm_nt(cu(A), cu(B)).cpu().numpy(), A @ B.T) < 1e-13
    out = cu(C0)
    gemm_nt(cu(A), cu(B), out=out, rowscale=cu(rs), colscale=cu(cs), adiv=cu(ad), alpha=-0.7, beta=1.5)
    ref = 1.5 * C0 - 0.7 * rs[:, None] * ((A * cs / ad) @ B.T)
    assert rel(out.cpu().numpy(), ref) < 1e-13
    # column slices of wider tensors on both sides
    wide_a, wide_c = cu(np.hstack([A, A])), cu(np.zeros((E, I + 3)))
    gemm_nt(wide_a[:, J:], cu(B), out=wide_c[:, 2:2 + I])
    assert rel(wide_c[:, 2:2 + I].cpu().numpy(), A @ B.T) < 1e-13
    assert float(wide_c[:, :2].abs().max()) == 0.0 and float(wide_c[:, 2 + I:].abs().max()) == 0.0


def test_class_gemv_gather_and_owner_sum(P):
    import torch
    rng = np.random.default_rng(3)
    E, I, J, nc = 500, 12, 27, 7
    M, x, y0 = rng.standard_normal((nc, I, J)), rng.standard_normal((E, J)), rng.standard_normal((E, I))
    cls = rng.integers(0, nc, E)
    out, cd, Md, xd = cu(y0), torch.as_tensor(cls, device="cuda"), cu(M), cu(x)   # keep the inputs alive
    P.lib_check(P.lib.hdg_class_gemv(E, I, J, cd.data_ptr(), Md.data_ptr(), xd.data_ptr(), J, out.data_ptr(), I, 2.0,
                                     -1.0, 0))
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), -y0 + 2.0 * np.einsum("eij,ej->ei", M[cls], x)) < 1e-13
    for nx, ny, p in [(5, 4, 2), (1, 6, 1), (6, 1, 3), (33, 17, 4)]:
        sysg = P.tr.TraceSystem(P.mesh(nx, ny), p, specs.constant(P.pb.ProblemSpec))
        lam = rng.standard_normal(sysg.ndof)
        np.testing.assert_array_equal(sysg._gather_device(cu(lam)).cpu().numpy(), sysg.layout.gather(lam))
        cl = rng.standard_normal((nx * ny, 4 * (p + 1)))
        rhs, cld = torch.empty(sysg.ndof, dtype=torch.float64, device="cuda"), cu(cl)
        P.lib_check(P.lib.hdg_sum_owners(nx, ny, p, cld.data_ptr(), rhs.data_ptr(), 0))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(rhs.cpu().numpy(), sysg.layout.sum_owners(cl))


@pytest.mark.parametrize("p", [1, 2, 4, 8, 10])
def test_galerkin_kernels(P, p):
    from paper_1705_09907_b200 import discretization as D
    rng = np.random.default_rng(p)
    if p >= 2:
        V = D.p_transfer_matrix(p)
        S = rng.standard_normal((37, 4 * (p + 1), 4 * (p + 1)))
        assert rel(D.galerkin_p(cu(S), V).cpu().numpy(), D.galerkin_p(S, V)) < 1e-13
    Sch, Q = rng.standard_normal((53, 4, 8, 8)), rng.standard_normal((53, 4, 8, 8))
    assert rel(D.galerkin_h(cu(Sch), Q).cpu().numpy(), D.galerkin_h(Sch, Q)) < 1e-13
    assert rel(D.galerkin_h(cu(Sch[:1]), Q[:1]).cpu().numpy(), D.galerkin_h(Sch[:1], Q[:1])) < 1e-13


@pytest.mark.parametrize("p,aniso", [(1, False), (3, True), (4, False), (8, True), (11, False), (12, False),
                                     (12, True)])
def test_condense_and_usolve_vs_dense_algebra(P, p, aniso):
    """hdg_condense_piecewise / hdg_piecewise_usolve against numpy solves of the same flux-first
    elimination, and (p <= 4) against the oracle's full local LU condensation.  p = 12 runs the
    packed (upper triangle of H) variant of both kernels."""
    from paper_1705_09907_b200.discretization import PiecewiseCondenser
    rng = np.random.default_rng(10 + p)
    E = 40
    pc = PiecewiseCondenser(p, 1.0 / 16, 1.0 / 12, 1.0)
    kx = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), E))
    ky = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), E)) if aniso else kx
    S = pc.blocks((kx, ky) if aniso else kx).cpu().numpy()
    for e in range(0, E, 7):
        k = (kx[e], ky[e])
        H = pc.stab + sum(k[d] * pc.Lapd[d] for d in range(2))
        U = np.linalg.solve(H, pc.Tu - sum(k[d] * pc.Gd[d] for d in range(2)))
        ref = sum(k[d] * pc.A0d[d] for d in range(2)) + pc.Ms + (sum(k[d] * pc.C0d[d] for d in range(2)) + pc.Fu) @ U
        assert rel(S[e], ref) < 1e-11
    rhs = rng.standard_normal((E, pc.nb))
    u = pc._usolve(cu(kx), cu(ky), cu(rhs)).cpu().numpy()
    for e in range(0, E, 7):
        H = pc.stab + kx[e] * pc.Lapd[0] + ky[e] * pc.Lapd[1]
        assert rel(u[e], np.linalg.solve(H, rhs[e])) < 1e-11


def test_condense_reports_breakdown(P):
    from paper_1705_09907_b200.discretization import NumericalBreakdown, PiecewiseCondenser
    pc = PiecewiseCondenser(2, 0.1, 0.1, 1.0)
    with pytest.raises(NumericalBreakdown):
        pc.blocks(np.array([1.0, -5.0, 2.0]))
