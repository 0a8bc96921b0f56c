"""GPU parity of the facet-plane (SoA) trace apply (hdg_soa.cuh, hdg_matvec_soa) against the CPU
oracle of trace.py:87-94, plus the layout contract: pack/unpack round trips bit-exactly and every
slot of an output vector is written (boundary / pad slots as zeros), so outputs chain as inputs."""

import numpy as np
import pytest

import specs
from oracle import hdg_oracle as O
from paper_1705_09907_b200 import HDGError

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def oracle_for(s, nx, ny, p):
    S = s.operator.S_cls[0]
    o = O.OracleTrace(O.Grid(nx, ny), p, None, _blocks=np.broadcast_to(S, (nx * ny,) + S.shape).copy())
    o.schur *= o.gmask[:, None, :]
    return o


@pytest.mark.parametrize("p", list(range(1, 13)))
@pytest.mark.parametrize("shape", [(37, 21), (64, 64), (31, 5), (32, 7), (62, 9), (63, 2), (2, 40), (93, 3)])
def test_planes_matvec_vs_oracle(P, p, shape):
    """Every order the facet-plane kernel is built for; meshes around the 31-column warp
    stride, thin strips (segments of one row) and wide/narrow aspect ratios."""
    nx, ny = shape
    s = P.tr.TraceSystem(P.mesh(nx, ny), p, specs.constant(P.pb.ProblemSpec))
    assert s.operator.shared
    x = np.random.default_rng(100 * p + nx + ny).uniform(-1, 1, s.ndof)
    y = s.matvec_free(s.facet_planes(x)).numpy()
    assert rel(y, oracle_for(s, nx, ny, p).matvec(x)) < TOL


@pytest.mark.parametrize("p", [1, 4, 8, 12])
def test_planes_roundtrip_and_every_slot_written(P, p):
    import torch
    s = P.tr.TraceSystem(P.mesh(70, 45), p, specs.constant(P.pb.ProblemSpec))
    op = s.operator
    x = torch.from_numpy(np.random.default_rng(p).uniform(-1, 1, s.ndof)).cuda()
    xs = op.to_planes(x)
    assert torch.equal(op.from_planes(xs), x)                        # bit-exact round trip
    ys = torch.full_like(xs, float("nan"))
    op.apply_planes(xs, out=ys)
    assert torch.isfinite(ys).all()                                  # no slot left unwritten
    assert torch.equal(op.to_planes(op.from_planes(ys)), ys)         # boundary / pad slots are zero
    assert rel(op.from_planes(ys).cpu().numpy(), s.matvec_free(x.cpu().numpy())) < TOL


@pytest.mark.parametrize("p", [2, 4])
def test_planes_chained_applies(P, p):
    """y = A(A(A x)) kept in planes equals three reference-layout applies."""
    s = P.tr.TraceSystem(P.mesh(96, 80), p, specs.constant(P.pb.ProblemSpec))
    x = np.random.default_rng(7).uniform(-1, 1, s.ndof)
    z = s.facet_planes(x)
    y = x
    for _ in range(3):
        z = s.matvec_free(z)
        y = s.matvec_free(y)
    assert rel(z.numpy(), y) < TOL


def test_planes_deterministic_and_linear(P):
    import torch
    s = P.tr.TraceSystem(P.mesh(128, 128), 4, specs.constant(P.pb.ProblemSpec))
    op = s.operator
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.rand(s.ndof, dtype=torch.float64, device="cuda", generator=g) - 0.5
    b = torch.rand(s.ndof, dtype=torch.float64, device="cuda", generator=g) - 0.5
    ya = op.from_planes(op.apply_planes(op.to_planes(a)))
    assert torch.equal(ya, op.from_planes(op.apply_planes(op.to_planes(a))))
    yb = op.from_planes(op.apply_planes(op.to_planes(b)))
    yab = op.from_planes(op.apply_planes(op.to_planes(2.0 * a - 3.0 * b)))
    assert float((yab - (2.0 * ya - 3.0 * yb)).abs().max()) <= 1e-13 * float(yab.abs().max())


def test_planes_config2_full_size(P):
    """BASELINE configs[1] (1024^2, p=4, K=I): facet-plane apply against the reference-layout
    kernel (itself pinned to the oracle) and symmetry <A x, y> = <x, A y>."""
    import torch
    n, p = 1024, 4
    s = P.tr.TraceSystem(P.mesh(n, n), p, specs.constant(P.pb.ProblemSpec))
    op = s.operator
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(s.ndof, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    v = torch.rand(s.ndof, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    Ax = op.from_planes(op.apply_planes(op.to_planes(x)))
    Av = op.from_planes(op.apply_planes(op.to_planes(v)))
    ref = s.matvec_free(x)
    assert float((Ax - ref).abs().max()) <= TOL * float(ref.abs().max())
    lhs, rhs_ = float(Ax @ v), float(x @ Av)
    assert abs(lhs - rhs_) <= 1e-11 * max(1.0, abs(lhs))


@pytest.mark.parametrize("shape", [(1, 1), (1, 5), (5, 1), (2, 2), (1, 40), (40, 1)])
def test_planes_degenerate_meshes(P, shape):
    """Empty and one-element-wide meshes (trace.py:90-91: ndof may be 0)."""
    nx, ny = shape
    s = P.tr.TraceSystem(P.mesh(nx, ny), 3, specs.constant(P.pb.ProblemSpec))
    x = np.random.default_rng(nx * 7 + ny).uniform(-1, 1, s.ndof)
    z = s.facet_planes(x)
    y = s.matvec_free(z).numpy()
    assert y.shape == (s.ndof,)
    if s.ndof:
        assert rel(y, oracle_for(s, nx, ny, 3).matvec(x)) < TOL
    np.testing.assert_array_equal(z.numpy(), x)


def test_planes_refuses_stored_levels(P):
    s = P.tr.TraceSystem(P.mesh(8, 8), 2, specs.manufactured(P.pb.ProblemSpec))
    assert not s.operator.shared
    with pytest.raises(HDGError):
        s.facet_planes(np.zeros(s.ndof))


