"""Device window kernels of the strip-partitioned V-cycle on one GPU: every
rank's DeviceStripBackend operation against the oracle restricted to the same window, and the
StripMG driver at world 1 against the oracle's global cycle."""

import numpy as np
import pytest

import specs
from oracle import hdg_oracle as O
from strip_oracle import OracleWindowBackend

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _np(t):
    return t.detach().cpu().numpy()


def _hier(P, n, p, hetero):
    if hetero:
        Kg = specs.hetero_K(n, seed=11)
        spec = P.pb.ProblemSpec(P.pb.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
        ospec = O.Spec(O.piecewise_coefficient(Kg), specs.zero, specs.zero, 1.0)
    else:
        spec, ospec = specs.manufactured(P.pb.ProblemSpec), specs.manufactured(O.Spec)
    levels = P.mg.build_hierarchy(P.mesh(n, n), p, spec, smoother=None)
    olevels = O.build_levels(O.Grid(n, n), p, ospec, smoother="blockjacobi")
    return levels, olevels


@pytest.mark.parametrize("world,n,p,hetero", [(2, 16, 2, False), (3, 24, 3, False), (2, 16, 2, True),
                                              (4, 32, 1, False)])
def test_window_ops_match_oracle(P, world, n, p, hetero):
    import torch
    from paper_1705_09907_b200.distributed import DeviceStripBackend, StripLayout, plan_strips
    levels, olevels = _hier(P, n, p, hetero)
    shapes = [(lev.mesh.n_x, lev.mesh.n_y, lev.p, None) for lev in levels]
    d, rows = plan_strips(shapes, world)
    assert d >= 1
    rng = np.random.default_rng(world * 100 + n)
    T = lambda a: torch.from_numpy(a)
    for rank in range(world):
        lay = [StripLayout(*shapes[l][:3], world, rank, rows=rows[l][rank]) for l in range(d + 2)]
        gb = DeviceStripBackend(levels, lay, d)
        ob = OracleWindowBackend(olevels, lay, d)
        for l in range(d + 1):
            own_f, own_c = lay[l].owned, lay[l + 1].owned
            b, x = rng.standard_normal(lay[l].ndof_l), rng.standard_normal(lay[l].ndof_l)
            bd, xd = T(b).cuda(), T(x).cuda()
            assert gb.link(l) == ob.link(l)
            # the window operator equals the global one restricted to the window, ghosts included
            assert rel(_np(gb.bj_sweep(l, bd, xd, 1, 2)), _np(ob.bj_sweep(l, T(b), T(x), 1, 2))) < TOL
            assert rel(_np(gb.bj_zero(l, bd, 1, 2)), _np(ob.bj_zero(l, T(b), 1, 2))) < TOL
            assert rel(_np(gb.residual(l, bd, xd)), _np(ob.residual(l, T(b), T(x)))) < TOL
            # transfers: exact on owned facets (window edges drop out-of-window terms)
            if gb.link(l) == "p":
                got, ref = gb.residual_restrict_p(l, bd, xd), ob.residual_restrict_p(l, T(b), T(x))
            else:
                got, ref = gb.restrict_h(l, xd), ob.restrict_h(l, T(x))
            assert rel(_np(got)[own_c], _np(ref)[own_c]) < TOL
            ec = rng.standard_normal(lay[l + 1].ndof_l)
            got = gb.prolong_add(l, T(ec).cuda(), xd.clone())
            ref = ob.prolong_add(l, T(ec), T(x))
            assert rel(_np(got)[own_f], _np(ref)[own_f]) < TOL


@pytest.mark.parametrize("visits", [1, 2])
def test_strip_mg_world1_matches_oracle_cycle(P, visits):
    import torch
    from paper_1705_09907_b200.distributed import strip_multigrid
    levels, olevels = _hier(P, 16, 2, False)
    mg = strip_multigrid(levels, world=1, rank=0)
    b = olevels[0].rhs
    x = mg.v_cycle(torch.from_numpy(b).cuda(), None, 2, 2, visits)
    ref = O.cycle(olevels, 0, b, np.zeros_like(b), 2, 2, visits)
    loc, glob = mg.layouts[0].owned_pairs()
    out = np.empty_like(ref)
    out[glob] = _np(x)[loc]
    assert rel(out, ref) < TOL


@pytest.mark.parametrize("case", ["aniso", "kI"])
def test_local_strip_hierarchy_world1_device(P, case):
    """The rank-local strip hierarchy (distributed.LocalStripHierarchy) with its device window
    kernels (DeviceStripBackend.from_local) at world 1: the strip V-cycle equals the oracle's
    global V-cycle (configs[4] coefficient law at reduced size, and K = I)."""
    import torch
    from paper_1705_09907_b200.distributed import local_strip_multigrid
    from test_local_strips_cpu import _specs
    n, p = 32, 3
    spec, ospec = _specs(case, n)
    mg, H = local_strip_multigrid(P.mesh(n, n), p, spec)
    olevels = O.build_levels(O.Grid(n, n), p, ospec, smoother="blockjacobi")
    b = np.random.default_rng(7).uniform(-1, 1, olevels[0].ndof)
    x = mg.v_cycle(torch.from_numpy(b[H.layouts[0].local_to_global].copy()).cuda(), None, 2, 2, 1)
    ref = O.cycle(olevels, 0, b, np.zeros_like(b), 2, 2, 1)
    loc, glob = H.layouts[0].owned_pairs()
    out = np.empty_like(ref)
    out[glob] = _np(x)[loc]
    assert rel(out, ref) < TOL


def test_row_chunked_operator_matches_whole(P):
    """RowChunkedOperator (element blocks condensed and streamed by row chunks,
    hdg_level_fill_stored_rows) applies exactly the operator of the whole-mesh build, on the
    configs[4] coefficient law; chunk boundaries at every row parity."""
    from paper_1705_09907_b200.trace import RowChunkedOperator
    from test_local_strips_cpu import _specs
    n, p = 24, 4
    spec, ospec = _specs("aniso", n)
    x = np.random.default_rng(8).uniform(-1, 1, 2 * n * (n - 1) * (p + 1))
    whole = P.tr.TraceSystem(P.mesh(n, n), p, spec).matvec_free(x)
    for rows in (1, 5, 8, 24):
        got = RowChunkedOperator(P.mesh(n, n), p, spec, rows_per_chunk=rows).apply(x)
        assert rel(got, whole) < 1e-14, rows
    o = O.OracleTrace(O.Grid(n, n), p, ospec)
    assert rel(whole, o.matvec(x)) < TOL
