"""Pin the CPU oracle to golden vectors frozen from the unmodified reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import hdg_oracle as O

import specs


def history_close(got, ref):
    """Residual histories: identical lengths (iteration counts); each entry within
    1e-5 relative or 1e-10 of the initial residual (north star: final within 1e-10)."""
    got, ref = np.asarray(got), np.asarray(ref)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-10 * ref[0])


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def bump_spec():
    return specs.manufactured(O.Spec)


@pytest.mark.parametrize("n,p", [(2, 1), (4, 2), (4, 3), (8, 1), (8, 2), (8, 5), (3, 2)])
def test_oracle_matvec_rhs_blocks(golden, n, p):
    g = golden("small_systems.npz")
    s = O.OracleTrace(O.Grid(n, n), p, bump_spec())
    key = f"n{n}p{p}"
    assert rel(s.matvec(g[key + "_x"]), g[key + "_y"]) < 1e-13
    assert rel(s.rhs, g[key + "_rhs"]) < 1e-12
    if key + "_schur" in g:
        assert rel(s.schur, g[key + "_schur"]) < 1e-13
    # CSR oracle agrees with the matrix-free form (test_trace.py:38-48)
    x = g[key + "_x"]
    assert rel(s.csr() @ x, s.matvec(x)) < 1e-13


@pytest.mark.parametrize("p", range(1, 9))
def test_oracle_kI_blocks(golden, p):
    g = golden("small_systems.npz")
    s = O.OracleTrace(O.Grid(4, 4), p, O.constant_spec(0.0, 1.0))
    assert rel(s.schur[5], g[f"kI_n4p{p}_schur5"]) < 1e-12
    assert rel(s.schur[0], g[f"kI_n4p{p}_schur0"]) < 1e-12


def test_injected_system_is_bit_identical():
    full = O.OracleTrace(O.Grid(16, 16), 2, O.constant_spec(0.0, 1.0))
    inj = O.injected_shared_system(16, 2)
    np.testing.assert_array_equal(full.schur, inj.schur)


@pytest.mark.parametrize("tag,n,p", [("m8p3", 8, 3), ("m4p2", 4, 2)])
def test_oracle_hierarchy(golden, tag, n, p):
    g = golden("hierarchies.npz")
    levels = O.build_levels(O.Grid(n, n), p, bump_spec(), smoother="baseline")
    for k, lev in enumerate(levels):
        assert tuple(g[f"{tag}_L{k}_shape"]) == (lev.grid.n_x, lev.p, lev.ndof)
        assert rel(lev.operator @ g[f"{tag}_L{k}_v"], g[f"{tag}_L{k}_Av"]) < 1e-12
        if lev.prolong is not None:
            assert rel(lev.prolong @ g[f"{tag}_L{k}_Pv_in"], g[f"{tag}_L{k}_Pv"]) < 1e-12
            assert rel(lev.prolong.T @ g[f"{tag}_L{k}_v"], g[f"{tag}_L{k}_PTv"]) < 1e-12
    assert rel([l.smoother.lam_max for l in levels[:-1]], g[f"{tag}_fsai_lam"]) < 1e-10
    x, mon = O.solve_mg(levels)
    ref = g[f"{tag}_fsai_res"]
    history_close(mon.residuals, ref)
    assert rel(x, g[f"{tag}_fsai_x"]) < 1e-10
    O.attach(levels, "blockjacobi", 0.8)
    b = levels[0].rhs
    assert rel(O.v_cycle(levels, b), g[f"{tag}_bj_x1"]) < 1e-12
    _, mon = O.solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    history_close(mon.residuals, g[f"{tag}_bj_res"])
    _, monw = O.solve_mg(levels, b=b, cyc="w", tol=1e-10, max_cycles=400)
    assert len(monw.residuals) == len(g[f"{tag}_bjw_res"])


def test_oracle_kI_hierarchy(golden):
    g = golden("hierarchies.npz")
    levels = O.build_levels(O.Grid(16, 16), 4, O.constant_spec(0.0, 1.0), smoother="blockjacobi")
    assert [l.ndof for l in levels] == list(g["kI16p4_ndofs"])
    b = g["kI16p4_b"]
    assert rel(O.v_cycle(levels, b), g["kI16p4_bj_x1"]) < 1e-12
    _, mon = O.solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    history_close(mon.residuals, g["kI16p4_bj_res"])


def test_oracle_heterogeneous(golden):
    g = golden("hierarchies.npz")
    spec = O.Spec(O.piecewise_coefficient(g["het8p2_K"]),
                  lambda x, y: np.zeros_like(np.asarray(x, float)),
                  lambda x, y: np.zeros_like(np.asarray(x, float)), 1.0)
    levels = O.build_levels(O.Grid(8, 8), 2, spec, smoother="blockjacobi")
    b = g["het8p2_b"]
    assert rel(levels[0].matvec(b), g["het8p2_y"]) < 1e-12
    for k, lev in enumerate(levels):
        v = np.random.default_rng(100 + k).standard_normal(lev.ndof)
        assert rel(lev.operator @ v, g[f"het8p2_L{k}_Av"]) < 1e-12
    assert rel(O.v_cycle(levels, b), g["het8p2_bj_x1"]) < 1e-12
    x, it = levels[0].system.solve_cg(b=b, tol=1e-10, precond=O.mg_preconditioner(levels))
    assert it == int(g["het8p2_pcg_iters"][0])
    assert rel(x, g["het8p2_pcg_x"]) < 1e-9


@pytest.mark.slow
def test_oracle_config1(golden):
    g = golden("config1.npz")
    grid, spec = O.config1_system()
    levels = O.build_levels(grid, 2, spec)[:6]
    O.attach(levels, "blockjacobi", 0.8)
    b = levels[0].rhs
    assert rel(b, g["b"]) < 1e-12
    assert rel(levels[0].matvec(b), g["Ab"]) < 1e-12
    x1 = O.v_cycle(levels, b)
    assert rel(x1, g["x1"]) < 1e-12
    r1 = np.linalg.norm(b - levels[0].matvec(x1)) / np.linalg.norm(b)
    assert abs(r1 - 0.267064) < 5e-7
    _, mon = O.solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    assert len(mon.residuals) == len(g["res"]) == 93
    np.testing.assert_allclose(mon.rho, np.array(g["res"][1:]) / g["res"][:-1], rtol=1e-5)


POST_CASES = [("m4p2", "m", 4, 2), ("m5p3", "m", 5, 3), ("m6p1", "m", 6, 1), ("kI4p4", "kI", 4, 4)]


@pytest.mark.parametrize("tag,kind,n,p", POST_CASES)
def test_oracle_reconstruct_postprocess(golden, tag, kind, n, p):
    g = golden("postprocess.npz")
    spec = specs.manufactured(O.Spec) if kind == "m" else specs.constant(O.Spec, 0.0, 1.0)
    s = O.OracleTrace(O.Grid(n, n), p, spec)
    q, u = O.reconstruct_all(s, g[f"{tag}_lam"])
    scale = lambda a: max(np.abs(a).max(), 1e-300)
    assert np.abs(q - g[f"{tag}_q"]).max() <= 1e-12 * scale(g[f"{tag}_q"])
    assert np.abs(u - g[f"{tag}_u"]).max() <= 1e-12 * scale(g[f"{tag}_u"])
    us = O.postprocess_all(s, g[f"{tag}_q"], g[f"{tag}_u"])
    assert np.abs(us - g[f"{tag}_ustar"]).max() <= 1e-12 * scale(g[f"{tag}_ustar"])
