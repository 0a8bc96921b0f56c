"""Freeze golden vectors from the UNMODIFIED reference `hdgmg` (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is imported read-only from /root/reference (it does not exist on
the GPU box, so nothing else may read it).  Every array written here comes out
of the reference's own public functions:
  TraceSystem (trace.py:29-69), matvec_free (:87-94), assemble_csr (:98-128),
  build_hierarchy (multigrid.py:301-342), p/h_prolongation (:215-298),
  v_cycle / solve_mg (:409-439), fsai_build (:123-159), solve_cg (trace.py:142-163).
Two builder additions ride on the reference objects: the
edge block-Jacobi smoother class `BJ` below (plugged into MGLevel.smoother, the
duck-typed slot multigrid.py:397-405 uses), and the nodal-source / piecewise-K
callables handed to ProblemSpec.
"""

import os
import sys
import time

import numpy as np

from hdgmg.basis import eval_matrix, gll_nodes_weights
from hdgmg.mesh import build_cartesian
from hdgmg.multigrid import build_hierarchy, mg_preconditioner, solve_mg, v_cycle
from hdgmg.problem import ProblemSpec, constant_problem, manufactured_problem
from hdgmg.trace import TraceSystem

OUT = os.path.dirname(os.path.abspath(__file__))


class BJ:
    """Edge block-Jacobi (north star; not in the reference): x += w D^-1 (b - A x)."""

    def __init__(self, A, n1, omega=0.8):
        A = A.tocsr()
        nb = A.shape[0] // n1
        D = np.stack([A[b * n1:(b + 1) * n1, b * n1:(b + 1) * n1].toarray() for b in range(nb)])
        self.Dinv = np.linalg.inv(D)
        self.n1, self.omega = n1, omega
        self.complexity = nb * n1 * n1 / A.nnz

    def smooth(self, matvec, b, x, steps):
        for _ in range(steps):
            r = (b - matvec(x)).reshape(-1, self.n1)
            x = x + self.omega * np.einsum("bij,bj->bi", self.Dinv, r).reshape(-1)
        return x


def attach_bj(levels, omega=0.8):
    for lev in levels[:-1]:
        lev.smoother = BJ(lev.operator, lev.p + 1, omega)
    return levels


def nodal_source(f, n, p):
    basis = gll_nodes_weights(p)

    def src(x, y):
        x = np.asarray(x, float)
        y = np.asarray(y, float)
        i = np.clip(np.floor(x * n).astype(np.int64), 0, n - 1)
        j = np.clip(np.floor(y * n).astype(np.int64), 0, n - 1)
        Ex = eval_matrix(basis, (2.0 * (x * n - i) - 1.0).ravel())
        Ey = eval_matrix(basis, (2.0 * (y * n - j) - 1.0).ravel())
        v = f[(j * n + i).ravel()].reshape(-1, p + 1, p + 1)
        return np.einsum("qb,qa,qba->q", Ey, Ex, v).reshape(x.shape)

    return src


def piecewise_K(Kg):
    ny, nx = Kg.shape

    def coef(x, y):
        i = np.clip(np.floor(np.asarray(x) * nx).astype(np.int64), 0, nx - 1)
        j = np.clip(np.floor(np.asarray(y) * ny).astype(np.int64), 0, ny - 1)
        return Kg[j, i]

    return coef


def zero(x, y):
    return np.zeros_like(np.asarray(x, float))


def one(x, y):
    return np.ones_like(np.asarray(x, float))


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print(f"wrote {name}: " + ", ".join(f"{k}{np.shape(v)}" for k, v in arrays.items()))


def small_systems():
    """matvec / rhs / blocks for the manufactured (tanh K, bump) problem."""
    spec = manufactured_problem()
    out = {}
    for n, p in [(2, 1), (4, 2), (4, 3), (8, 1), (8, 2), (8, 5), (3, 2)]:
        s = TraceSystem(build_cartesian(n, n), p, spec)
        rng = np.random.default_rng(n * 100 + p)  # test_trace.py:43
        x = rng.standard_normal(s.ndof)
        out[f"n{n}p{p}_x"] = x
        out[f"n{n}p{p}_y"] = s.matvec_free(x)
        out[f"n{n}p{p}_rhs"] = s.rhs
        if n <= 4:
            out[f"n{n}p{p}_schur"] = s.schur
    # K = I, tau = 1 blocks (the shared-block class, F2) at p = 1..8
    for p in range(1, 9):
        s = TraceSystem(build_cartesian(4, 4), p, constant_problem(0.0, 1.0))
        out[f"kI_n4p{p}_schur5"] = s.schur[5]   # interior element of 4x4
        out[f"kI_n4p{p}_schur0"] = s.schur[0]   # corner element
    save("small_systems.npz", **out)


def hierarchies():
    """Transfers + Galerkin operators + cycles on small hierarchies."""
    out = {}
    spec = manufactured_problem()
    for tag, n, p in [("m8p3", 8, 3), ("m4p2", 4, 2)]:
        levels = build_hierarchy(build_cartesian(n, n), p, spec, smoother="baseline")
        rng = np.random.default_rng(7)
        for k, lev in enumerate(levels):
            v = rng.standard_normal(lev.ndof)
            out[f"{tag}_L{k}_v"] = v
            out[f"{tag}_L{k}_Av"] = lev.operator @ v
            out[f"{tag}_L{k}_shape"] = np.array([lev.mesh.n_x, lev.p, lev.ndof])
            if lev.prolong is not None:
                vc = rng.standard_normal(lev.prolong.shape[1])
                out[f"{tag}_L{k}_Pv"] = lev.prolong @ vc
                out[f"{tag}_L{k}_Pv_in"] = vc
                out[f"{tag}_L{k}_PTv"] = lev.prolong.T @ v
        x, mon = solve_mg(levels, cycle="v")
        out[f"{tag}_fsai_res"] = np.array(mon.residuals)
        out[f"{tag}_fsai_x"] = x
        out[f"{tag}_fsai_lam"] = np.array([lev.smoother.lam_max for lev in levels[:-1]])
        attach_bj(levels)
        b = levels[0].rhs
        out[f"{tag}_bj_x1"] = v_cycle(levels, b)
        x, mon = solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
        out[f"{tag}_bj_res"] = np.array(mon.residuals)
        xw, monw = solve_mg(levels, b=b, cycle="w", tol=1e-10, max_cycles=400)
        out[f"{tag}_bjw_res"] = np.array(monw.residuals)
    # K = I with g_D = 0 (the shared-block path), 16x16 p=4, seeded trace RHS
    levels = build_hierarchy(build_cartesian(16, 16), 4, constant_problem(0.0, 1.0), smoother=None)
    attach_bj(levels)
    b = np.random.default_rng(3).uniform(-1, 1, levels[0].ndof)
    out["kI16p4_b"] = b
    out["kI16p4_bj_x1"] = v_cycle(levels, b)
    x, mon = solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    out["kI16p4_bj_res"] = np.array(mon.residuals)
    out["kI16p4_ndofs"] = np.array([lev.ndof for lev in levels])
    # heterogeneous piecewise-constant K (cfg3 flavour), 8x8 p=2, MG-PCG and V-cycle
    rng = np.random.default_rng(2)
    Kg = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), (8, 8)))
    spec_h = ProblemSpec(piecewise_K(Kg), zero, zero, 1.0)
    levels = build_hierarchy(build_cartesian(8, 8), 2, spec_h, smoother=None)
    attach_bj(levels)
    b = rng.uniform(-1, 1, levels[0].ndof)
    out["het8p2_K"] = Kg
    out["het8p2_b"] = b
    out["het8p2_y"] = levels[0].system.matvec_free(b)
    out["het8p2_bj_x1"] = v_cycle(levels, b)
    x, mon = solve_mg(levels, b=b, tol=1e-10, max_cycles=2000)
    out["het8p2_bj_res"] = np.array(mon.residuals)
    system = levels[0].system
    system.rhs = b  # solve_cg reads self.rhs (trace.py:145)
    xc, it = system.solve_cg(tol=1e-10, precond=mg_preconditioner(levels))
    out["het8p2_pcg_iters"] = np.array([it])
    out["het8p2_pcg_x"] = xc
    for k, lev in enumerate(levels):
        v = np.random.default_rng(100 + k).standard_normal(lev.ndof)
        out[f"het8p2_L{k}_Av"] = lev.operator @ v
    save("hierarchies.npz", **out)


def postprocessing():
    """reconstruct_all (trace.py:171-178) and postprocess_all (:180-185) of random traces."""
    out = {}
    for tag, spec, n, p in [("m4p2", manufactured_problem(), 4, 2), ("m5p3", manufactured_problem(), 5, 3),
                            ("m6p1", manufactured_problem(), 6, 1), ("kI4p4", constant_problem(0.0, 1.0), 4, 4)]:
        s = TraceSystem(build_cartesian(n, n), p, spec)
        lam = np.random.default_rng(7 * n + p).standard_normal(s.ndof)
        q, u = s.reconstruct_all(lam)
        out[f"{tag}_lam"], out[f"{tag}_q"], out[f"{tag}_u"] = lam, q, u
        out[f"{tag}_ustar"] = s.postprocess_all(q, u)
    save("postprocess.npz", **out)


def config1():
    """BASELINE configs[0]: 64x64, p=2, K=1, g_D=0, nodal f ~ U[-1,1] (seed 0);
    one matvec + one V(2,2) BJ(0.8) cycle on levels[:6] (down to 4x4); full solve."""
    n, p = 64, 2
    f = np.random.default_rng(0).uniform(-1.0, 1.0, (n * n, (p + 1) ** 2))
    spec = ProblemSpec(one, nodal_source(f, n, p), zero, 1.0)
    t = time.time()
    levels = build_hierarchy(build_cartesian(n, n), p, spec, smoother=None)[:6]
    attach_bj(levels)
    print(f"cfg1 hierarchy {time.time() - t:.1f}s", [(l.mesh.n_x, l.p, l.ndof) for l in levels])
    fine = levels[0]
    b = fine.rhs
    Ab = fine.matvec(b)
    x1 = v_cycle(levels, b)
    r1 = np.linalg.norm(b - fine.matvec(x1)) / np.linalg.norm(b)
    x, mon = solve_mg(levels, b=b, tol=1e-10, max_cycles=400)
    print(f"cfg1: 1 cycle rel res {r1:.6f}; solve {len(mon.residuals) - 1} cycles, "
          f"rate {mon.asymptotic_rate():.5f}, final {mon.residuals[-1] / np.linalg.norm(b):.3e}")
    save("config1.npz", b=b, Ab=Ab, x1=x1, r1=np.array([r1]), res=np.array(mon.residuals), x=x)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "hier", "cfg1", "post"]
    if "small" in which:
        small_systems()
    if "hier" in which:
        hierarchies()
    if "cfg1" in which:
        config1()
    if "post" in which:
        postprocessing()
