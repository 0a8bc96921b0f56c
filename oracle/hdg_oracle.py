"""CPU ORACLE for the HDG trace matvec + geometric-multigrid hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_1705_09907_b200/`) imports this file; only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py` may.  It is the checker, never the thing measured or shipped.

What it is: a plain numpy/scipy restatement of the reference `hdgmg`
package's algorithm for the hot path (reference = `/root/reference`, which is
NOT available on the GPU box).  Each function cites the reference file:line it
follows.  The restatement is deliberately loop-based and literal (per-element
local solves, explicit CSR assembly, CSR Galerkin products), i.e. a different
code path from the product's batched/vectorised setup and CUDA kernels.

Parity pin: `tests/golden/make_golden.py` ran the UNMODIFIED reference in the
build container and froze its outputs in `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this oracle against every one of them.

Additions that the reference does not contain (all marked "builder restatement"):
  * `BlockJacobiSmoother` - the north-star edge block-Jacobi smoother;
  * `nodal_source` - "f uniform per element DOF" adapter;
  * `piecewise_coefficient` - per-element constant K callable;
  * `injected_shared_system` - the K=I large-mesh system built from one block
    (SURVEY 8c (2)); bit-identical to a full build (pinned in tests).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from numpy.polynomial import legendre as npleg
from scipy.linalg import lu_factor, lu_solve
from scipy.special import roots_jacobi

SNAP = 1e-14  # basis.py:17 NODE_SNAP_TOL
OUT_NORMAL = ((0.0, -1.0), (1.0, 0.0), (0.0, 1.0), (-1.0, 0.0))  # mesh.py:15 (b, r, t, l)


# ----------------------------------------------------------------------------- basis
# basis.py:42-116


def bary(nodes):
    """basis.py:42-56 - product-formula barycentric weights, max|w|=1, w0>0."""
    x = np.asarray(nodes, float)
    w = np.empty(x.size)
    for j in range(x.size):
        prod = 1.0
        for k in range(x.size):
            if k != j:
                prod *= x[j] - x[k]
        w[j] = 1.0 / prod
    w /= np.abs(w).max()
    return -w if w[0] < 0 else w


@dataclass(frozen=True)
class Rule:
    nodes: np.ndarray
    weights: np.ndarray
    bw: np.ndarray


def gll(p):
    """basis.py:59-69 - GLL nodes: +-1 and the roots of P^(1,1)_{p-1}."""
    if p < 1:
        raise ValueError("GLL needs p >= 1")
    x = np.empty(p + 1)
    x[0], x[-1] = -1.0, 1.0
    if p > 1:
        x[1:-1] = roots_jacobi(p - 1, 1.0, 1.0)[0]
    c = np.zeros(p + 1)
    c[p] = 1.0
    w = 2.0 / (p * (p + 1) * npleg.legval(x, c) ** 2)
    return Rule(x, w, bary(x))


def gauss(p):
    """basis.py:72-77 - Gauss-Legendre with p+1 points."""
    x, w = npleg.leggauss(p + 1)
    return Rule(x, w, bary(x))


def lagrange_at(rule, pts):
    """basis.py:91-105 - V[q, j] = l_j(pts[q]) by the 2nd barycentric form, snapping."""
    pts = np.atleast_1d(np.asarray(pts, float))
    out = np.zeros((pts.size, rule.nodes.size))
    for q, t in enumerate(pts):
        d = t - rule.nodes
        hit = np.flatnonzero(np.abs(d) < SNAP)
        if hit.size:
            out[q, hit[0]] = 1.0
            # the reference sets every snapped column to 1 (at most one can hit)
            out[q, hit] = 1.0
            continue
        row = rule.bw / d
        out[q] = row / row.sum()
    return out


def deriv_at_nodes(rule):
    """basis.py:108-116 - D[i, j] = l_j'(x_i), diagonal by negative row sum."""
    x, w = rule.nodes, rule.bw
    n = x.size
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i, j] = (w[j] / w[i]) / (x[i] - x[j])
        D[i, i] = -D[i].sum()
    return D


class RefElem:
    """basis.py:119-181 - GLL interpolation, GL quadrature with p+1 points."""

    def __init__(self, p):
        self.p = p
        self.basis = gll(p)
        self.quad = gauss(p)
        self.E = lagrange_at(self.basis, self.quad.nodes)  # interp_1d
        self.dE = self.E @ deriv_at_nodes(self.basis)       # deriv_1d
        self.w2 = np.kron(self.quad.weights, self.quad.weights)
        self.I2 = np.kron(self.E, self.E)
        self.Dxi = np.kron(self.E, self.dE)
        self.Deta = np.kron(self.dE, self.E)

    def quad_xy(self, x0, y0, dx, dy):
        """basis.py:157-162 - row index eta, column xi; flatten = j*nq + i."""
        qx = x0 + dx * (self.quad.nodes + 1.0) / 2.0
        qy = y0 + dy * (self.quad.nodes + 1.0) / 2.0
        return np.tile(qx, qy.size), np.repeat(qy, qx.size)


# ------------------------------------------------------------------------------ mesh
# mesh.py:112-196


class Grid:
    """Structured mesh with the reference facet numbering (mesh.py:3-8, 112-163)."""

    def __init__(self, nx, ny, x0=0.0, x1=1.0, y0=0.0, y1=1.0, children=None):
        if nx < 1 or ny < 1:
            raise ValueError("mesh needs positive element counts")
        self.n_x, self.n_y = nx, ny
        self.x0, self.y0 = x0, y0
        self.dx, self.dy = (x1 - x0) / nx, (y1 - y0) / ny
        self.extent = ((x0, x1), (y0, y1))
        nh = nx * (ny + 1)
        nv = ny * (nx + 1)
        self.n_h = nh
        self.n_facets = nh + nv
        self.n_elems = nx * ny
        self.axis = np.r_[np.zeros(nh, np.int8), np.ones(nv, np.int8)]
        self.e2f = np.empty((self.n_elems, 4), np.int64)
        self.f2e = np.full((self.n_facets, 2, 2), -1, np.int64)
        H = lambda i, j: j * nx + i                      # mesh.py:112-113
        V = lambda i, j: nh + i * ny + j                 # mesh.py:116-117
        for j in range(ny):
            for i in range(nx):
                e = j * nx + i
                fb, fr, ft, fl = H(i, j), V(i + 1, j), H(i, j + 1), V(i, j)
                self.e2f[e] = (fb, fr, ft, fl)
                self.f2e[ft, 0] = (e, 2)
                self.f2e[fb, 1] = (e, 0)
                self.f2e[fr, 0] = (e, 1)
                self.f2e[fl, 1] = (e, 3)
        self.boundary = np.zeros(self.n_facets, bool)
        for i in range(nx):
            self.boundary[H(i, 0)] = self.boundary[H(i, ny)] = True
        for j in range(ny):
            self.boundary[V(0, j)] = self.boundary[V(nx, j)] = True
        self.children = children

    @property
    def interior(self):
        return np.flatnonzero(~self.boundary)

    def origin(self, e):
        return self.x0 + (e % self.n_x) * self.dx, self.y0 + (e // self.n_x) * self.dy

    def facet_xy(self, f, t):
        """mesh.py:76-90 - physical points at tangent parameter t in [-1, 1]."""
        t = np.asarray(t, float)
        if self.axis[f] == 0:
            i, j = f % self.n_x, f // self.n_x
            s = self.dx * (t + 1.0) / 2.0
            return self.x0 + i * self.dx + s, self.y0 + j * self.dy + 0.0 * s
        k = f - self.n_h
        i, j = k // self.n_y, k % self.n_y
        s = self.dy * (t + 1.0) / 2.0
        return self.x0 + i * self.dx + 0.0 * s, self.y0 + j * self.dy + s


def coarsen_grid(g):
    """mesh.py:166-196 - 2x2 agglomeration; children (SW, SE, NW, NE)."""
    if g.n_x % 2 or g.n_y % 2:
        raise ValueError("odd mesh cannot be coarsened")
    nx, ny = g.n_x // 2, g.n_y // 2
    kids = np.empty((nx * ny, 4), np.int64)
    for cj in range(ny):
        for ci in range(nx):
            base = 2 * cj * g.n_x + 2 * ci
            kids[cj * nx + ci] = (base, base + 1, base + g.n_x, base + g.n_x + 1)
    x0, x1, y0, y1 = g.x0, g.x0 + g.n_x * g.dx, g.y0, g.y0 + g.n_y * g.dy
    return Grid(nx, ny, x0, x1, y0, y1, children=kids)


# ------------------------------------------------------------------------ local solve
# local.py:35-237


def side_nodes(p):
    """local.py:35-43 - volume node ids per side, ordered along the tangent."""
    n = p + 1
    k = np.arange(n)
    return (k, p + k * n, p * n + k, k * n)


class ElementCore:
    """Per-(mesh, p) reference data - local.py:46-70."""

    def __init__(self, grid, p):
        self.grid, self.p, self.n1 = grid, p, p + 1
        self.ref = RefElem(p)
        self.nb = (p + 1) ** 2
        q = self.ref.quad
        self.mass1 = self.ref.E.T @ np.diag(q.weights) @ self.ref.E
        lens = (grid.dx, grid.dy, grid.dx, grid.dy)
        self.fmass = [0.5 * lens[s] * self.mass1 for s in range(4)]
        self.sides = side_nodes(p)
        self.jac = grid.dx * grid.dy / 4.0

    def project(self, func, e, s):
        """local.py:72-78 - facet L2 projection onto the GLL trace basis."""
        f = self.grid.e2f[e, s]
        x, y = self.grid.facet_xy(f, self.ref.quad.nodes)
        g = np.asarray(func(x, y), float)
        return np.linalg.solve(self.mass1, self.ref.E.T @ (self.ref.quad.weights * g))


class Local:
    """One element's factorised local system + condensed block (local.py:81-98, 204-237)."""

    def __init__(self, core, e, spec, tau_per_facet=None):
        g, n1, nb = core.grid, core.n1, core.nb
        ref = core.ref
        x0, y0 = g.origin(e)
        qx, qy = ref.quad_xy(x0, y0, g.dx, g.dy)
        kq = spec.coefficient(qx, qy)                                # local.py:138
        # builder restatement: a (Kxx, Kyy) pair = anisotropic diagonal K, with one
        # flux mass per component; a scalar field is the reference's isotropic case
        kx, ky = (kq if isinstance(kq, tuple) else (kq, kq))
        kx, ky = np.asarray(kx, float), np.asarray(ky, float)
        if np.any(kx <= 0) or np.any(ky <= 0):
            raise RuntimeError(f"coefficient not positive on element {e}")
        fq = np.asarray(spec.source(qx, qy), float)
        wj = ref.w2 * core.jac
        M = ref.I2.T @ np.diag(wj / kx) @ ref.I2                    # local.py:144
        My = ref.I2.T @ np.diag(wj / ky) @ ref.I2
        Bx = 0.5 * g.dy * ref.I2.T @ np.diag(ref.w2) @ ref.Dxi     # local.py:146
        By = 0.5 * g.dx * ref.I2.T @ np.diag(ref.w2) @ ref.Deta
        facets = g.e2f[e]
        tau = (np.full(4, spec.tau) if tau_per_facet is None
               else np.asarray(tau_per_facet, float)[facets])
        inner = ~g.boundary[facets]
        nt = 4 * n1
        stab = np.zeros((nb, nb))
        T = np.zeros((3 * nb, nt))        # [trace_to_flux; trace_to_potential]
        F = np.zeros((nt, 3 * nb))        # facet_coupling
        Ms = np.zeros((nt, nt))           # facet_mass_stab
        for s in range(4):                                           # local.py:162-176
            m = core.fmass[s]
            ids = core.sides[s]
            r = slice(s * n1, (s + 1) * n1)
            stab[np.ix_(ids, ids)] += tau[s] * m
            for d in (0, 1):
                nd = OUT_NORMAL[s][d]
                if nd != 0.0:
                    T[d * nb + ids, r] += nd * m
                    F[r, d * nb + ids] += nd * m
            T[2 * nb + ids, r] += -tau[s] * m
            F[r, 2 * nb + ids] += tau[s] * m
            if inner[s]:
                Ms[r, r] += tau[s] * m
        lam_bc = np.zeros(nt)                                        # local.py:179-184
        for s in range(4):
            if not inner[s]:
                lam_bc[s * n1:(s + 1) * n1] = core.project(spec.dirichlet, e, s)
        load = -T @ lam_bc
        load[2 * nb:] += ref.I2.T @ (wj * fq)
        cmask = np.repeat(inner, n1)                                 # local.py:186-188
        T[:, ~cmask] = 0.0
        Lmat = np.zeros((3 * nb, 3 * nb))                            # local.py:116-126
        Lmat[:nb, :nb] = M
        Lmat[nb:2 * nb, nb:2 * nb] = My
        Lmat[:2 * nb, 2 * nb:] = -np.hstack([Bx, By]).T
        Lmat[2 * nb:, :2 * nb] = np.hstack([Bx, By])
        Lmat[2 * nb:, 2 * nb:] = stab
        self.lu = lu_factor(Lmat)                                    # local.py:208
        self.trace_cols, self.load, self.inner = T, load, inner
        sol = lu_solve(self.lu, np.column_stack([T, load]))          # local.py:233-236
        self.schur = F @ sol[:, :-1] + Ms
        self.schur_load = F @ sol[:, -1]


# ---------------------------------------------------------------------- trace system
# trace.py:26-131


class OracleTrace:
    """trace.py:26-69 - stacked condensed blocks + gather/owner maps."""

    def __init__(self, grid, p, spec, tau_per_facet=None, *, _blocks=None):
        self.mesh = self.grid = grid
        self.spec = spec
        self.p, self.n1 = p, p + 1
        self.core = ElementCore(grid, p)
        self.interior = grid.interior
        self.n_blocks = self.interior.size
        self.ndof = self.n1 * self.n_blocks
        self.block_of = np.full(grid.n_facets, -1, np.int64)
        self.block_of[self.interior] = np.arange(self.n_blocks)
        blk = self.block_of[grid.e2f]
        self.side_ok = blk >= 0
        self.gidx = (np.where(self.side_ok, blk, 0)[:, :, None] * self.n1
                     + np.arange(self.n1)).reshape(grid.n_elems, -1)
        self.gmask = np.repeat(self.side_ok, self.n1, axis=1)
        self.owners = grid.f2e[self.interior]
        if _blocks is None:
            self.locals = [Local(self.core, e, spec, tau_per_facet) for e in range(grid.n_elems)]
            self.schur = np.stack([l.schur for l in self.locals])
            loads = np.stack([l.schur_load for l in self.locals])
            self.rhs = self._sum_owners(loads)
        else:
            self.locals = None
            self.schur = _blocks
            self.rhs = np.zeros(self.ndof)
        self._csr = None

    def _sum_owners(self, per_elem):
        """trace.py:73-79 - facet block = slot-0 owner + slot-1 owner."""
        y3 = per_elem.reshape(self.grid.n_elems, 4, self.n1)
        o = self.owners
        return (y3[o[:, 0, 0], o[:, 0, 1]] + y3[o[:, 1, 0], o[:, 1, 1]]).reshape(-1)

    def matvec(self, x):
        """trace.py:87-94 - gather, per-element GEMV, two-owner sum."""
        x = np.asarray(x, float)
        if self.ndof == 0:
            return np.zeros(0)
        xe = np.where(self.gmask, x[self.gidx], 0.0)
        return self._sum_owners(np.einsum("eij,ej->ei", self.schur, xe))

    def csr(self):
        """trace.py:98-128 - explicit assembly of every interior (row, col) block."""
        if self._csr is None:
            n1 = self.n1
            R, C, Vv = [], [], []
            ar = np.arange(n1)
            for e in range(self.grid.n_elems):
                b = self.block_of[self.grid.e2f[e]]
                for si in range(4):
                    if b[si] < 0:
                        continue
                    for sj in range(4):
                        if b[sj] < 0:
                            continue
                        rr, cc = np.meshgrid(b[si] * n1 + ar, b[sj] * n1 + ar, indexing="ij")
                        R.append(rr.ravel())
                        C.append(cc.ravel())
                        Vv.append(self.schur[e, si * n1:(si + 1) * n1, sj * n1:(sj + 1) * n1].ravel())
            if R:
                self._csr = sp.coo_matrix((np.concatenate(Vv), (np.concatenate(R), np.concatenate(C))),
                                          shape=(self.ndof, self.ndof)).tocsr()
            else:
                self._csr = sp.csr_matrix((0, 0))
        return self._csr

    def solve_direct(self, b=None):
        b = self.rhs if b is None else b
        if self.ndof == 0:
            return np.zeros(0)
        return spla.splu(self.csr().tocsc()).solve(b)

    def solve_cg(self, b=None, tol=1e-12, maxiter=5000, precond=None, x0=None, hist=None):
        """trace.py:142-163 - (preconditioned) CG; returns (x, iterations).  `hist` (a list, test
        instrumentation only) receives ||r|| at every stop test."""
        b = self.rhs if b is None else b
        x = np.zeros_like(b) if x0 is None else x0.copy()
        r = b - self.matvec(x)
        z = precond(r) if precond else r
        d = z.copy()
        rz = r @ z
        bn = np.linalg.norm(b) or 1.0
        for it in range(maxiter):
            rn = np.linalg.norm(r)
            if hist is not None:
                hist.append(rn)
            if rn <= tol * bn:
                return x, it
            ad = self.matvec(d)
            a = rz / (d @ ad)
            x += a * d
            r -= a * ad
            z = precond(r) if precond else r
            rz2 = r @ z
            d = z + (rz2 / rz) * d
            rz = rz2
        return x, maxiter


def reconstruct_all(system, lam):
    """trace.py:171-178 / local.py:240-251: (q, u) per element from the trace solution."""
    nb = system.core.nb
    q = np.empty((system.grid.n_elems, 2 * nb))
    u = np.empty((system.grid.n_elems, nb))
    xe = np.where(system.gmask, np.asarray(lam, float)[system.gidx], 0.0)
    for e, l in enumerate(system.locals):
        sol = lu_solve(l.lu, l.load - l.trace_cols @ xe[e])
        q[e], u[e] = sol[:2 * nb], sol[2 * nb:]
    return q, u


def postprocess_all(system, q, u):
    """trace.py:180-185 / local.py:254-299: superconvergent potential of order p+1 per element,
    a local Neumann problem (grad u*, grad w) = -(K^-1 q_h, grad w) with the element mean of u*
    pinned to that of u_h (KKT system, LU-solved).  A (Kxx, Kyy) pair divides each flux
    component by its own coefficient (builder extension)."""
    g, p = system.grid, system.p
    ref_p, ref = RefElem(p), RefElem(p + 1)
    nb, nb2 = (p + 1) ** 2, (p + 2) ** 2
    cross = lagrange_at(ref_p.basis, ref.quad.nodes)
    interp = np.kron(cross, cross)
    w2 = ref.w2
    stiff = (g.dy / g.dx) * ref.Dxi.T @ (w2[:, None] * ref.Dxi) \
        + (g.dx / g.dy) * ref.Deta.T @ (w2[:, None] * ref.Deta)
    jac = g.dx * g.dy / 4.0
    mean_row = jac * (ref.I2.T @ w2)
    kkt = np.zeros((nb2 + 1, nb2 + 1))
    kkt[:nb2, :nb2] = stiff
    kkt[:nb2, nb2] = mean_row
    kkt[nb2, :nb2] = mean_row
    lu = lu_factor(kkt)
    out = np.empty((g.n_elems, nb2))
    for e in range(g.n_elems):
        qx, qy = ref.quad_xy(*g.origin(e), g.dx, g.dy)
        kq = system.spec.coefficient(qx, qy)
        kx, ky = (kq if isinstance(kq, tuple) else (kq, kq))
        qh_x = interp @ q[e, :nb]
        qh_y = interp @ q[e, nb:]
        rhs = -0.5 * g.dy * ref.Dxi.T @ (w2 * qh_x / np.asarray(kx, float))
        rhs += -0.5 * g.dx * ref.Deta.T @ (w2 * qh_y / np.asarray(ky, float))
        mean_u = jac * w2 @ (interp @ u[e])
        out[e] = lu_solve(lu, np.concatenate([rhs, [mean_u]]))[:-1]
    return out


def exact_trace(system, func):
    """trace.py:188-195: facet L2 projection of func onto the interior trace space."""
    lam = np.zeros(system.ndof)
    n1 = system.n1
    for bi, f in enumerate(system.interior):
        e, side = system.grid.f2e[f, 0]
        lam[bi * n1:(bi + 1) * n1] = system.core.project(func, e, side)
    return lam


def injected_shared_system(n, p, dom=1.0):
    """Builder restatement: the K=I, tau=1 system on an n x n mesh
    from ONE condensed block taken from an 8x8 mesh of the same spacing; Dirichlet
    columns zeroed as local.py:186-188 does.  Bit-identical to a full build (tests)."""
    h = dom / n
    small = Grid(8, 8, 0.0, 8 * h, 0.0, 8 * h)
    Sref = Local(ElementCore(small, p), 36, constant_spec(0.0, 1.0)).schur
    g = Grid(n, n, 0.0, dom, 0.0, dom)
    n1 = p + 1
    E = g.n_elems
    blocks = np.broadcast_to(Sref, (E, 4 * n1, 4 * n1)).copy()
    sys_ = OracleTrace(g, p, None, _blocks=blocks)
    blocks *= sys_.gmask[:, None, :]
    return sys_


# ----------------------------------------------------------------------- problem data


@dataclass(frozen=True)
class Spec:
    """problem.py:9-28 - coefficient, source, Dirichlet datum (vectorised), tau."""
    coefficient: object
    source: object
    dirichlet: object
    tau: float = 1.0


def constant_spec(value=0.0, kappa=1.0, tau=1.0):
    """problem.py:92-106."""
    return Spec(lambda x, y: np.full_like(np.asarray(x, float), kappa),
                lambda x, y: np.zeros_like(np.asarray(x, float)),
                lambda x, y: np.full_like(np.asarray(x, float), value), tau)


def nodal_source(f_nodal, n, p):
    """Builder restatement: source = sum_I f[e, I] phi_I on element e,
    e located by floor(x n), floor(y n) on the unit square; e = j n + i, I = a + b (p+1)."""
    basis = gll(p)
    f_nodal = np.asarray(f_nodal, float)

    def src(x, y):
        x = np.asarray(x, float)
        y = np.asarray(y, float)
        i = np.clip(np.floor(x * n).astype(np.int64), 0, n - 1)
        j = np.clip(np.floor(y * n).astype(np.int64), 0, n - 1)
        xi = 2.0 * (x * n - i) - 1.0
        eta = 2.0 * (y * n - j) - 1.0
        Ex = lagrange_at(basis, xi.ravel())
        Ey = lagrange_at(basis, eta.ravel())
        vals = f_nodal[(j * n + i).ravel()].reshape(-1, p + 1, p + 1)  # [q, b, a]
        return np.einsum("qb,qa,qba->q", Ey, Ex, vals).reshape(x.shape)

    return src


def piecewise_anisotropic(Kxx, Kyy):
    """Builder restatement: per-element diagonal K = diag(Kxx, Kyy) as a pair."""
    fx, fy = piecewise_coefficient(Kxx), piecewise_coefficient(Kyy)
    return lambda x, y: (fx(x, y), fy(x, y))


def piecewise_coefficient(Kgrid):
    """Builder restatement: K = Kg[floor(y ny), floor(x nx)] on [0,1]^2."""
    Kgrid = np.asarray(Kgrid, float)
    ny, nx = Kgrid.shape

    def coef(x, y):
        x = np.asarray(x, float)
        y = np.asarray(y, float)
        i = np.clip(np.floor(x * nx).astype(np.int64), 0, nx - 1)
        j = np.clip(np.floor(y * ny).astype(np.int64), 0, ny - 1)
        return Kgrid[j, i]

    return coef


# ---------------------------------------------------------------------------- transfers
# multigrid.py:215-298


def p_transfer(fine, coarse):
    """multigrid.py:215-219 - I_{n_blocks} (x) V, V = coarse basis at fine GLL nodes."""
    V = lagrange_at(coarse.core.ref.basis, fine.core.ref.basis.nodes)
    return sp.kron(sp.identity(fine.n_blocks, format="csr"), sp.csr_matrix(V)).tocsr()


def _tensor_eval(rule, xi, eta):
    """multigrid.py:222-226."""
    Ex = lagrange_at(rule, xi)
    Ey = lagrange_at(rule, eta)
    return np.einsum("nj,ni->nji", Ey, Ex).reshape(len(xi), -1)


def h_transfer(fine, coarse):
    """multigrid.py:229-298 - halves of coarse facets + reconstruction on cross facets."""
    gf, gc = fine.grid, coarse.grid
    if gc.children is None:
        raise ValueError("coarse mesh does not record its fine children")
    n1 = fine.n1
    nodes = fine.core.ref.basis.nodes
    halves = (lagrange_at(fine.core.ref.basis, (nodes - 1.0) / 2.0),
              lagrange_at(fine.core.ref.basis, (nodes + 1.0) / 2.0))
    R, C, Vv = [], [], []
    ar = np.arange(n1)

    def put(bf, bc, mat):
        rr, cc = np.meshgrid(bf * n1 + ar, bc * n1 + ar, indexing="ij")
        R.append(rr.ravel())
        C.append(cc.ravel())
        Vv.append(np.asarray(mat).ravel())

    for fc in coarse.interior:                                  # multigrid.py:256-267
        bc = coarse.block_of[fc]
        if gc.axis[fc] == 0:
            i, j = fc % gc.n_x, fc // gc.n_x
            k0 = 2 * j * gf.n_x + 2 * i
        else:
            k = fc - gc.n_h
            i, j = k // gc.n_y, k % gc.n_y
            k0 = gf.n_h + 2 * i * gf.n_y + 2 * j
        put(fine.block_of[k0], bc, halves[0])
        put(fine.block_of[k0 + 1], bc, halves[1])
    nb = coarse.core.nb
    for c in range(gc.n_elems):                                 # multigrid.py:271-293
        lc = coarse.locals[c]
        ucols = lu_solve(lc.lu, lc.trace_cols)[2 * nb:]
        x0, y0 = gc.origin(c)
        sw, se, nw, _ = gc.children[c]
        for f in (gf.e2f[sw, 1], gf.e2f[nw, 1], gf.e2f[sw, 2], gf.e2f[se, 2]):
            px, py = gf.facet_xy(f, nodes)
            xi = 2.0 * (px - x0) / gc.dx - 1.0
            eta = 2.0 * (py - y0) / gc.dy - 1.0
            tmap = -_tensor_eval(coarse.core.ref.basis, xi, eta) @ ucols
            sides = coarse.block_of[gc.e2f[c]]
            for s in range(4):
                if sides[s] >= 0:
                    put(fine.block_of[f], sides[s], tmap[:, s * n1:(s + 1) * n1])
    return sp.coo_matrix((np.concatenate(Vv), (np.concatenate(R), np.concatenate(C))),
                         shape=(fine.ndof, coarse.ndof)).tocsr()


# ---------------------------------------------------------------------------- smoothers


class BlockJacobiSmoother:
    """Builder restatement of the north-star edge block-Jacobi:
    D = per-facet n1 x n1 diagonal blocks of the level operator, x += w D^-1 (b - A x)."""

    def __init__(self, A, n1, omega=0.8):
        A = A.tocsr()
        nbk = A.shape[0] // n1
        D = np.empty((nbk, n1, n1))
        for b in range(nbk):
            D[b] = A[b * n1:(b + 1) * n1, b * n1:(b + 1) * n1].toarray()
        self.Dinv = np.linalg.inv(D) if nbk else D
        self.n1, self.omega = n1, omega
        self.complexity = nbk * n1 * n1 / max(A.nnz, 1)

    def apply_inverse(self, r):
        return np.einsum("bij,bj->bi", self.Dinv, r.reshape(-1, self.n1)).reshape(-1)

    def smooth(self, matvec, b, x, steps):
        for _ in range(steps):
            x = x + self.omega * self.apply_inverse(b - matvec(x))
        return x


class ChebyshevBlockJacobi(BlockJacobiSmoother):
    """Builder restatement: block-Jacobi steps with Chebyshev weights 1/theta_k on
    [0.15 lam, 1.05 lam], lam = lambda_max(D^-1 A) by 20 power steps from seed 1234 (the
    reference's FSAI weighting and estimate, multigrid.py:76-81, 162-173)."""

    def __init__(self, A, n1):
        super().__init__(A, n1, 1.0)
        A = A.tocsr()
        v = np.random.default_rng(1234).standard_normal(A.shape[0])
        lam = 1.0
        for _ in range(20):
            w = self.apply_inverse(A @ v)
            lam = np.linalg.norm(w)
            if lam == 0.0:
                lam = 1.0
                break
            v = w / lam
        self.lam_max, self.lo, self.hi = lam, 0.15 * lam, 1.05 * lam

    def sweep_weights(self, steps):
        k = np.arange(1, steps + 1)
        return 1.0 / (0.5 * (self.hi + self.lo) + 0.5 * (self.hi - self.lo) * np.cos(np.pi * (2 * k - 1) / (2 * steps)))

    def smooth(self, matvec, b, x, steps):
        for w in self.sweep_weights(steps):
            x = x + w * self.apply_inverse(b - matvec(x))
        return x


CHEB_LO, CHEB_LO_AGGR = 0.15, 0.30  # multigrid.py:43-44


class FSAI:
    """multigrid.py:47-88 and 123-173 (baseline pattern, aggressiveness 1 and 2)."""

    def __init__(self, A, power=1, omega=1.0, max_complexity=2.85):
        A = A.tocsr()
        n = A.shape[0]
        pat = sp.tril(A, format="csr") if power == 1 else _power_pattern(A, power, max_complexity)
        pat.sort_indices()
        rows = []
        for i in range(n):
            cols = pat.indices[pat.indptr[i]:pat.indptr[i + 1]]
            sub = A[cols][:, cols].toarray()
            e = np.zeros(cols.size)
            e[-1] = 1.0
            g = np.linalg.solve(sub, e)
            if g[-1] <= 0:
                raise RuntimeError(f"non-SPD principal submatrix in FSAI row {i}")
            rows.append((cols, g / math.sqrt(g[-1])))
        indptr = np.r_[0, np.cumsum([c.size for c, _ in rows])]
        idx = np.concatenate([c for c, _ in rows]) if rows else np.zeros(0, np.int64)
        dat = np.concatenate([g for _, g in rows]) if rows else np.zeros(0)
        self.G = sp.csr_matrix((dat, idx, indptr), shape=(n, n))
        self.Gt = self.G.T.tocsr()
        self.omega, self.aggressiveness = omega, power
        self.complexity = (2 * self.G.nnz - n) / A.nnz
        v = np.random.default_rng(1234).standard_normal(n)   # multigrid.py:162-173
        lam = 1.0
        for _ in range(20):
            w = self.Gt @ (self.G @ (A @ v))
            lam = np.linalg.norm(w)
            if lam == 0.0:
                lam = 1.0
                break
            v = w / lam
        self.lam_max = lam
        self.cheb_fraction = CHEB_LO if power == 1 else CHEB_LO_AGGR

    def apply_inverse(self, r):
        return self.Gt @ (self.G @ r)

    def sweep_weights(self, steps):
        lo, hi = self.cheb_fraction * self.lam_max, self.lam_max
        k = np.arange(1, steps + 1)
        return self.omega / (0.5 * (hi + lo) + 0.5 * (hi - lo) * np.cos(np.pi * (2 * k - 1) / (2 * steps)))

    def smooth(self, matvec, b, x, steps):
        if steps < 1:
            return x
        for w in self.sweep_weights(steps):
            x = x + w * self.apply_inverse(b - matvec(x))
        return x


def _power_pattern(A, power, max_complexity):
    """multigrid.py:91-120 - lower(|A|^power) filtered to the complexity budget."""
    absA = sp.csr_matrix((np.abs(A.data), A.indices, A.indptr), shape=A.shape)
    W = absA
    for _ in range(power - 1):
        W = (W @ absA).tocsr()
    low = sp.tril(W, format="coo")
    base = sp.tril(A, format="coo")
    budget = int((max_complexity * A.nnz + A.shape[0]) // 2)
    if low.nnz <= budget:
        return low.tocsr()
    keys = set(zip(base.row.tolist(), base.col.tolist()))
    inb = np.array([(i, j) in keys for i, j in zip(low.row.tolist(), low.col.tolist())], bool)
    extra = np.flatnonzero(~inb)
    room = max(budget - int(inb.sum()), 0)
    pick = extra[np.argsort(-low.data[extra], kind="stable")][:room]
    keep = np.concatenate([np.flatnonzero(inb), pick])
    return sp.coo_matrix((np.ones(keep.size), (low.row[keep], low.col[keep])), shape=A.shape).tocsr()


# ---------------------------------------------------------------------------- hierarchy


class Level:
    """multigrid.py:179-212 (fields used by the cycle)."""

    def __init__(self, system, kind):
        self.system, self.kind = system, kind
        self.p, self.grid = system.p, system.grid
        self.operator = None
        self.matrix_free = True
        self.rhs = None
        self.smoother = None
        self.prolong = None
        self._lu = None

    @property
    def ndof(self):
        return self.operator.shape[0]

    def matvec(self, x):
        return self.system.matvec(x) if self.matrix_free else self.operator @ x

    def coarse_solve(self, b):
        if self._lu is None:
            self._lu = spla.splu(self.operator.tocsc())
        return self._lu.solve(b)


def build_levels(grid, p, spec, tau_per_facet=None, coarse_cap=4096, smoother=None, omega=None):
    """multigrid.py:301-342 - p-levels p..1, then h-halving at p=1; Galerkin coarse operators.
    smoother: None | "blockjacobi" | "baseline" | "aggressive"."""
    if p < 1:
        raise ValueError("fine order must be >= 1")
    levels = []
    for q in range(p, 0, -1):
        levels.append(Level(OracleTrace(grid, q, spec, tau_per_facet), "p-level"))
        if len(levels) > 1:
            levels[-2].prolong = p_transfer(levels[-2].system, levels[-1].system)
    g = grid
    while g.n_x % 2 == 0 and g.n_y % 2 == 0 and g.n_x >= 4 and g.n_y >= 4:
        g = coarsen_grid(g)
        levels.append(Level(OracleTrace(g, 1, spec, tau_per_facet), "h-level"))
        levels[-2].prolong = h_transfer(levels[-2].system, levels[-1].system)
    levels[0].operator = levels[0].system.csr()
    levels[0].rhs = levels[0].system.rhs
    for k in range(1, len(levels)):
        P = levels[k - 1].prolong
        levels[k].operator = (P.T @ levels[k - 1].operator @ P).tocsr()
        levels[k].rhs = P.T @ levels[k - 1].rhs
        levels[k].matrix_free = False
    levels[-1].kind = "coarsest"
    if levels[-1].ndof > coarse_cap:
        raise ValueError(f"coarsest level has {levels[-1].ndof} unknowns, above cap {coarse_cap}")
    if smoother is not None:
        attach(levels, smoother, omega)
    return levels


def attach(levels, mode, omega=None):
    """multigrid.py:345-352; omega defaults: 0.8 block-Jacobi (north star), 1.0 FSAI."""
    for lev in levels[:-1]:
        if mode == "blockjacobi":
            lev.smoother = BlockJacobiSmoother(lev.operator, lev.p + 1, 0.8 if omega is None else omega)
        elif mode == "bj-chebyshev":
            lev.smoother = ChebyshevBlockJacobi(lev.operator, lev.p + 1)
        else:
            lev.smoother = FSAI(lev.operator, {"baseline": 1, "aggressive": 2}[mode],
                                1.0 if omega is None else omega)
    return levels


# ------------------------------------------------------------------------------- cycles
# multigrid.py:358-463


class Monitor:
    """multigrid.py:358-390."""

    def __init__(self, floor=1e-13):
        self.residuals, self.floor = [], floor

    def record(self, r):
        self.residuals.append(float(r))

    @property
    def rho(self):
        r = self.residuals
        return [r[i + 1] / r[i] if r[i] > 0 else 0.0 for i in range(len(r) - 1)]

    def asymptotic_rate(self, last=5):
        if len(self.residuals) < 2:
            return 0.0
        scale = self.residuals[0] or 1.0
        ok = [q for q, rn in zip(self.rho, self.residuals[1:]) if rn > self.floor * scale and q > 0.0]
        if not ok:
            ok = [q for q in self.rho if q > 0.0]
        tail = ok[-last:]
        return float(np.exp(np.mean(np.log(tail)))) if tail else 0.0

    def diverged(self, window=5):
        q = self.rho
        return len(q) >= window and all(v >= 1.0 for v in q[-window:])


def cycle(levels, k, b, x, nu1, nu2, visits):
    """multigrid.py:393-406."""
    lev = levels[k]
    if k == len(levels) - 1:
        return lev.coarse_solve(b)
    if lev.smoother is not None:
        x = lev.smoother.smooth(lev.matvec, b, x, nu1)
    rc = lev.prolong.T @ (b - lev.matvec(x))
    ec = np.zeros(levels[k + 1].ndof)
    for _ in range(visits):
        ec = cycle(levels, k + 1, rc, ec, nu1, nu2, visits)
    x = x + lev.prolong @ ec
    if lev.smoother is not None:
        x = lev.smoother.smooth(lev.matvec, b, x, nu2)
    return x


def v_cycle(levels, b, x0=None, nu1=2, nu2=2):
    x = np.zeros_like(b) if x0 is None else np.asarray(x0, float)
    return cycle(levels, 0, b, x, nu1, nu2, 1)


def solve_mg(levels, b=None, x0=None, cyc="v", nu1=2, nu2=2, tol=1e-12, max_cycles=50):
    """multigrid.py:421-439."""
    fine = levels[0]
    b = fine.rhs if b is None else b
    x = np.zeros_like(b) if x0 is None else np.asarray(x0, float).copy()
    visits = {"v": 1, "w": 2}[cyc]
    mon = Monitor()
    bn = np.linalg.norm(b) or 1.0
    mon.record(np.linalg.norm(b - fine.matvec(x)))
    for _ in range(max_cycles):
        if mon.residuals[-1] <= tol * bn:
            break
        x = cycle(levels, 0, b, x, nu1, nu2, visits)
        mon.record(np.linalg.norm(b - fine.matvec(x)))
        if mon.diverged():
            break
    return x, mon


def fmg(levels, nu1=2, nu2=2, cycles_per_level=1):
    """multigrid.py:442-454."""
    x = levels[-1].coarse_solve(levels[-1].rhs)
    for k in range(len(levels) - 2, -1, -1):
        x = levels[k].prolong @ x
        for _ in range(cycles_per_level):
            x = v_cycle(levels[k:], levels[k].rhs, x, nu1, nu2)
    return x


def mg_preconditioner(levels, nu1=2, nu2=2):
    """multigrid.py:457-463."""
    return lambda r: v_cycle(levels, r, None, nu1, nu2)


# --------------------------------------------------------------------------- configs


def config1_system(n=64, p=2, seed=0):
    """cfg1 inputs (BASELINE.json configs[0]): K=1, g_D=0, tau=1,
    f = default_rng(seed).uniform(-1, 1, (E, (p+1)^2)) nodal per element."""
    f = np.random.default_rng(seed).uniform(-1.0, 1.0, (n * n, (p + 1) ** 2))
    spec = Spec(lambda x, y: np.ones_like(np.asarray(x, float)), nodal_source(f, n, p),
                lambda x, y: np.zeros_like(np.asarray(x, float)), 1.0)
    return Grid(n, n), spec
