"""h/p geometric multigrid on the GPU (drop-in for hdgmg.multigrid, multigrid.py:1-463).

Same level schedule (p -> 1 on the fine mesh, then mesh halving at p = 1:
multigrid.py:301-342), Galerkin coarse operators and transposed-prolongation
restriction.  Every coarse Galerkin operator is applied by the same edge kernel
as the fine level: P^T A P is assembled in ELEMENT form, S_c = sum Q^T S Q
(exact; one block per level for K = I, F5).  The cycle itself
(multigrid.py:393-418) runs natively (hdg_mg_cycle) and is replayed from a CUDA
graph; only ||r|| crosses to the host, once per cycle (multigrid.py:431-436).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device as dev
from ._lib import check, lib
from .discretization import (ElementClasses, classify_rows, galerkin_h, galerkin_p, h_child_maps,
                             h_cross_maps, h_halves, p_transfer_matrix, ref_element)
from .fsai import FSAISmoother, NotSPDError, StructuredFSAI, fsai_build, structured_fsai_supported  # noqa: F401
from .mesh import coarsen
from .trace import BlockOperator, TraceLayout, TraceSystem


class HierarchyError(ValueError):
    """multigrid.py:30."""


# device-condensed levels above this size drop their element blocks after the hierarchy build
RELEASE_NDOF = 4_000_000
# Chebyshev block-Jacobi ("bj-chebyshev") interval on the spectrum of D^-1 A
CHEB_BJ_LOWER = 0.15
CHEB_BJ_SAFETY = 1.05


# ------------------------------------------------------------------------- operators


class DeviceOperator:
    """Stands where the reference keeps a scipy CSR level operator (multigrid.py:192):
    `.shape`, `A @ x` (device apply), `.tocsr()` for host inspection."""

    def __init__(self, block_op):
        self.block_op = block_op
        self.shape = (block_op.ndof, block_op.ndof)

    def __matmul__(self, x):
        return self.block_op.apply(x)

    def tocsr(self):
        return self.block_op.tocsr()

    @property
    def nnz(self):
        return self.tocsr().nnz

    def toarray(self):
        return self.tocsr().toarray()


class _Restriction:
    def __init__(self, P):
        self.P = P
        self.shape = (P.shape[1], P.shape[0])

    def __matmul__(self, r):
        return self.P.restrict(r)


class Prolongation:
    """Operator form of p_prolongation / h_prolongation (multigrid.py:215-298):
    `P @ e`, `P.T @ r` run the transfer kernels; `.tocsr()` assembles it on the host."""

    def __init__(self, fine_op, coarse_op, kind, V=None, halves=None, cross=None):
        self.fine_op, self.coarse_op, self.kind = fine_op, coarse_op, kind
        self.V, self.halves, self.cross = V, halves, cross
        self.shape = (fine_op.ndof, coarse_op.ndof)
        self._handle = None

    @property
    def handle(self):
        if self._handle is None:
            h = ctypes.c_void_p()
            if self.kind == "p":
                V = np.ascontiguousarray(self.V)
                check(lib.hdg_transfer_create_p(self.fine_op.handle, self.coarse_op.handle, V.ctypes.data,
                                                ctypes.byref(h)))
            else:
                hv = np.ascontiguousarray(self.halves)
                cr = np.ascontiguousarray(self.cross)
                check(lib.hdg_transfer_create_h(self.fine_op.handle, self.coarse_op.handle, hv.ctypes.data,
                                                cr.ctypes.data, cr.shape[0], ctypes.byref(h)))
            self._handle = h
        return self._handle

    def __del__(self):
        if self._handle is not None:
            try:
                lib.hdg_transfer_destroy(self._handle)
            except Exception:
                pass

    @property
    def T(self):
        return _Restriction(self)

    def __matmul__(self, e):
        ed, was_np = dev.to_device(e)
        x = dev.zeros(self.shape[0])
        check(lib.hdg_prolong_add(self.handle, dev.ptr(ed), dev.ptr(x), dev.stream()))
        return dev.back(x, was_np)

    def prolong_add(self, e, x):
        check(lib.hdg_prolong_add(self.handle, dev.ptr(e), dev.ptr(x), dev.stream()))

    def restrict(self, r):
        rd, was_np = dev.to_device(r)
        out = dev.empty(self.shape[1])
        check(lib.hdg_restrict(self.handle, dev.ptr(rd), dev.ptr(out), dev.stream()))
        return dev.back(out, was_np)

    def tocsr(self):
        """Host assembly by probing with unit vectors of the coarse space (small levels)."""
        import scipy.sparse as sp
        nc = self.shape[1]
        cols = []
        for c in range(nc):
            e = np.zeros(nc)
            e[c] = 1.0
            cols.append(sp.csr_matrix(np.asarray(self @ e)).T)
        return sp.hstack(cols).tocsr() if cols else sp.csr_matrix(self.shape)


# --------------------------------------------------------------------------- smoothers


class BlockJacobiSmoother:
    """Edge block-Jacobi (north star): x <- x + omega D^-1 (b - A x), D the
    per-facet n1 x n1 diagonal blocks of the level operator, Jacobi (double-buffered).
    Fills the duck-typed MGLevel.smoother slot (multigrid.py:397-405)."""

    def __init__(self, block_op, omega=0.8):
        self.block_op = block_op
        self.omega = float(omega)
        self.aggressiveness = 0
        self.lam_max = None
        block_op.set_blockjacobi(self.omega)
        self._complexity = None

    @property
    def complexity(self):
        """Stored smoother entries / nnz(A) (cf. multigrid.py:154-156): n_blocks n1^2 over the
        operator's nonzeros - counted on the assembled CSR for levels up to 1M dofs (the oracle's
        count), else the structural count of the 7-facet stencil (identical unless an element
        block holds exact zeros)."""
        if self._complexity is None:
            lay = self.block_op.layout
            n1 = lay.n1
            if lay.ndof <= 1_000_000:
                A = self.block_op.tocsr()
                A.eliminate_zeros()
                nnz = A.nnz
            else:
                nnz = structural_nnz(lay.nx, lay.ny, n1)
            self._complexity = lay.n_blocks * n1 * n1 / max(nnz, 1)
        return self._complexity

    def smooth(self, matvec, b, x, steps):
        """`matvec` is accepted for signature parity; the sweep applies this level's operator."""
        if steps < 1:
            return x
        bd, was_np = dev.to_device(b)
        xd = dev.to_device(x)[0].clone()
        work = dev.empty(xd.numel())
        check(lib.hdg_bj_sweeps(self.block_op.handle, dev.ptr(bd), dev.ptr(xd), dev.ptr(work), int(steps),
                                dev.stream()))
        return dev.back(xd, was_np)

    def sweep_weights(self, steps):
        if self.lam_max is None:
            return np.full(steps, self.omega)
        lo, hi = self.cheb_lo, self.cheb_hi
        k = np.arange(1, steps + 1)
        return 1.0 / (0.5 * (hi + lo) + 0.5 * (hi - lo) * np.cos(np.pi * (2 * k - 1) / (2 * steps)))

    def enable_chebyshev(self, frac=CHEB_BJ_LOWER, safety=CHEB_BJ_SAFETY, iters=20, seed=1234):
        """Chebyshev weights on [frac lam, safety lam], lam = lambda_max(D^-1 A) from a 20-step
        power iteration with seed 1234 (the reference FSAI estimate, multigrid.py:162-173)."""
        n = self.block_op.ndof
        v = dev.to_device(np.random.default_rng(seed).standard_normal(n))[0]
        lam = 1.0
        for _ in range(iters):
            w = self.apply_inverse(self.block_op.apply(v))
            lam = float(w.norm())
            if lam == 0.0:
                lam = 1.0
                break
            v = w / lam
        self.lam_max = lam
        self.cheb_lo, self.cheb_hi = frac * lam, safety * lam
        check(lib.hdg_level_set_bj_chebyshev(self.block_op.handle, self.cheb_lo, self.cheb_hi))
        return self

    def apply_inverse(self, r):
        """D^-1 r via one sweep from zero: omega D^-1 r, rescaled."""
        rd, was_np = dev.to_device(r)
        z = dev.zeros(rd.numel())
        out = dev.empty(rd.numel())
        check(lib.hdg_bj_sweep(self.block_op.handle, dev.ptr(rd), dev.ptr(z), dev.ptr(out), dev.stream()))
        return dev.back(out / self.omega, was_np)


def structural_nnz(nx, ny, n1):
    """Nonzeros of the condensed operator on an nx x ny mesh: every interior facet couples with
    itself and the interior facets of its two elements (at most 7 blocks, trace.py:98-128)."""
    nx, ny = int(nx), int(ny)
    if nx < 1 or ny < 1:
        return 0
    hj = np.arange(1, ny)                        # interior horizontal lines
    vi = np.arange(1, nx)                        # interior vertical lines
    hline = lambda j: ((j >= 1) & (j <= ny - 1)).astype(np.int64)
    vline = lambda i: ((i >= 1) & (i <= nx - 1)).astype(np.int64)
    i = np.arange(nx)
    # h(i, j): itself, h(i, j -+ 1), v(i | i+1, j-1), v(i | i+1, j)
    per_h = (1 + hline(hj - 1) + hline(hj + 1))[:, None] + 2 * (vline(i) + vline(i + 1))[None, :]
    j = np.arange(ny)
    # v(i, j): itself, v(i -+ 1, j), h(i-1 | i, j), h(i-1 | i, j+1)
    per_v = (1 + vline(vi - 1) + vline(vi + 1))[:, None] + 2 * (hline(j) + hline(j + 1))[None, :]
    return int(per_h.sum() + per_v.sum()) * n1 * n1


# ------------------------------------------------------------------------------ levels


class _LevelSystem:
    """What MGLevel.system offers on coarse levels: geometry + the level operator."""

    def __init__(self, mesh, p, block_op):
        self.mesh, self.p = mesh, p
        self.layout = block_op.layout
        self.operator = block_op
        self.ndof, self.n_blocks = block_op.ndof, block_op.layout.n_blocks
        self.ops = type("Ops", (), {"n1": p + 1, "nb": (p + 1) ** 2, "p": p, "ref": ref_element(p)})()

    @property
    def block_of(self):
        return self.layout.block_of

    def matvec_free(self, x):
        return self.operator.apply(x)


@dataclass
class MGLevel:
    """multigrid.py:179-212."""

    mesh: object
    p: int
    system: object = field(repr=False)
    kind: str = "fine"
    operator: object = field(default=None, repr=False)
    matrix_free: bool = True
    rhs: object = field(default=None, repr=False)
    smoother: object = field(default=None, repr=False)
    prolong: object = field(default=None, repr=False)
    _coarse_inv: object = field(default=None, repr=False)

    @property
    def ndof(self):
        return self.operator.shape[0]

    @property
    def block_op(self):
        return self.operator.block_op

    def matvec(self, x):
        return self.operator @ x

    def coarse_inverse(self):
        if self._coarse_inv is None:
            A = self.operator.tocsr().toarray()
            self._coarse_inv = np.ascontiguousarray(np.linalg.inv(A)) if A.size else np.zeros((0, 0))
        return self._coarse_inv

    def coarse_solve(self, b):
        """multigrid.py:209-212 on the device (dense inverse GEMV)."""
        mg = _native_mg([self])
        bd, was_np = dev.to_device(b)
        x = dev.empty(self.ndof)
        check(lib.hdg_coarse_solve(mg.handle, dev.ptr(bd), dev.ptr(x), dev.stream()))
        return dev.back(x, was_np)


def p_prolongation(fine_sys, coarse_sys):
    """multigrid.py:215-219 as a device operator."""
    return Prolongation(fine_sys.operator, coarse_sys.operator, "p", V=p_transfer_matrix(fine_sys.p))


def _coarse_classes(mesh_c, spec, tau_per_facet):
    """Sample K on the coarse p = 1 elements (the rediscretised system h_prolongation uses,
    multigrid.py:270-273) -> u_cols per coarse class."""
    ref = ref_element(1)
    nx, ny = mesh_c.n_x, mesh_c.n_y
    e = np.arange(nx * ny)
    x0 = mesh_c.x0 + (e % nx) * mesh_c.dx
    y0 = mesh_c.y0 + (e // nx) * mesh_c.dy
    qx, qy = ref.element_quad_points(x0, y0, mesh_c.dx, mesh_c.dy)
    kq = spec.coefficient(qx, qy)
    aniso = isinstance(kq, tuple)
    kx, ky = (kq if aniso else (kq, kq))
    kx = np.asarray(kx, float).reshape(len(e), -1)
    ky = np.asarray(ky, float).reshape(len(e), -1)
    if tau_per_facet is None:
        tau = np.full((len(e), 4), float(spec.tau))
    else:
        nh = nx * (ny + 1)
        j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        f = np.stack([j * nx + i, nh + (i + 1) * ny + j, (j + 1) * nx + i, nh + i * ny + j], -1).reshape(-1, 4)
        tau = np.asarray(tau_per_facet, float)[f]
    nq = kx.shape[1]
    rows, inv = classify_rows(np.hstack([kx, ky, tau]) if aniso else np.hstack([kx, tau]))
    nk = 2 * nq if aniso else nq
    cls = ElementClasses(1, mesh_c.dx, mesh_c.dy, rows[:, :nq], rows[:, nk:],
                         kq_y=rows[:, nq:nk] if aniso else None)
    return cls.ucols, inv


def _h_level(fine_op, mesh_c, spec, tau_per_facet):
    """Galerkin blocks of the h-coarsened level and the h-transfer maps."""
    ucols, ucls = _coarse_classes(mesh_c, spec, tau_per_facet)
    cross_u = h_cross_maps(ucols)                     # (Cu, 4, 2, 8)
    halves = h_halves()
    nxf = fine_op.mesh.n_x
    ncx, ncy = mesh_c.n_x, mesh_c.n_y
    cj, ci = np.meshgrid(np.arange(ncy), np.arange(ncx), indexing="ij")
    base = (2 * cj * nxf + 2 * ci).ravel()
    kids = np.stack([base, base + 1, base + nxf, base + nxf + 1], axis=1)
    kid_cls = fine_op.elem_class[kids]                # (Ec, 4)
    rows, inv = classify_rows(np.hstack([ucls[:, None], kid_cls]))
    Q = h_child_maps(halves, cross_u[rows[:, 0]])
    if isinstance(fine_op.S_cls, np.ndarray):
        S_children = fine_op.S_cls[rows[:, 1:]]       # (C, 4, 8, 8)
    else:
        import torch
        S_children = fine_op.S_cls[torch.as_tensor(rows[:, 1:], device=fine_op.S_cls.device)]
    S_c = galerkin_h(S_children, Q)
    cross = cross_u if cross_u.shape[0] == 1 else cross_u[ucls]
    return S_c, inv, halves, cross


def h_prolongation(fine_sys, coarse_sys, spec=None, tau_per_facet=None):
    """multigrid.py:229-298 as a device operator (coarse K sampled from `spec`)."""
    if getattr(coarse_sys.mesh, "child_elements", None) is None:
        raise HierarchyError("coarse mesh does not record its fine children")
    spec = spec or coarse_sys.spec
    _, _, halves, cross = _h_level(fine_sys.operator, coarse_sys.mesh, spec, tau_per_facet)
    return Prolongation(fine_sys.operator, coarse_sys.operator, "h", halves=halves, cross=cross)


def build_hierarchy(mesh, p, spec, tau_per_facet=None, coarse_cap=4096, smoother="baseline", omega=None,
                    threads=1):
    """multigrid.py:301-342: orders p..1 on the fine mesh, then halving at p = 1, Galerkin
    operators, P^T-cascaded right-hand sides.  smoother: "baseline" | "aggressive" (FSAI, the
    reference default, omega 1.0) | "blockjacobi" (north star, omega 0.8) | None."""
    if p < 1:
        raise HierarchyError("fine order must be >= 1")
    fine = TraceSystem(mesh, p, spec, tau_per_facet, threads=threads)
    levels = [MGLevel(mesh, p, fine, kind="p-level", operator=DeviceOperator(fine.operator),
                      matrix_free=True, rhs=fine.rhs)]
    op = fine.operator

    # The baseline FSAI (the reference default) is set up on the device from each level's element
    # blocks as soon as the level exists (StructuredFSAI), so large levels can then drop their
    # blocks; the aggressive FSAI builds from host CSR and keeps them.
    struct_fsai = smoother == "baseline"
    keep_blocks = smoother is not None and smoother not in _BJ_MODES and not struct_fsai
    w_fsai = 1.0 if omega is None else float(omega)
    early = {}

    def retire(prev, lev):
        if struct_fsai and structured_fsai_supported(prev):
            early[id(lev)] = StructuredFSAI(prev, w_fsai)
        # large device-condensed levels: keep only the native facet stream (memory)
        if not keep_blocks and not isinstance(prev.S_cls, np.ndarray) and prev.ndof > RELEASE_NDOF:
            prev.release_blocks()

    _extend_levels(levels, op, mesh, p, spec, tau_per_facet, retire)
    levels[-1].kind = "coarsest"
    if levels[-1].ndof > coarse_cap:                                  # :336-339
        raise HierarchyError(f"coarsest level has {levels[-1].ndof} unknowns, above cap {coarse_cap}")
    for k in range(1, len(levels)):                                   # :333 rhs_k = P^T rhs_{k-1}
        prev = levels[k - 1]
        levels[k].rhs = _LazyRhs(prev, k) if prev.rhs is not None else None
    if smoother is not None:
        attach_smoothers(levels, smoother, omega, prebuilt=early)
    return levels


def _extend_levels(levels, op, mesh, p, spec, tau_per_facet, retire=None):
    """Append the coarse levels below (mesh, p, op): orders p-1..1 on the same mesh, then mesh
    halving at p = 1 (multigrid.py:317-327), Galerkin operators in element form."""
    retire = retire or (lambda prev, lev: None)
    for q in range(p - 1, 0, -1):                                   # multigrid.py:317-321
        V = p_transfer_matrix(q + 1)
        cop = BlockOperator(mesh, q, galerkin_p(op.S_cls, V), op.elem_class)
        levels[-1].prolong = Prolongation(op, cop, "p", V=V)
        levels.append(MGLevel(mesh, q, _LevelSystem(mesh, q, cop), kind="p-level",
                              operator=DeviceOperator(cop), matrix_free=False))
        retire(op, levels[-2])
        op = cop
    m = mesh
    while m.n_x % 2 == 0 and m.n_y % 2 == 0 and m.n_x >= 4 and m.n_y >= 4:   # :322-327
        m = coarsen(m)
        S_c, inv, halves, cross = _h_level(op, m, spec, tau_per_facet)
        cop = BlockOperator(m, 1, S_c, inv)
        levels[-1].prolong = Prolongation(op, cop, "h", halves=halves, cross=cross)
        levels.append(MGLevel(m, 1, _LevelSystem(m, 1, cop), kind="h-level",
                              operator=DeviceOperator(cop), matrix_free=False))
        retire(op, levels[-2])
        op = cop
    return levels


def level_schedule(nx, ny, p):
    """(nx, ny, p) of every level build_hierarchy makes (multigrid.py:317-327), fine first."""
    out = [(nx, ny, q) for q in range(p, 0, -1)]
    while nx % 2 == 0 and ny % 2 == 0 and nx >= 4 and ny >= 4:
        nx, ny = nx // 2, ny // 2
        out.append((nx, ny, 1))
    return out


def hierarchy_from_operator(mesh, p, op, spec, tau_per_facet=None, coarse_cap=4096, smoother="blockjacobi",
                            omega=None):
    """The hierarchy below an already-built level operator `op` on (mesh, p): the replicated coarse
    tail of a strip-partitioned hierarchy starts from an agglomerated level (distributed.py)."""
    levels = [MGLevel(mesh, p, _LevelSystem(mesh, p, op), kind="p-level" if p > 1 else "h-level",
                      operator=DeviceOperator(op), matrix_free=False)]
    _extend_levels(levels, op, mesh, p, spec, tau_per_facet)
    levels[-1].kind = "coarsest"
    if levels[-1].ndof > coarse_cap:
        raise HierarchyError(f"coarsest level has {levels[-1].ndof} unknowns, above cap {coarse_cap}")
    if smoother is not None and len(levels) > 1:
        attach_smoothers(levels, smoother, omega)
    return levels


class _LazyRhs:
    """rhs_k = P^T rhs_{k-1} (multigrid.py:333), evaluated on first use on the device."""

    def __init__(self, prev, k):
        self.prev, self.k, self.val = prev, k, None

    def resolve(self):
        if self.val is None:
            r = self.prev.rhs.resolve() if isinstance(self.prev.rhs, _LazyRhs) else self.prev.rhs
            self.val = self.prev.prolong.T @ np.asarray(r)
        return self.val


def _rhs(level):
    return level.rhs.resolve() if isinstance(level.rhs, _LazyRhs) else level.rhs


_BJ_MODES = ("blockjacobi", "bj", "bj-chebyshev", "chebyshev")


def attach_smoothers(levels, mode, omega=None, prebuilt=None):
    """multigrid.py:345-352 on every level but the coarsest.  mode: "baseline" (FSAI on the
    pattern of A), "aggressive" (pattern of A^2), an int power, or "blockjacobi".  omega
    defaults: FSAI 1.0 (reference), block-Jacobi 0.8 (north star)."""
    if mode in ("blockjacobi", "bj"):
        w = 0.8 if omega is None else float(omega)
        for lev in levels[:-1]:
            lev.smoother = BlockJacobiSmoother(lev.block_op, w)
        return levels
    if mode in ("bj-chebyshev", "chebyshev"):
        for lev in levels[:-1]:
            lev.smoother = BlockJacobiSmoother(lev.block_op, 1.0).enable_chebyshev()
        return levels
    power = {"baseline": 1, "aggressive": 2}.get(mode, mode)
    if not isinstance(power, int) or isinstance(power, bool) or power < 1:
        raise ValueError(f"unknown smoother mode {mode!r}")
    w = 1.0 if omega is None else float(omega)
    prebuilt = prebuilt or {}
    for lev in levels[:-1]:
        if id(lev) not in prebuilt and getattr(lev.block_op, "S_cls", True) is None:
            raise HierarchyError("FSAI needs the level's element blocks, released after building a large "
                                 "device-condensed hierarchy: pass smoother=%r to build_hierarchy" % (mode,))
    for lev in levels[:-1]:
        if id(lev) in prebuilt and prebuilt[id(lev)].omega == w:
            lev.smoother = prebuilt[id(lev)]
        elif structured_fsai_supported(lev.block_op, power):
            lev.smoother = StructuredFSAI(lev.block_op, w)       # device setup (baseline pattern)
        else:
            lev.smoother = fsai_build(lev.operator.tocsr(), power, w).bind(lev.block_op)
    return levels


# ------------------------------------------------------------------------------ cycles


class ConvergenceMonitor:
    """multigrid.py:358-390."""

    def __init__(self, floor=1e-13):
        self.residuals = []
        self.floor = floor

    def record(self, rnorm):
        self.residuals.append(float(rnorm))

    @property
    def rho(self):
        r = self.residuals
        return [r[i + 1] / r[i] if r[i] > 0 else 0.0 for i in range(len(r) - 1)]

    def asymptotic_rate(self, last=5):
        if len(self.residuals) < 2:
            return 0.0
        scale = self.residuals[0] or 1.0
        valid = [rho for rho, rn in zip(self.rho, self.residuals[1:]) if rn > self.floor * scale and rho > 0.0]
        if not valid:
            valid = [rho for rho in self.rho if rho > 0.0]
        tail = valid[-last:]
        return float(np.exp(np.mean(np.log(tail)))) if tail else 0.0

    def diverged(self, window=5):
        rho = self.rho
        return len(rho) >= window and all(r >= 1.0 for r in rho[-window:])


class _NativeMG:
    def __init__(self, levels):
        n = len(levels)
        hs = (ctypes.c_void_p * n)(*[lev.block_op.handle.value for lev in levels])
        ts = (ctypes.c_void_p * max(n - 1, 1))(*[levels[k].prolong.handle.value for k in range(n - 1)])
        h = ctypes.c_void_p()
        check(lib.hdg_mg_create(hs, ts, n, ctypes.byref(h)))
        self.handle = h
        self.levels = levels
        inv = levels[-1].coarse_inverse()
        check(lib.hdg_mg_set_coarse_inverse(h, inv.ctypes.data if inv.size else None, inv.shape[0]))

    def __del__(self):
        try:
            lib.hdg_mg_destroy(self.handle)
        except Exception:
            pass


def set_fused_tail(levels, enable=True):
    """Run the small trailing p = 1 levels of the device cycle as one cooperative kernel
    (default) or as separate launches (hdgb200.h: hdg_mg_set_fused_tail)."""
    check(lib.hdg_mg_set_fused_tail(_native_mg(levels).handle, int(bool(enable))))


def set_records(levels, mode=1):
    """Facet-record cycle on the constant-coefficient p-ladder of the finest mesh (hdgb200.h:
    hdg_mg_set_records): 0 off, 1 automatic, 2 whenever the levels qualify, 3 as 2 with the
    p-prolongation as a separate kernel, 4 as 2 with every qualifying h-coarsened level on records too."""
    check(lib.hdg_mg_set_records(_native_mg(levels).handle, int(mode)))


def record_levels(levels):
    """Number of leading levels the last device cycle ran on facet records (0: reference layout)."""
    return int(lib.hdg_mg_record_levels(_native_mg(levels).handle))


def _native_mg(levels):
    """The native level stack of `levels` (a hierarchy or a suffix / slice of one).  It is cached
    on the hierarchy's first level, so it lives exactly as long as the levels do: dropping the
    hierarchy frees its device workspaces and CUDA graphs (cyclic garbage, collected by gc)."""
    first = levels[0]
    cache = first.__dict__.setdefault("_native_cache", {})
    key = tuple(id(lev) for lev in levels)
    mg = cache.get(key)
    if mg is None or any(a is not b for a, b in zip(mg.levels, levels)):
        for lev in levels[:-1]:
            if not isinstance(lev.smoother, (BlockJacobiSmoother, FSAISmoother)):
                raise NotImplementedError("the device cycle needs a block-Jacobi or FSAI smoother on every level")
        mg = _NativeMG(list(levels))
        cache[key] = mg
    return mg


def release_native(levels):
    """Free the native cycle state (workspaces, graphs) cached on `levels` now, instead of at
    garbage collection."""
    for lev in levels:
        lev.__dict__.pop("_native_cache", None)


def _run_cycle(levels, b, x0, nu1, nu2, visits, use_graph=True):
    mg = _native_mg(levels)
    bd, was_np = dev.to_device(b)
    x = dev.empty(bd.numel())
    x0d = None if x0 is None else dev.to_device(x0)[0]
    check(lib.hdg_mg_cycle(mg.handle, dev.ptr(bd), dev.ptr(x0d), dev.ptr(x), int(nu1), int(nu2), int(visits),
                           int(use_graph), dev.stream()))
    return dev.back(x, was_np)


def v_cycle(levels, b, x0=None, nu1=2, nu2=2):
    """multigrid.py:409-412 (x0 is not mutated)."""
    return _run_cycle(levels, b, x0, nu1, nu2, 1)


def cycle_records(levels, b, x0=None, nu1=2, nu2=2, visits=1, out=None):
    """One cycle (multigrid.py:393-406) on vectors held as facet records of the fine level
    (TraceSystem.facet_planes): FacetPlanes in, FacetPlanes out, no layout change at the boundary
    (hdgb200.h: hdg_mg_cycle_records).  The hierarchy needs record levels (set_records)."""
    from .trace import FacetPlanes
    mg = _native_mg(levels)
    x = dev.empty(b.data.numel()) if out is None else out.data
    check(lib.hdg_mg_cycle_records(mg.handle, dev.ptr(b.data), dev.ptr(None if x0 is None else x0.data), dev.ptr(x),
                                   int(nu1), int(nu2), int(visits), 1, dev.stream()))
    return FacetPlanes(b.system, x) if out is None else out


def w_cycle(levels, b, x0=None, nu1=2, nu2=2):
    """multigrid.py:415-418."""
    return _run_cycle(levels, b, x0, nu1, nu2, 2)


def solve_mg(levels, b=None, x0=None, cycle="v", nu1=2, nu2=2, tol=1e-12, max_cycles=50):
    """multigrid.py:421-439: cycles until ||b - A x|| <= tol ||b||, all vectors on the device."""
    fine = levels[0]
    if b is None:
        b = _rhs(fine)
    bd, was_np = dev.to_device(b)
    n = bd.numel()
    x = dev.zeros(n) if x0 is None else dev.to_device(x0)[0].clone()
    visits = {"v": 1, "w": 2}[cycle]
    mg = _native_mg(levels)
    mon = ConvergenceMonitor()
    hist = np.zeros(max(int(max_cycles), 0) + 1)
    ncyc = ctypes.c_int(0)
    # the whole loop (stop test, cycles, monitor residuals, divergence) runs natively: hdg_solve_mg
    check(lib.hdg_solve_mg(mg.handle, dev.ptr(bd), dev.ptr(x), int(nu1), int(nu2), visits, float(tol),
                           int(max_cycles), hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                           ctypes.byref(ncyc), dev.stream()))
    for v in hist[:ncyc.value + 1] if n else [0.0]:
        mon.record(v)
    return dev.back(x, was_np), mon


def fmg(levels, nu1=2, nu2=2, cycles_per_level=1):
    """multigrid.py:442-454."""
    x = levels[-1].coarse_solve(_rhs(levels[-1]))
    for k in range(len(levels) - 2, -1, -1):
        x = levels[k].prolong @ x
        for _ in range(cycles_per_level):
            x = v_cycle(levels[k:], _rhs(levels[k]), x, nu1, nu2)
    return x


class MGPreconditioner:
    """multigrid.py:457-463: one V-cycle from zero (device in, device out).  Callable like the
    reference's closure; TraceSystem.solve_cg recognises it and runs the whole preconditioned
    CG natively (hdg_pcg)."""

    def __init__(self, levels, nu1=2, nu2=2):
        self.levels, self.nu1, self.nu2 = levels, nu1, nu2

    def __call__(self, r):
        return v_cycle(self.levels, r, None, self.nu1, self.nu2)

    def native(self):
        return _native_mg(self.levels)


def mg_preconditioner(levels, nu1=2, nu2=2):
    """multigrid.py:457-463."""
    return MGPreconditioner(levels, nu1, nu2)
