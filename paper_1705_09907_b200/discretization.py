"""Host-side setup math: reference element, batched static condensation, Galerkin blocks.

This is SETUP, not the hot path: it produces the condensed element blocks the CUDA
kernels stream (or hold in the constant bank), the transfer matrices, and the
condensed right-hand side.  It is written batched over *element classes*: elements
whose coefficient samples and stabilisation agree share one block (K = I gives a
single class per level), so setup cost scales with the number of
distinct elements, not the mesh size.

Reference algorithm restated (vectorised, batched):
  basis.py:42-181   GLL/GL rules, barycentric evaluation, tensor reference element
  local.py:133-237  local blocks, LU/condensation:  S = F L^-1 T + tau M_facet
  local.py:178-188  Dirichlet folding (loads) and column masking
  trace.py:67-79    condensed RHS as the two-owner facet sum
  multigrid.py:215-298, 328-334   transfers and Galerkin coarse operators, in element
                    form S_c = sum_children Q^T S Q (exact: SURVEY F4)
"""

from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as npleg
from scipy.special import roots_jacobi

NODE_SNAP_TOL = 1e-14  # basis.py:17
NORMALS = np.array([[0.0, -1.0], [1.0, 0.0], [0.0, 1.0], [-1.0, 0.0]])  # mesh.py:15


# ----------------------------------------------------------------------------- 1D rules


class Rule1D:
    __slots__ = ("order", "nodes", "weights", "bary")

    def __init__(self, order, nodes, weights):
        self.order = order
        self.nodes = np.asarray(nodes, float)
        self.weights = np.asarray(weights, float)
        d = self.nodes[:, None] - self.nodes[None, :]
        np.fill_diagonal(d, 1.0)
        w = 1.0 / d.prod(axis=1)
        w = w / np.abs(w).max()
        self.bary = -w if w[0] < 0 else w

    @property
    def n(self):
        return self.order + 1


def gll_rule(p):
    """basis.py:59-69."""
    if p < 1:
        raise ValueError("GLL basis needs order p >= 1 (at least two points)")
    x = np.empty(p + 1)
    x[0], x[-1] = -1.0, 1.0
    if p > 1:
        x[1:-1] = roots_jacobi(p - 1, 1.0, 1.0)[0]
    Pp = npleg.legval(x, np.eye(p + 1)[p])
    return Rule1D(p, x, 2.0 / (p * (p + 1) * Pp ** 2))


def gl_rule(p):
    """basis.py:72-77 (p+1 Gauss points)."""
    x, w = npleg.leggauss(p + 1)
    return Rule1D(p, x, w)


def eval_matrix(rule, points):
    """basis.py:91-105: V[q, j] = l_j(points[q]) (second barycentric form, node snapping)."""
    pts = np.atleast_1d(np.asarray(points, float))
    d = pts[:, None] - rule.nodes[None, :]
    hit = np.abs(d) < NODE_SNAP_TOL
    V = rule.bary[None, :] / np.where(hit, 1.0, d)
    snapped = hit.any(axis=1)
    V[snapped] = 0.0
    V[hit] = 1.0
    free = ~snapped
    V[free] /= V[free].sum(axis=1, keepdims=True)
    return V


def diff_matrix(rule):
    """basis.py:108-116."""
    x, w = rule.nodes, rule.bary
    d = x[:, None] - x[None, :]
    np.fill_diagonal(d, 1.0)
    D = (w[None, :] / w[:, None]) / d
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, -D.sum(axis=1))
    return D


class RefElement:
    """basis.py:119-181: GLL interpolation nodes, GL quadrature with p+1 points."""

    def __init__(self, p):
        self.p = p
        self.n1 = p + 1
        self.nb = (p + 1) ** 2
        self.basis = gll_rule(p)
        self.quad = gl_rule(p)
        self.interp_1d = eval_matrix(self.basis, self.quad.nodes)
        self.deriv_1d = self.interp_1d @ diff_matrix(self.basis)
        self.w2 = np.kron(self.quad.weights, self.quad.weights)
        self.interp_2d = np.kron(self.interp_1d, self.interp_1d)
        self.dxi_2d = np.kron(self.interp_1d, self.deriv_1d)
        self.deta_2d = np.kron(self.deriv_1d, self.interp_1d)
        k = np.arange(self.n1)
        # local.py:35-43 volume node ids per side along the tangent
        self.side_nodes = (k, p + k * self.n1, p * self.n1 + k, k * self.n1)
        self.mass1 = self.interp_1d.T @ (self.quad.weights[:, None] * self.interp_1d)

    def element_quad_points(self, x0, y0, dx, dy):
        """basis.py:157-162 for every element at once: x0, y0 arrays (E,) -> (E, nq^2)."""
        qx = np.asarray(x0)[:, None] + dx * (self.quad.nodes + 1.0) / 2.0
        qy = np.asarray(y0)[:, None] + dy * (self.quad.nodes + 1.0) / 2.0
        nq = self.quad.nodes.size
        return np.repeat(qx[:, None, :], nq, axis=1).reshape(len(qx), -1), \
            np.repeat(qy[:, :, None], nq, axis=2).reshape(len(qy), -1)


_REF_CACHE = {}


def ref_element(p):
    if p not in _REF_CACHE:
        _REF_CACHE[p] = RefElement(p)
    return _REF_CACHE[p]


# ------------------------------------------------------------------- batched condensation


class ElementClasses:
    """Distinct (coefficient samples, tau) rows -> condensed operators per class.

    Attributes (C = number of classes):
      S     (C, 4n1, 4n1)  condensed block with ALL sides unmasked
      Z     (C, 4n1, 3nb)  F L^-1, maps local loads to condensed loads
      T     (C, 3nb, 4n1)  trace columns (unmasked), for the Dirichlet fold of the loads
      ucols (C, nb, 4n1)   u response to trace data, (L^-1 T)[2nb:] (h-transfer, multigrid.py:273)
    """

    def __init__(self, p, dx, dy, kq, tau, kq_y=None):
        """kq: (C, nq^2) coefficient samples (isotropic, local.py:138); with kq_y the pair is
        the anisotropic diagonal K (Kxx, Kyy) - one flux mass per component."""
        ref = ref_element(p)
        self.p, self.ref = p, ref
        n1, nb = ref.n1, ref.nb
        kq = np.atleast_2d(np.asarray(kq, float))
        kqy = kq if kq_y is None else np.atleast_2d(np.asarray(kq_y, float))
        tau = np.atleast_2d(np.asarray(tau, float))
        if np.any(kq <= 0.0) or np.any(kqy <= 0.0):
            raise NumericalBreakdown("coefficient not positive")
        C = kq.shape[0]
        jac = dx * dy / 4.0
        wj = ref.w2 * jac
        I2 = ref.interp_2d
        Bx = 0.5 * dy * I2.T @ (ref.w2[:, None] * ref.dxi_2d)       # local.py:146
        By = 0.5 * dx * I2.T @ (ref.w2[:, None] * ref.deta_2d)      # local.py:147
        lens = (dx, dy, dx, dy)
        fm = [0.5 * lens[s] * ref.mass1 for s in range(4)]           # local.py:68-69
        M = np.einsum("qi,cq,qj->cij", I2, wj[None, :] / kq, I2)     # local.py:144
        My = M if kq_y is None else np.einsum("qi,cq,qj->cij", I2, wj[None, :] / kqy, I2)
        L = np.zeros((C, 3 * nb, 3 * nb))
        L[:, :nb, :nb] = M
        L[:, nb:2 * nb, nb:2 * nb] = My
        G = np.hstack([Bx, By])
        L[:, :2 * nb, 2 * nb:] = -G.T
        L[:, 2 * nb:, :2 * nb] = G
        T = np.zeros((C, 3 * nb, 4 * n1))
        F = np.zeros((C, 4 * n1, 3 * nb))
        Ms = np.zeros((C, 4 * n1, 4 * n1))
        for s in range(4):                                           # local.py:162-176
            idx = ref.side_nodes[s]
            cols = slice(s * n1, (s + 1) * n1)
            ts = tau[:, s][:, None, None]
            L[:, 2 * nb + idx[:, None], 2 * nb + idx[None, :]] += ts * fm[s]
            for d in range(2):
                ns = NORMALS[s, d]
                if ns != 0.0:
                    T[:, d * nb + idx, cols] += ns * fm[s]
                    F[:, cols, d * nb + idx] += ns * fm[s]
            T[:, 2 * nb + idx, cols] += -ts * fm[s]
            F[:, cols, 2 * nb + idx] += ts * fm[s]
            Ms[:, cols, cols] += ts * fm[s]
        X = np.linalg.solve(L, T)                                    # L^-1 T (local.py:233-234)
        self.L = L                                                   # for reconstruction (local.py:249)
        self.S = F @ X + Ms                                          # local.py:235
        self.Z = np.swapaxes(np.linalg.solve(np.swapaxes(L, 1, 2), np.swapaxes(F, 1, 2)), 1, 2)
        self.T = T
        self.ucols = X[:, 2 * nb:, :]
        self.n = C


class NumericalBreakdown(RuntimeError):
    """local.py:27."""


# ------------------------------------------------------------------ device kernel wrappers
# torch allocates and views; the arithmetic is the hand-written kernels of csrc/hdg_setup.cu.

def gemm_nt(A, B, out=None, rowscale=None, colscale=None, adiv=None, alpha=1.0, beta=0.0):
    """out = beta out + alpha diag(rowscale) ((A * colscale / adiv) B^T) on the device
    (hdgb200.h: hdg_gemm_nt).  A (E, J) and out (E, I) may be column slices of wider row-major
    tensors (unit column stride); B (I, J) contiguous."""
    import torch
    from . import _device as dev
    from ._lib import check, lib
    E, J = A.shape
    B = B.contiguous()
    I = B.shape[0]
    assert B.shape[1] == J and A.stride(1) == 1
    if out is None:
        out = torch.empty((E, I), dtype=torch.float64, device=A.device)
        beta = 0.0
    assert out.shape == (E, I) and out.stride(1) == 1
    if adiv is not None:
        assert adiv.shape == (E, J) and adiv.stride(1) == 1
    check(lib.hdg_gemm_nt(E, I, J, A.data_ptr(), A.stride(0) if E > 1 else J, B.data_ptr(), out.data_ptr(),
                          out.stride(0) if E > 1 else I, dev.ptr(rowscale), dev.ptr(colscale), dev.ptr(adiv),
                          0 if adiv is None else (adiv.stride(0) if E > 1 else J), float(alpha), float(beta),
                          dev.stream()))
    return out


def _status_check(status, what):
    if int(status.item()) != 0:
        raise NumericalBreakdown(f"{what}: non-positive pivot in an element's potential block")



class PiecewiseCondenser:
    """Batched condensation on the GPU for elements with an element-wise CONSTANT coefficient
    K_e and uniform tau (configs 3/5-style heterogeneous media).

    With flux mass M/K_e (local.py:144 when kq is constant on the element), eliminating the
    flux first gives an nb x nb SPD system per element instead of the 3nb x 3nb LU
    (local.py:208):  (Stab + K Lap) u = T_u - K G,   q = K M^-1 (T_q + B^T u), so
        S(K) = K A0 + Ms + (K C0 + F_u) (Stab + K Lap)^-1 (T_u - K G)
    with K-independent A0 = F_q M^-1 T_q, C0 = F_q M^-1 B^T, G = B M^-1 T_q,
    Lap = B M^-1 B^T.  Same operator as local.py:223-237 up to rounding (checked against the
    oracle in tests).  Returns S for all given K as a CUDA float64 tensor (E, 4n1, 4n1)."""

    def __init__(self, p, dx, dy, tau):
        ref = ref_element(p)
        n1, nb = ref.n1, ref.nb
        self.p, self.n1, self.nb = p, n1, nb
        wj = ref.w2 * (dx * dy / 4.0)
        I2 = ref.interp_2d
        M = I2.T @ (wj[:, None] * I2)
        Bx = 0.5 * dy * I2.T @ (ref.w2[:, None] * ref.dxi_2d)
        By = 0.5 * dx * I2.T @ (ref.w2[:, None] * ref.deta_2d)
        lens = (dx, dy, dx, dy)
        fm = [0.5 * lens[s] * ref.mass1 for s in range(4)]
        stab = np.zeros((nb, nb))
        Tq = np.zeros((2 * nb, 4 * n1))
        Tu = np.zeros((nb, 4 * n1))
        Fq = np.zeros((4 * n1, 2 * nb))
        Fu = np.zeros((4 * n1, nb))
        Ms = np.zeros((4 * n1, 4 * n1))
        for s in range(4):
            idx = ref.side_nodes[s]
            cols = slice(s * n1, (s + 1) * n1)
            stab[np.ix_(idx, idx)] += tau * fm[s]
            for d in range(2):
                ns = NORMALS[s, d]
                if ns != 0.0:
                    Tq[d * nb + idx, cols] += ns * fm[s]
                    Fq[cols, d * nb + idx] += ns * fm[s]
            Tu[idx, cols] += -tau * fm[s]
            Fu[cols, idx] += tau * fm[s]
            Ms[cols, cols] += tau * fm[s]
        Mi = np.linalg.inv(M)
        B = (Bx, By)
        # per flux component d (K_d multiplies each term: anisotropic diagonal K)
        self.Lapd = [B[d] @ Mi @ B[d].T for d in range(2)]
        self.Gd = [B[d] @ Mi @ Tq[d * nb:(d + 1) * nb] for d in range(2)]
        self.A0d = [Fq[:, d * nb:(d + 1) * nb] @ Mi @ Tq[d * nb:(d + 1) * nb] for d in range(2)]
        self.C0d = [Fq[:, d * nb:(d + 1) * nb] @ Mi @ B[d].T for d in range(2)]
        self.BMid = [B[d] @ Mi for d in range(2)]
        self.FqMid = [Fq[:, d * nb:(d + 1) * nb] @ Mi for d in range(2)]
        self.MiBt = [Mi @ B[d].T for d in range(2)]
        self.Mi, self.Tq = Mi, Tq
        self.stab, self.Tu, self.Fu, self.Ms = stab, Tu, Fu, Ms

    def _dev(self):
        import torch
        if not hasattr(self, "_t"):
            T = {}
            for k in ("stab", "Tu", "Fu", "Ms"):
                T[k] = torch.as_tensor(np.ascontiguousarray(getattr(self, k)), device="cuda")
            for k in ("Mi", "Tq"):
                T[k] = torch.as_tensor(np.ascontiguousarray(getattr(self, k)), device="cuda")
            for k in ("Lapd", "Gd", "A0d", "C0d", "BMid", "FqMid", "MiBt"):
                T[k] = [torch.as_tensor(np.ascontiguousarray(m), device="cuda") for m in getattr(self, k)]
            self._t = T
        return self._t

    @staticmethod
    def _pair(K):
        if isinstance(K, tuple):
            return np.asarray(K[0], float), np.asarray(K[1], float)
        K = np.asarray(K, float)
        return K, K

    def _kpair(self, K):
        import torch
        kx, ky = (torch.as_tensor(k, dtype=torch.float64, device="cuda").contiguous() for k in self._pair(K))
        return kx, ky

    def _usolve(self, kx, ky, rhs):
        """rhs_e <- (Stab + kx Lap_x + ky Lap_y)^-1 rhs_e in place (hdgb200.h: hdg_piecewise_usolve)."""
        import torch
        from . import _device as dev
        from ._lib import check, lib
        t = self._dev()
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        check(lib.hdg_piecewise_usolve(self.nb, kx.numel(), kx.data_ptr(), ky.data_ptr(), t["stab"].data_ptr(),
                                       t["Lapd"][0].data_ptr(), t["Lapd"][1].data_ptr(), rhs.data_ptr(),
                                       status.data_ptr(), dev.stream()))
        _status_check(status, "potential solve")
        return rhs

    def condensed_loads(self, K, load_q, load_u):
        return self.condensed_loads_device(K, load_q, load_u).cpu().numpy()

    def condensed_loads_device(self, K, load_q, load_u):
        """F L(K)^-1 [load_q; load_u] per element (local.py:236), the same elimination:
        u = H^-1 (f_u - sum_d K_d B_d M^-1 f_q,d), out = sum_d K_d (F_q,d M^-1 f_q,d + C_d u) + F_u u."""
        import torch
        t = self._dev()
        k = self._kpair(K)
        fq = torch.as_tensor(load_q, dtype=torch.float64, device="cuda").contiguous()
        rhs = torch.as_tensor(load_u, dtype=torch.float64, device="cuda").clone().contiguous()
        nb = self.nb
        f = (fq[:, :nb], fq[:, nb:])
        for d in range(2):
            gemm_nt(f[d], t["BMid"][d], out=rhs, rowscale=k[d], alpha=-1.0, beta=1.0)
        u = self._usolve(k[0], k[1], rhs)
        out = gemm_nt(u, t["Fu"])
        for d in range(2):
            gemm_nt(f[d], t["FqMid"][d], out=out, rowscale=k[d], beta=1.0)
            gemm_nt(u, t["C0d"][d], out=out, rowscale=k[d], beta=1.0)
        return out

    def reconstruct(self, K, load, lam_e):
        """(q, u) of every element from its trace values (local.py:240-251) by the same
        elimination: f = load - T lam_e, (Stab + sum_d K_d Lap_d) u = f_u - sum_d K_d B_d M^-1 f_q,d,
        q_d = K_d M^-1 (f_q,d + B_d^T u).  load (E, 3nb), lam_e (E, 4n1) CUDA tensors."""
        import torch
        t = self._dev()
        k = self._kpair(K)
        nb, E = self.nb, k[0].numel()
        f = load.clone()
        gemm_nt(lam_e, t["Tq"], out=f[:, :2 * nb], alpha=-1.0, beta=1.0)
        gemm_nt(lam_e, t["Tu"], out=f[:, 2 * nb:], alpha=-1.0, beta=1.0)
        fd = (f[:, :nb], f[:, nb:2 * nb])
        u = f[:, 2 * nb:].contiguous()
        for d in range(2):
            gemm_nt(fd[d], t["BMid"][d], out=u, rowscale=k[d], alpha=-1.0, beta=1.0)
        self._usolve(k[0], k[1], u)
        q = torch.empty((E, 2 * nb), dtype=torch.float64, device="cuda")
        for d in range(2):
            qd = q[:, d * nb:(d + 1) * nb]
            gemm_nt(fd[d], t["Mi"], out=qd, rowscale=k[d])
            gemm_nt(u, t["MiBt"][d], out=qd, rowscale=k[d], beta=1.0)
        return q, u

    def blocks(self, K):
        """S for every element; K: (E,) isotropic or a (Kxx, Kyy) pair of (E,) arrays.  One CTA per
        element eliminates [H | B] in shared memory (hdgb200.h: hdg_condense_piecewise; from p = 12
        the kernel keeps only H's upper triangle); orders whose packed matrix still exceeds shared
        memory (p > 12) use the batched library solve."""
        import torch
        from . import _device as dev
        from ._lib import check, lib
        t = self._dev()
        kx, ky = self._kpair(K)
        E, m, nb = kx.numel(), 4 * self.n1, self.nb
        out = torch.empty((E, m, m), dtype=torch.float64, device="cuda")
        if 8 * (nb * (nb + m) - nb * (nb - 1) // 2 + nb) > 227 * 1024:
            return self._blocks_library(kx, ky, out)
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        check(lib.hdg_condense_piecewise(nb, m, E, kx.data_ptr(), ky.data_ptr(), t["stab"].data_ptr(),
                                         t["Lapd"][0].data_ptr(), t["Lapd"][1].data_ptr(), t["Tu"].data_ptr(),
                                         t["Gd"][0].data_ptr(), t["Gd"][1].data_ptr(), t["A0d"][0].data_ptr(),
                                         t["A0d"][1].data_ptr(), t["Ms"].data_ptr(), out.data_ptr(),
                                         status.data_ptr(), dev.stream()))
        _status_check(status, "local condensation")
        return out

    def _blocks_library(self, kx, ky, out, chunk=1 << 13):
        import torch
        t = self._dev()
        for s0 in range(0, kx.numel(), chunk):
            k = (kx[s0:s0 + chunk][:, None, None], ky[s0:s0 + chunk][:, None, None])
            H = t["stab"] + sum(k[d] * t["Lapd"][d] for d in range(2))
            U = torch.linalg.solve(H, t["Tu"] - sum(k[d] * t["Gd"][d] for d in range(2)))
            out[s0:s0 + chunk] = sum(k[d] * t["A0d"][d] for d in range(2)) + t["Ms"] + \
                (sum(k[d] * t["C0d"][d] for d in range(2)) + t["Fu"]) @ U
        return out


class UnsupportedOrder(ValueError):
    """local.py:31."""


class PostprocessOps:
    """Shared data of the order-raising local Neumann solve p -> p+1 (local.py:254-279):
    order-p basis at the order-(p+1) GL points, stiffness, mean constraint, KKT matrix."""

    def __init__(self, p, dx, dy):
        if p < 1:
            raise UnsupportedOrder("postprocessing needs p >= 1")
        lo, ref = ref_element(p), ref_element(p + 1)
        self.p, self.ref, self.nb = p, ref, ref.nb
        cross = eval_matrix(lo.basis, ref.quad.nodes)
        self.interp_from_p = np.kron(cross, cross)
        self.w2 = ref.w2
        self.dxi2, self.deta2 = ref.dxi_2d, ref.deta_2d
        self.stiff = (dy / dx) * self.dxi2.T @ (self.w2[:, None] * self.dxi2) \
            + (dx / dy) * self.deta2.T @ (self.w2[:, None] * self.deta2)
        self.jac = dx * dy / 4.0
        self.mean_row = self.jac * (ref.interp_2d.T @ self.w2)
        n = self.nb
        self.kkt = np.zeros((n + 1, n + 1))
        self.kkt[:n, :n] = self.stiff
        self.kkt[:n, n] = self.mean_row
        self.kkt[n, :n] = self.mean_row


def classify_rows(rows):
    """Unique rows -> (unique_rows, inverse).  Fast path when every row is equal."""
    rows = np.ascontiguousarray(rows)
    if rows.shape[0] == 0:
        return rows, np.zeros(0, np.int64)
    if np.all(rows == rows[0]):
        return rows[:1], np.zeros(rows.shape[0], np.int64)
    uniq, inv = np.unique(rows, axis=0, return_inverse=True)
    return uniq, inv.reshape(-1)


# ----------------------------------------------------------------- transfers / Galerkin


def p_transfer_matrix(p_fine):
    """multigrid.py:217: coarse (p-1) GLL basis evaluated at the fine GLL nodes, n1f x n1c."""
    return eval_matrix(gll_rule(p_fine - 1), gll_rule(p_fine).nodes)


def galerkin_p(S, V):
    """S_c = Q^T S Q with Q = I_4 (x) V (the p-prolongation acts facet-locally).
    numpy in -> numpy out; CUDA tensor in -> CUDA tensor out (batched on the device)."""
    Q = np.kron(np.eye(4), V)
    if not isinstance(S, np.ndarray):
        import torch
        from . import _device as dev
        from ._lib import check, lib
        S = S.contiguous()
        n1, n1c = V.shape
        Vd = torch.as_tensor(np.ascontiguousarray(V, dtype=np.float64), device=S.device)
        out = torch.empty((S.shape[0], 4 * n1c, 4 * n1c), dtype=torch.float64, device=S.device)
        check(lib.hdg_galerkin_p(S.shape[0], n1, n1c, S.data_ptr(), Vd.data_ptr(), out.data_ptr(), dev.stream()))
        return out
    return np.einsum("ai,cij,jb->cab", Q.T, S, Q)


def h_halves():
    """multigrid.py:243 at p = 1: half[h][k][c] = l_c((t_k -+ 1)/2)."""
    b = gll_rule(1)
    return np.stack([eval_matrix(b, (b.nodes - 1.0) / 2.0), eval_matrix(b, (b.nodes + 1.0) / 2.0)])


def h_cross_maps(ucols):
    """multigrid.py:269-293: trace maps of the four cross facets of a coarse element,
    -V_f u_cols, in coarse reference coordinates.  ucols (C, nb=4, 8) -> (C, 4, 2, 8).
    Cross facet order: right of SW, right of NW, top of SW, top of SE."""
    b = gll_rule(1)
    t = b.nodes
    pts = [(np.zeros(2), (t - 1.0) / 2.0), (np.zeros(2), (t + 1.0) / 2.0),
           ((t - 1.0) / 2.0, np.zeros(2)), ((t + 1.0) / 2.0, np.zeros(2))]
    out = np.empty((ucols.shape[0], 4, 2, 8))
    for cf, (xi, eta) in enumerate(pts):
        Vf = np.einsum("nj,ni->nji", eval_matrix(b, eta), eval_matrix(b, xi)).reshape(2, 4)
        out[:, cf] = -np.einsum("nq,cqk->cnk", Vf, ucols)
    return out


def h_child_maps(halves, cross):
    """Q_k (C, 4 children, 8, 8): child k's (b, r, t, l) traces from the coarse element's
    8 trace dofs.  Children (SW, SE, NW, NE) as mesh.py:182-191."""
    C = cross.shape[0]
    Q = np.zeros((C, 4, 8, 8))

    def half(k, side_child, side_coarse, h):
        Q[:, k, 2 * side_child:2 * side_child + 2, 2 * side_coarse:2 * side_coarse + 2] = halves[h]

    def xf(k, side_child, cf):
        Q[:, k, 2 * side_child:2 * side_child + 2, :] = cross[:, cf]

    # SW
    half(0, 0, 0, 0); xf(0, 1, 0); xf(0, 2, 2); half(0, 3, 3, 0)
    # SE
    half(1, 0, 0, 1); half(1, 1, 1, 0); xf(1, 2, 3); xf(1, 3, 0)
    # NW
    xf(2, 0, 2); xf(2, 1, 1); half(2, 2, 2, 0); half(2, 3, 3, 1)
    # NE
    xf(3, 0, 3); half(3, 1, 1, 1); half(3, 2, 2, 1); xf(3, 3, 1)
    return Q


def galerkin_h(S_children, Q):
    """S_c = sum_k Q_k^T S_k Q_k.  S_children (C, 4, 8, 8), Q (C, 4, 8, 8)."""
    if not isinstance(S_children, np.ndarray):
        import torch
        from . import _device as dev
        from ._lib import check, lib
        Sc = S_children.contiguous()
        C = Sc.shape[0]
        Qt = torch.as_tensor(Q, dtype=torch.float64, device=Sc.device).contiguous()
        shared = int(Qt.shape[0] == 1 and C != 1)
        assert shared or Qt.shape[0] == C
        out = torch.empty((C, 8, 8), dtype=torch.float64, device=Sc.device)
        check(lib.hdg_galerkin_h(C, Sc.data_ptr(), Qt.data_ptr(), shared, out.data_ptr(), dev.stream()))
        return out
    return np.einsum("ckia,ckij,ckjb->cab", Q, S_children, Q)
