"""Global trace system on the GPU (drop-in for hdgmg.trace, trace.py:26-233).

`TraceSystem(mesh, p, spec)` keeps the reference constructor and attributes;
`matvec_free` runs the edge-centric sm_100a kernel through the C ABI
(include/hdgb200.h: hdg_matvec).  Element blocks are condensed on the host per
element *class* (discretization.ElementClasses) and handed to the library once:
one shared block (constant K and tau) or a stored per-element stack.
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp

from . import _device as dev
from ._lib import check, lib
from .discretization import (ElementClasses, NumericalBreakdown, PiecewiseCondenser, PostprocessOps,  # noqa: F401
                             UnsupportedOrder, classify_rows, ref_element)


class LocalOps:
    """The slice of local.py:46-78 that callers read (n1, nb, ref, p)."""

    def __init__(self, mesh, p):
        self.mesh, self.p = mesh, p
        self.ref = ref_element(p)
        self.n1, self.nb = p + 1, (p + 1) ** 2


class TraceLayout:
    """Facet numbering and ownership for a structured mesh (trace.py:36-65, mesh.py:112-154)."""

    def __init__(self, mesh, p):
        self.mesh, self.p = mesh, p
        self.nx, self.ny = mesh.n_x, mesh.n_y
        self.n1 = p + 1
        self.nh = self.nx * (self.ny - 1)
        self.n_blocks = self.nh + (self.nx - 1) * self.ny
        self.ndof = self.n1 * self.n_blocks

    @property
    def interior(self):
        nx, ny = self.nx, self.ny
        nh_all = nx * (ny + 1)
        h = (np.arange(1, ny)[:, None] * nx + np.arange(nx)[None, :]).ravel()
        v = (nh_all + np.arange(1, nx)[:, None] * ny + np.arange(ny)[None, :]).ravel()
        return np.concatenate([h, v]).astype(np.int64)

    @property
    def block_of(self):
        nx, ny = self.nx, self.ny
        out = np.full(nx * (ny + 1) + ny * (nx + 1), -1, np.int64)
        out[self.interior] = np.arange(self.n_blocks)
        return out

    def side_mask(self):
        """(E, 4) True where the element side is an interior facet (trace.py:58-59)."""
        nx, ny = self.nx, self.ny
        j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        return np.stack([j > 0, i < nx - 1, j < ny - 1, i > 0], axis=-1).reshape(-1, 4)

    def sum_owners(self, per_elem):
        """trace.py:73-79: facet block = slot-0 owner + slot-1 owner, vectorised."""
        n1, nx, ny = self.n1, self.nx, self.ny
        y = np.asarray(per_elem).reshape(ny, nx, 4, n1)
        h = y[:-1, :, 2] + y[1:, :, 0]                     # (ny-1, nx): below TOP + above BOTTOM
        v = y[:, :-1, 1] + y[:, 1:, 3]                     # (ny, nx-1): left RIGHT + right LEFT
        return np.concatenate([h.reshape(-1), np.swapaxes(v, 0, 1).reshape(-1)])

    def gather(self, x):
        """trace.py:81-92: (E, 4 n1) element traces, zero on Dirichlet sides."""
        n1, nx, ny = self.n1, self.nx, self.ny
        x = np.asarray(x, float)
        H = np.zeros((ny + 1, nx, n1))
        H[1:ny] = x[:self.nh * n1].reshape(ny - 1, nx, n1)
        V = np.zeros((nx + 1, ny, n1))
        V[1:nx] = x[self.nh * n1:].reshape(nx - 1, ny, n1)
        b = H[:-1]
        t = H[1:]
        l = np.swapaxes(V[:-1], 0, 1)
        r = np.swapaxes(V[1:], 0, 1)
        return np.stack([b, r, t, l], axis=2).reshape(nx * ny, 4 * n1)


class BlockOperator:
    """A trace operator given by element classes: blocks S_cls (C, 4n1, 4n1) with every
    side unmasked and the class of each element.  Owns the native hdg_level."""

    def __init__(self, mesh, p, S_cls, elem_class):
        self.layout = TraceLayout(mesh, p)
        self.mesh, self.p = mesh, p
        # host numpy (few classes) or a CUDA tensor (GPU-condensed heterogeneous media)
        self.S_cls = S_cls if not isinstance(S_cls, np.ndarray) and hasattr(S_cls, "is_cuda") \
            else np.ascontiguousarray(S_cls, dtype=np.float64)
        self.elem_class = np.asarray(elem_class, np.int64)
        self._handle = None
        self._bj_omega = None

    @property
    def ndof(self):
        return self.layout.ndof

    @property
    def shared(self):
        return self.S_cls.shape[0] == 1

    @property
    def handle(self):
        if self._handle is None:
            dev.require_cuda()
            h = ctypes.c_void_p()
            nx, ny = self.mesh.n_x, self.mesh.n_y
            if self.shared:
                blk = np.ascontiguousarray(self.S_cls[0])
                check(lib.hdg_level_create_shared(nx, ny, self.p, blk.ctypes.data, ctypes.byref(h)))
            else:
                import torch
                S = self.S_cls if isinstance(self.S_cls, torch.Tensor) else torch.from_numpy(self.S_cls).cuda()
                E = self.elem_class.size
                if S.shape[0] == E and np.array_equal(self.elem_class, np.arange(E)):
                    blocks = S.contiguous()          # identity classes: no gather copy
                else:
                    blocks = S.index_select(0, torch.from_numpy(self.elem_class).cuda()).contiguous()
                check(lib.hdg_level_create_stored(nx, ny, self.p, blocks.data_ptr(), ctypes.byref(h)))
                del blocks, S
            self._handle = h
        return self._handle

    def set_blockjacobi(self, omega):
        check(lib.hdg_level_set_blockjacobi(self.handle, float(omega)))
        self._bj_omega = float(omega)

    def operator_bytes(self):
        return int(lib.hdg_level_operator_bytes(self.handle))

    def __del__(self):
        if self._handle is not None:
            try:
                lib.hdg_level_destroy(self._handle)
            except Exception:
                pass

    # -- device applies ----------------------------------------------------------------
    def apply(self, x):
        xd, was_np = dev.to_device(x)
        if xd.numel() != self.ndof:
            raise ValueError(f"expected {self.ndof} trace values, got {xd.numel()}")
        y = dev.empty(self.ndof)
        if self.ndof:
            check(lib.hdg_matvec(self.handle, dev.ptr(xd), dev.ptr(y), dev.stream()))
        return dev.back(y, was_np)

    # -- facet-plane device layout (shared-block levels; hdg_soa.cuh) ------------------------
    def planes_length(self):
        n = ctypes.c_int64()
        check(lib.hdg_soa_length(self.handle, ctypes.byref(n)))
        return int(n.value)

    def to_planes(self, x, out=None):
        xd, _ = dev.to_device(x)
        if xd.numel() != self.ndof:
            raise ValueError(f"expected {self.ndof} trace values, got {xd.numel()}")
        xs = dev.empty(self.planes_length()) if out is None else out
        check(lib.hdg_soa_pack(self.handle, dev.ptr(xd), dev.ptr(xs), dev.stream()))
        return xs

    def from_planes(self, xs, out=None):
        y = dev.empty(self.ndof) if out is None else out
        check(lib.hdg_soa_unpack(self.handle, dev.ptr(xs), dev.ptr(y), dev.stream()))
        return y

    def apply_planes(self, xs, out=None):
        ys = dev.empty(self.planes_length()) if out is None else out
        check(lib.hdg_matvec_soa(self.handle, dev.ptr(xs), dev.ptr(ys), dev.stream()))
        return ys

    def residual_norm(self, b, x):
        """||b - A x|| on the device; one scalar crosses to the host."""
        out = dev.empty(1)
        check(lib.hdg_residual(self.handle, dev.ptr(b), dev.ptr(x), None, dev.ptr(out), dev.stream()))
        return float(out.item()) ** 0.5

    # -- host views (tests, tooling, coarse inverse) -------------------------------------
    def release_blocks(self):
        """Drop the element-class blocks once the native level holds its facet stream and the
        next coarser level has been formed (large heterogeneous hierarchies)."""
        _ = self.handle
        self.S_cls = None
        import torch
        torch.cuda.empty_cache()   # the native library allocates with cudaMalloc, not torch

    def host_classes(self):
        if self.S_cls is None:
            raise RuntimeError("element blocks were released after building the hierarchy")
        S = self.S_cls
        return S if isinstance(S, np.ndarray) else S.cpu().numpy()

    def schur(self):
        """Reference-layout blocks (E, 4n1, 4n1) with Dirichlet columns zeroed (local.py:186-188)."""
        S = self.host_classes()[self.elem_class].copy()
        cm = np.repeat(self.layout.side_mask(), self.p + 1, axis=1)
        return S * cm[:, None, :]

    def tocsr(self):
        """trace.py:98-128, vectorised: scatter interior (row, col) blocks."""
        lay = self.layout
        n1 = lay.n1
        if lay.ndof == 0:
            return sp.csr_matrix((0, 0))
        S = self.schur()
        nx, ny = lay.nx, lay.ny
        e = np.arange(nx * ny)
        i, j = e % nx, e // nx
        blk = np.full((nx * ny, 4), -1, np.int64)
        blk[:, 0] = np.where(j > 0, (j - 1) * nx + i, -1)
        blk[:, 2] = np.where(j < ny - 1, j * nx + i, -1)
        blk[:, 3] = np.where(i > 0, lay.nh + (i - 1) * ny + j, -1)
        blk[:, 1] = np.where(i < nx - 1, lay.nh + i * ny + j, -1)
        dof = (blk[:, :, None] * n1 + np.arange(n1)).reshape(-1, 4 * n1)
        ok = np.repeat(blk >= 0, n1, axis=1)
        rr = np.broadcast_to(dof[:, :, None], S.shape)
        cc = np.broadcast_to(dof[:, None, :], S.shape)
        m = ok[:, :, None] & ok[:, None, :]
        return sp.coo_matrix((S[m], (rr[m], cc[m])), shape=(lay.ndof, lay.ndof)).tocsr()


def element_blocks_device(op):
    """(E, 4n1, 4n1) CUDA tensor of a BlockOperator's per-element blocks (classes expanded)."""
    import torch
    S = op.S_cls if isinstance(op.S_cls, torch.Tensor) else torch.from_numpy(op.S_cls)
    S = S.to(device="cuda", dtype=torch.float64)
    E = op.elem_class.size
    if S.shape[0] == E and np.array_equal(op.elem_class, np.arange(E)):
        return S.contiguous()
    return S.index_select(0, torch.from_numpy(op.elem_class).cuda()).contiguous()


class RowChunkedOperator:
    """The stored trace operator of (mesh, p, spec) condensed and streamed chunk by chunk of
    element rows (hdg_level_create_stored_empty / hdg_level_fill_stored_rows): the element blocks
    of the whole mesh never exist at once.  configs[4]'s 8192^2 p=4 fine level on one GPU: 214.7 GB
    of blocks, 107 GB of half-stored stream.  Offers the BlockOperator apply interface."""

    def __init__(self, mesh, p, spec, rows_per_chunk=256, tau_per_facet=None):
        import torch
        from .mesh import Mesh
        dev.require_cuda()
        self.mesh, self.p = mesh, p
        self.layout = TraceLayout(mesh, p)
        self.S_cls = None
        h = ctypes.c_void_p()
        nx, ny = mesh.n_x, mesh.n_y
        check(lib.hdg_level_create_stored_empty(nx, ny, p, ctypes.byref(h)))
        self._handle = h
        for a in range(0, ny, rows_per_chunk):
            b = min(ny, a + rows_per_chunk)
            ea = max(a - 1, 0)
            win = Mesh(nx, b - ea, mesh.x0, mesh.y0 + ea * mesh.dy, mesh.dx, mesh.dy)
            tau = None
            if tau_per_facet is not None:
                raise NotImplementedError("row-chunked build with per-facet tau")
            ts = TraceSystem(win, p, spec, tau, with_rhs=False)
            blocks = element_blocks_device(ts.operator)
            del ts
            check(lib.hdg_level_fill_stored_rows(h, a, b - a, blocks.data_ptr(), dev.stream()))
            torch.cuda.synchronize()
            del blocks
            torch.cuda.empty_cache()

    @property
    def handle(self):
        return self._handle

    @property
    def ndof(self):
        return self.layout.ndof

    def operator_bytes(self):
        return int(lib.hdg_level_operator_bytes(self._handle))

    def apply(self, x):
        xd, was_np = dev.to_device(x)
        y = dev.empty(self.ndof)
        check(lib.hdg_matvec(self._handle, dev.ptr(xd), dev.ptr(y), dev.stream()))
        return dev.back(y, was_np)

    def __del__(self):
        try:
            lib.hdg_level_destroy(self._handle)
        except Exception:
            pass


class TraceSystem:
    """Condensed HDG system A lam = b on the interior facet skeleton (trace.py:26-69)."""

    # more distinct element classes than this are condensed on the GPU (PiecewiseCondenser)
    GPU_CLASSES = 4096

    def __init__(self, mesh, p, spec, tau_per_facet=None, threads=1, with_rhs=True):
        """with_rhs=False skips the condensed load (operator-only windows of strip / chunked
        builds)."""
        self.mesh, self.p, self.spec = mesh, p, spec
        self.ops = LocalOps(mesh, p)
        self.layout = TraceLayout(mesh, p)
        self.n_blocks, self.ndof = self.layout.n_blocks, self.layout.ndof
        nx, ny = mesh.n_x, mesh.n_y
        E = nx * ny
        tau = self._element_tau(spec, tau_per_facet)
        kq_rows, Ke, aniso = self._sample_coefficient(spec)               # local.py:137-140
        self.anisotropic = aniso
        nq2 = self.ops.ref.quad.nodes.size ** 2
        self.piecewise = None
        if Ke is not None and np.all(tau == tau[0]):
            # element-wise constant K (a pair for anisotropic diagonal K), uniform tau
            keys = np.stack(Ke, axis=1) if aniso else Ke[:, None]
            uk, inv = np.unique(keys, axis=0, return_inverse=True)
            inv = np.asarray(inv).reshape(-1)
            if uk.shape[0] > self.GPU_CLASSES:
                # many distinct elements: condense every element on the GPU, in element order
                # (identity classes => the stored-block relayout reads S without a gather)
                self.piecewise = PiecewiseCondenser(p, mesh.dx, mesh.dy, float(tau[0, 0]))
                self.classes = None
                self.elem_class = np.arange(E, dtype=np.int64)
                self.class_K = Ke
                self.operator = BlockOperator(mesh, p, self.piecewise.blocks(Ke), self.elem_class)
                self.rhs = self._condensed_rhs(spec) if with_rhs else None
                return
            kx = np.repeat(uk[:, :1], nq2, axis=1)
            ky = np.repeat(uk[:, -1:], nq2, axis=1) if aniso else None
            rows = np.hstack([kx] + ([ky] if aniso else []) + [np.repeat(tau[:1], uk.shape[0], axis=0)])
        else:
            rows, inv = classify_rows(np.hstack([kq_rows, tau]))
        nk = 2 * nq2 if aniso else nq2
        self.classes = ElementClasses(p, mesh.dx, mesh.dy, rows[:, :nq2], rows[:, nk:],
                                      kq_y=rows[:, nq2:nk] if aniso else None)
        self.elem_class = np.asarray(inv).reshape(-1)
        self.operator = BlockOperator(mesh, p, self.classes.S, self.elem_class)
        self.rhs = self._condensed_rhs(spec) if with_rhs else None

    def _quad_points(self, e0, e1):
        m = self.mesh
        e = np.arange(e0, e1)
        x0 = m.x0 + (e % m.n_x) * m.dx
        y0 = m.y0 + (e // m.n_x) * m.dy
        return self.ops.ref.element_quad_points(x0, y0, m.dx, m.dy)

    def _sample_coefficient(self, spec, chunk=1 << 16):
        """K at every element's GL points (local.py:137-138), in chunks.  A coefficient returning
        a (Kxx, Kyy) pair is the anisotropic diagonal extension.  Returns
        (rows, K_e, anisotropic): K_e (an (E,) array or a pair) when K is constant on every
        element, else rows of samples (E, nq^2 [x2])."""
        E = self.mesh.n_x * self.mesh.n_y
        parts, const, aniso = [], True, False
        kx_e, ky_e = np.empty(E), np.empty(E)
        for e0 in range(0, E, chunk):
            qx, qy = self._quad_points(e0, min(E, e0 + chunk))
            kq = spec.coefficient(qx, qy)
            aniso = isinstance(kq, tuple)
            kx, ky = (kq if aniso else (kq, kq))
            kx = np.asarray(kx, float).reshape(qx.shape)
            ky = np.asarray(ky, float).reshape(qx.shape)
            if np.any(kx <= 0.0) or np.any(ky <= 0.0):
                raise NumericalBreakdown("coefficient not positive")
            parts.append(np.hstack([kx, ky]) if aniso else kx)
            if const and np.all(kx == kx[:, :1]) and np.all(ky == ky[:, :1]):
                kx_e[e0:e0 + kx.shape[0]] = kx[:, 0]
                ky_e[e0:e0 + kx.shape[0]] = ky[:, 0]
            else:
                const = False
        if const:
            return None, ((kx_e, ky_e) if aniso else kx_e), aniso
        return np.concatenate(parts), None, aniso

    @classmethod
    def from_blocks(cls, mesh, p, S_cls, elem_class=None, rhs=None):
        """A system from explicit condensed blocks (e.g. the K = I shared block)."""
        self = cls.__new__(cls)
        self.mesh, self.p, self.spec = mesh, p, None
        self.ops = LocalOps(mesh, p)
        self.layout = TraceLayout(mesh, p)
        self.n_blocks, self.ndof = self.layout.n_blocks, self.layout.ndof
        S_cls = np.asarray(S_cls, float).reshape(-1, 4 * (p + 1), 4 * (p + 1))
        if elem_class is None:
            elem_class = np.zeros(mesh.n_x * mesh.n_y, np.int64)
        self.classes = None
        self.elem_class = np.asarray(elem_class, np.int64)
        self.operator = BlockOperator(mesh, p, S_cls, self.elem_class)
        self.rhs = np.zeros(self.ndof) if rhs is None else np.asarray(rhs, float)
        return self

    # -- setup helpers ----------------------------------------------------------------------
    def _element_tau(self, spec, tau_per_facet):
        E = self.mesh.n_x * self.mesh.n_y
        if tau_per_facet is None:
            return np.full((E, 4), float(spec.tau))
        return np.asarray(tau_per_facet, float)[self.mesh_elem_to_facets()]  # local.py:151-154

    def mesh_elem_to_facets(self):
        m = self.mesh
        nx, ny = m.n_x, m.n_y
        nh = nx * (ny + 1)
        j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        return np.stack([j * nx + i, nh + (i + 1) * ny + j, (j + 1) * nx + i, nh + i * ny + j],
                        axis=-1).reshape(-1, 4)

    def _condense_loads(self, idx, load):
        """condensed loads of elements idx (local.py:236)"""
        nb = self.ops.nb
        if self.piecewise is not None:
            K = self.class_K
            K = (K[0][idx], K[1][idx]) if isinstance(K, tuple) else K[idx]
            return self.piecewise.condensed_loads(K, load[:, :2 * nb], load[:, 2 * nb:])
        if self.classes.n == 1:
            return load @ self.classes.Z[0].T
        return np.einsum("eij,ej->ei", self.classes.Z[self.elem_class[idx]], load)

    def _trace_cols(self, idx):
        """unmasked trace columns T (local.py:158-176) of elements idx"""
        if self.piecewise is not None:
            pc = self.piecewise
            T = np.zeros((len(idx), 3 * pc.nb, 4 * pc.n1))
            # T_q is K-independent; T_u = -tau m on the side nodes (also K-independent)
            return T + self._Tfull()[None]
        return self.classes.T[self.elem_class[idx]]

    def _Tfull(self):
        ref, m = self.ops.ref, self.mesh
        n1, nb = ref.n1, ref.nb
        tau = float(self.spec.tau)
        lens = (m.dx, m.dy, m.dx, m.dy)
        T = np.zeros((3 * nb, 4 * n1))
        for s in range(4):
            fm = 0.5 * lens[s] * ref.mass1
            idx = ref.side_nodes[s]
            cols = slice(s * n1, (s + 1) * n1)
            for d in range(2):
                ns = (0.0, -1.0, 1.0, 0.0, 0.0, 1.0, -1.0, 0.0)[2 * s + d]
                if ns != 0.0:
                    T[d * nb + idx, cols] += ns * fm
            T[2 * nb + idx, cols] += -tau * fm
        return T

    def _element_loads(self, spec, chunk=1 << 16):
        """Yield (element indices, raw loads (n, 3nb)) for elements with a nonzero load:
        source (local.py:184) and the Dirichlet fold of the boundary datum (local.py:179-184)."""
        ref = self.ops.ref
        n1, nb = ref.n1, ref.nb
        m = self.mesh
        E = m.n_x * m.n_y
        wj = ref.w2 * (m.dx * m.dy / 4.0)
        for e0 in range(0, E, chunk):
            qx, qy = self._quad_points(e0, min(E, e0 + chunk))
            fs = np.asarray(spec.source(qx, qy), float).reshape(qx.shape)
            if not np.any(fs):
                continue
            load = np.zeros((fs.shape[0], 3 * nb))
            load[:, 2 * nb:] = (fs * wj) @ ref.interp_2d
            yield np.arange(e0, e0 + fs.shape[0]), load
        yield from self._boundary_loads(spec)

    def _boundary_loads(self, spec):
        """Dirichlet fold of the boundary datum (local.py:179-184): (boundary elements, loads)."""
        ref = self.ops.ref
        n1 = ref.n1
        m = self.mesh
        inner = self.layout.side_mask()
        bnd_e, bnd_s = np.nonzero(~inner)
        if bnd_e.size:
            t = ref.quad.nodes
            nx = m.n_x
            i, j = bnd_e % nx, bnd_e // nx
            sx = np.where(bnd_s == 1, i + 1, i)
            sy = np.where(bnd_s == 2, j + 1, j)
            px = m.x0 + sx * m.dx
            py = m.y0 + sy * m.dy
            horiz = (bnd_s == 0) | (bnd_s == 2)
            ln = np.where(horiz, m.dx, m.dy)
            sl = ln[:, None] * (t[None, :] + 1.0) / 2.0
            X = px[:, None] + np.where(horiz, 1.0, 0.0)[:, None] * sl
            Y = py[:, None] + np.where(horiz, 0.0, 1.0)[:, None] * sl
            g = np.asarray(spec.dirichlet(X, Y), float).reshape(X.shape)
            if np.any(g):
                rhs1 = (g * ref.quad.weights[None, :]) @ ref.interp_1d
                proj = np.linalg.solve(ref.mass1, rhs1.T).T                # local.py:72-78
                ub, inv = np.unique(bnd_e, return_inverse=True)
                lam_bc = np.zeros((ub.size, 4 * n1))
                for k in range(n1):
                    lam_bc[inv, bnd_s * n1 + k] = proj[:, k]
                yield ub, -np.einsum("eij,ej->ei", self._trace_cols(ub), lam_bc)

    def _element_loads_device(self, spec, chunk=1 << 16):
        """_element_loads with the loads built on the device: the source load (f w J) interp_2d is
        a hdg_gemm_nt product of the sampled source; the Dirichlet fold touches boundary elements
        only and is uploaded.  Yields (element index CUDA tensor, load (n, 3nb) CUDA tensor)."""
        import torch
        from .discretization import gemm_nt
        ref = self.ops.ref
        nb = ref.nb
        m = self.mesh
        E = m.n_x * m.n_y
        wj = torch.as_tensor(np.ascontiguousarray(ref.w2 * (m.dx * m.dy / 4.0)), device="cuda")
        interpT = torch.as_tensor(np.ascontiguousarray(ref.interp_2d.T), device="cuda")
        for e0 in range(0, E, chunk):
            qx, qy = self._quad_points(e0, min(E, e0 + chunk))
            fs = np.asarray(spec.source(qx, qy), float).reshape(qx.shape)
            if not np.any(fs):
                continue
            load = torch.zeros((fs.shape[0], 3 * nb), dtype=torch.float64, device="cuda")
            gemm_nt(torch.as_tensor(np.ascontiguousarray(fs), device="cuda"), interpT, out=load[:, 2 * nb:], colscale=wj)
            yield torch.arange(e0, e0 + fs.shape[0], device="cuda"), load
        for idx, ld in self._boundary_loads(spec):
            yield torch.as_tensor(idx, device="cuda"), torch.as_tensor(np.ascontiguousarray(ld), device="cuda")

    def _condense_loads_device(self, idx, load):
        """condensed loads (local.py:236) of elements idx (CUDA index tensor), on the device"""
        import torch
        from .discretization import gemm_nt
        nb, n1 = self.ops.nb, self.ops.n1
        if self.piecewise is not None:
            K = self.class_K
            ih = idx.cpu().numpy()
            K = (K[0][ih], K[1][ih]) if isinstance(K, tuple) else K[ih]
            return self.piecewise.condensed_loads_device(K, load[:, :2 * nb], load[:, 2 * nb:])
        Z = torch.as_tensor(np.ascontiguousarray(self.classes.Z), device="cuda")
        if self.classes.n == 1:
            return gemm_nt(load, Z[0])
        cls = torch.as_tensor(self.elem_class, dtype=torch.int64, device="cuda")[idx].contiguous()
        out = torch.empty((load.shape[0], 4 * n1), dtype=torch.float64, device="cuda")
        check(lib.hdg_class_gemv(load.shape[0], 4 * n1, 3 * nb, cls.data_ptr(), Z.data_ptr(), load.data_ptr(), 3 * nb,
                                 out.data_ptr(), 4 * n1, 1.0, 0.0, dev.stream()))
        return out

    def _condensed_rhs(self, spec):
        """Loads condensed per element (local.py:236), summed over owners (trace.py:67).  With a
        GPU: loads, condensation and the owner sum are device kernels (hdg_gemm_nt /
        hdg_class_gemv / hdg_piecewise_usolve / hdg_sum_owners); without one (CPU-only setup tests)
        the same arithmetic runs in numpy."""
        n1 = self.ops.n1
        E = self.mesh.n_x * self.mesh.n_y
        if self.ndof == 0:
            return np.zeros(0)
        if dev.cuda_available():
            import torch
            cl = torch.zeros((E, 4 * n1), dtype=torch.float64, device="cuda")
            for idx, load in self._element_loads_device(spec):
                cl.index_add_(0, idx, self._condense_loads_device(idx, load))
            rhs = dev.empty(self.ndof)
            check(lib.hdg_sum_owners(self.mesh.n_x, self.mesh.n_y, self.p, cl.data_ptr(), rhs.data_ptr(), dev.stream()))
            return rhs.cpu().numpy()
        cl = np.zeros((E, 4 * n1))
        for idx, load in self._element_loads(spec):
            cl[idx] += self._condense_loads(idx, load)
        return self.layout.sum_owners(cl)

    def reconstruct_all(self, lam):
        """trace.py:171-178 / local.py:240-251: volume (q, u) on every element from the trace
        solution, batched on the device: sol = L^-1 (load - T lam_e) per element class (two
        GEMMs), or the flux-first elimination per element for GPU-condensed media.  numpy in ->
        numpy out; a CUDA tensor in -> CUDA tensors out."""
        import torch
        nb, n1 = self.ops.nb, self.ops.n1
        E = self.mesh.n_x * self.mesh.n_y
        lam_d, was_np = dev.to_device(lam)
        if lam_d.numel() != self.ndof:
            raise ValueError(f"expected {self.ndof} trace values, got {lam_d.numel()}")
        lam_e = self._gather_device(lam_d)
        load = torch.zeros((E, 3 * nb), dtype=torch.float64, device="cuda")
        for idx, ld in self._element_loads_device(self.spec):
            load.index_add_(0, idx, ld)
        if self.piecewise is not None:
            q, u = self.piecewise.reconstruct(self.class_K, load, lam_e)
            return dev.back(q, was_np), dev.back(u, was_np)
        if self.classes is None:
            raise NotImplementedError("reconstruction needs the element classes (from_blocks system)")
        from .discretization import gemm_nt
        # sol = L^-1 (load - T lam_e): Z1 = L^-1 T applied to lam_e and L^-1 to the load
        Linv = np.linalg.inv(self.classes.L)
        if self.classes.n == 1:
            LinvT = torch.as_tensor(np.ascontiguousarray(Linv[0] @ self.classes.T[0]), device="cuda")
            sol = gemm_nt(load, torch.as_tensor(np.ascontiguousarray(Linv[0]), device="cuda"))
            gemm_nt(lam_e, LinvT, out=sol, alpha=-1.0, beta=1.0)
        else:
            cls = torch.as_tensor(self.elem_class, dtype=torch.int64, device="cuda").contiguous()
            Ld = torch.as_tensor(np.ascontiguousarray(Linv), device="cuda")
            Td = torch.as_tensor(np.ascontiguousarray(self.classes.T), device="cuda")
            rhs = load.clone()
            st = dev.stream()
            check(lib.hdg_class_gemv(E, 3 * nb, 4 * n1, cls.data_ptr(), Td.data_ptr(), lam_e.data_ptr(), 4 * n1,
                                     rhs.data_ptr(), 3 * nb, -1.0, 1.0, st))
            sol = torch.empty_like(load)
            check(lib.hdg_class_gemv(E, 3 * nb, 3 * nb, cls.data_ptr(), Ld.data_ptr(), rhs.data_ptr(), 3 * nb,
                                     sol.data_ptr(), 3 * nb, 1.0, 0.0, st))
        return dev.back(sol[:, :2 * nb].contiguous(), was_np), dev.back(sol[:, 2 * nb:].contiguous(), was_np)

    def _gather_device(self, lam_d):
        """(E, 4n1) element trace values, 0 on Dirichlet sides (trace.py:81-85), on the device
        (hdgb200.h: hdg_gather_elements)."""
        import torch
        lay = self.layout
        out = torch.empty((lay.nx * lay.ny, 4 * lay.n1), dtype=torch.float64, device="cuda")
        check(lib.hdg_gather_elements(lay.nx, lay.ny, self.p, dev.ptr(lam_d), out.data_ptr(), dev.stream()))
        return out

    def postprocess_all(self, q, u, chunk=1 << 16):
        """trace.py:180-185 / local.py:282-299: superconvergent order-(p+1) potential per element,
        batched on the device: order-raising interpolation and the K^-1 weighted flux load as
        GEMMs, then one LU-factored KKT solve for all elements at once (E right-hand sides).
        A (Kxx, Kyy) coefficient divides each flux component by its own K."""
        import torch
        m = self.mesh
        pops = PostprocessOps(self.p, m.dx, m.dy)
        qd, was_np = dev.to_device(q)
        ud, _ = dev.to_device(u)
        nb = self.ops.nb
        E = m.n_x * m.n_y
        qd, ud = qd.reshape(E, 2 * nb), ud.reshape(E, nb)
        from .discretization import gemm_nt
        cu = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")   # noqa: E731
        interp, w2 = cu(pops.interp_from_p), cu(pops.w2)
        dxi2T, deta2T = cu(pops.dxi2.T), cu(pops.deta2.T)
        n = pops.nb
        kinv = cu(np.linalg.inv(pops.kkt)[:n])                          # the potential rows of the KKT inverse
        mean_w = cu((pops.jac * (pops.w2 @ pops.interp_from_p))[None, :])   # mean_u = jac w2 . (interp u)
        out = torch.empty((E, n), dtype=torch.float64, device="cuda")
        ref = pops.ref
        for e0 in range(0, E, chunk):
            e1 = min(E, e0 + chunk)
            e = np.arange(e0, e1)
            qx, qy = ref.element_quad_points(m.x0 + (e % m.n_x) * m.dx, m.y0 + (e // m.n_x) * m.dy, m.dx, m.dy)
            kq = self.spec.coefficient(qx, qy)
            aniso = isinstance(kq, tuple)
            kx_h, ky_h = kq if aniso else (kq, kq)
            kx = cu(np.asarray(kx_h, float).reshape(qx.shape))
            ky = cu(np.asarray(ky_h, float).reshape(qx.shape)) if aniso else kx
            qh_x = gemm_nt(qd[e0:e1, :nb], interp)                       # order-raising interpolation
            qh_y = gemm_nt(qd[e0:e1, nb:], interp)
            B = torch.empty((e1 - e0, n + 1), dtype=torch.float64, device="cuda")
            gemm_nt(qh_x, dxi2T, out=B[:, :n], colscale=w2, adiv=kx, alpha=-0.5 * m.dy)
            gemm_nt(qh_y, deta2T, out=B[:, :n], colscale=w2, adiv=ky, alpha=-0.5 * m.dx, beta=1.0)
            gemm_nt(ud[e0:e1], mean_w, out=B[:, n:])
            gemm_nt(B, kinv, out=out[e0:e1])                             # KKT solve, all elements at once
        return dev.back(out, was_np)

    # -- reference attributes -----------------------------------------------------------------
    @property
    def interior(self):
        return self.layout.interior

    @property
    def block_of(self):
        return self.layout.block_of

    @property
    def schur(self):
        return self.operator.schur()

    # -- matrix-free application --------------------------------------------------------------
    def matvec_free(self, x):
        """y = A x on the GPU (trace.py:87-94).  numpy in -> numpy out; CUDA tensor -> tensor;
        FacetPlanes (device-resident facet-plane layout) -> FacetPlanes."""
        if isinstance(x, FacetPlanes):
            if x.system is not self:
                raise ValueError("FacetPlanes belongs to another TraceSystem")
            return FacetPlanes(self, self.operator.apply_planes(x.data))
        if self.ndof == 0:
            return np.zeros(0) if not hasattr(x, "is_cuda") else x.new_zeros(0)
        return self.operator.apply(x)

    def facet_planes(self, x):
        """Keep a trace vector resident on the device in the facet-plane layout (node k of every
        facet line contiguous): repeated matvec_free calls on it stream coalesced rows.  Shared-block
        (constant coefficient) systems; raises otherwise."""
        return FacetPlanes(self, self.operator.to_planes(x))

    def gather_element(self, x, e):
        """trace.py:81-85 (host view)."""
        if self.ndof == 0:
            return np.zeros(4 * self.ops.n1)
        return self.layout.gather(np.asarray(x, float))[e]

    def assemble_csr(self):
        """trace.py:98-128 (host CSR; used as a checker and for the coarse inverse)."""
        return self.operator.tocsr()

    def matvec_csr(self, x):
        return self.assemble_csr() @ x

    # -- solvers ------------------------------------------------------------------------------
    def solve_cg(self, tol=1e-12, maxiter=5000, matvec=None, precond=None, x0=None, b=None):
        """trace.py:142-163 on the device: vectors stay in HBM, the three scalars per
        iteration the reference computes (r.z, d.Ad, ||r||) cross to the host.
        `b` extends the reference signature (which always solves with self.rhs)."""
        bd, was_np = dev.to_device(self.rhs if b is None else b)
        n = bd.numel()
        s = dev.stream()
        native_pc = precond is None or hasattr(precond, "native")
        if matvec is None and native_pc:
            # the whole loop natively (hdg_pcg): iteration body = one CUDA graph, one D2H of ||r||^2
            x = dev.zeros(n) if x0 is None else dev.to_device(x0)[0].clone()
            mg = precond.native() if precond is not None else None
            hist = np.zeros(int(maxiter) + 1)
            its = ctypes.c_int(0)
            check(lib.hdg_pcg(self.operator.handle, mg.handle if mg is not None else None, dev.ptr(bd), dev.ptr(x),
                              int(x0 is not None), float(tol), int(maxiter),
                              int(getattr(precond, "nu1", 2)), int(getattr(precond, "nu2", 2)),
                              hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(its), s))
            self.cg_residuals = hist[:min(its.value, int(maxiter)) + 1]
            return dev.back(x, was_np), its.value
        mv = matvec or self.operator.apply
        x = dev.zeros(n) if x0 is None else dev.to_device(x0)[0].clone()
        r = bd - mv(x) if x0 is not None else bd.clone()
        z = precond(r) if precond else r
        d = z.clone()
        scratch = dev.empty(1)

        def dot(a, c):
            check(lib.hdg_dot(dev.ptr(a), dev.ptr(c), n, dev.ptr(scratch), s))
            return float(scratch.item())

        rz = dot(r, z)
        bnorm = dot(bd, bd) ** 0.5 or 1.0
        for it in range(maxiter):
            if dot(r, r) ** 0.5 <= tol * bnorm:
                return dev.back(x, was_np), it
            ad = mv(d)
            alpha = rz / dot(d, ad)
            check(lib.hdg_cg_update(dev.ptr(x), dev.ptr(r), dev.ptr(d), dev.ptr(ad), alpha, n, s))
            z = precond(r) if precond else r
            rz_new = dot(r, z)
            check(lib.hdg_xpby(dev.ptr(z), rz_new / rz, dev.ptr(d), n, s))
            rz = rz_new
        return dev.back(x, was_np), maxiter


def exact_trace(system, func):
    """trace.py:188-195: facet L2 projection of func onto the interior trace space (host)."""
    ref = system.ops.ref
    lay = system.layout
    m = system.mesh
    nx, ny, n1 = lay.nx, lay.ny, lay.n1
    t = ref.quad.nodes
    # interior facets in block order with their start point and tangent (mesh.py:76-90)
    jh, ih = np.meshgrid(np.arange(1, ny), np.arange(nx), indexing="ij")
    iv, jv = np.meshgrid(np.arange(1, nx), np.arange(ny), indexing="ij")
    px = np.concatenate([m.x0 + ih.ravel() * m.dx, m.x0 + iv.ravel() * m.dx])
    py = np.concatenate([m.y0 + jh.ravel() * m.dy, m.y0 + jv.ravel() * m.dy])
    horiz = np.r_[np.ones(ih.size, bool), np.zeros(iv.size, bool)]
    ln = np.where(horiz, m.dx, m.dy)
    sl = ln[:, None] * (t[None, :] + 1.0) / 2.0
    X = px[:, None] + np.where(horiz, 1.0, 0.0)[:, None] * sl
    Y = py[:, None] + np.where(horiz, 0.0, 1.0)[:, None] * sl
    g = np.asarray(func(X, Y), float).reshape(X.shape)
    rhs = (g * ref.quad.weights[None, :]) @ ref.interp_1d
    return np.linalg.solve(ref.mass1, rhs.T).T.reshape(-1) if g.size else np.zeros(0)


def flop_memop_count(system, mode):
    """trace.py:201-233 (analytic counters, reference byte model)."""
    n1 = system.ops.n1
    rows = system.ndof
    if mode == "csr":
        nnz = system.assemble_csr().nnz
        flops = 2 * nnz - rows
        bytes_ = 8 * nnz + 4 * (nnz + rows + 1) + 8 * (2 * rows)
    elif mode == "free":
        rowlen = 4 * n1
        flops = system.n_blocks * (2 * 2 * n1 * rowlen - n1)
        bytes_ = 8 * system.mesh.n_x * system.mesh.n_y * rowlen * rowlen + 8 * (2 * rows)
        bytes_ += 4 * system.n_blocks * (1 + 2 + 2 * rowlen)
    elif mode == "dense":
        flops = 2 * rows * rows - rows
        bytes_ = 8 * (rows * rows + 2 * rows)
    else:
        raise ValueError(f"unknown matvec mode {mode!r}")
    return {"flops": int(flops), "bytes": int(bytes_), "ai": flops / bytes_ if bytes_ else 0.0}


class FacetPlanes:
    """A trace vector of one TraceSystem held on the device in the facet-plane layout
    (include/hdgb200.h: hdg_soa_*).  matvec_free(FacetPlanes) -> FacetPlanes; .numpy() / .tensor()
    return the reference layout (trace.py:39-41)."""

    __slots__ = ("system", "data")

    def __init__(self, system, data):
        self.system, self.data = system, data

    def tensor(self, out=None):
        return self.system.operator.from_planes(self.data, out)

    def numpy(self):
        return self.tensor().cpu().numpy()
