"""Strip-partitioned trace operator across GPUs.

Rank g owns element rows [r0, r1) of an nx x ny mesh: the horizontal facets h(., j) and the
vertical facets v(., j) for j in [r0, r1) (bottom and left sides of its elements; Dirichlet
facets excluded).  It keeps a LOCAL mesh of element rows [lo, hi) = [max(r0-2, 0),
min(r1+1, ny)) in the reference layout, so the single-GPU kernel applies unchanged: the
owned facets' stencils only reach facets that are interior to the local mesh.  Per apply,
three facet rows cross each strip boundary:

    from the rank below: h(., r0-1) and v(., r0-1)   (its top element row)
    from the rank above: h(., r1)                     (its bottom facet row)

exchanged with NCCL point-to-point (torch.distributed batch_isend_irecv; gloo on CPU for the
tests).  The redundant ghost-row outputs are ignored.  Dots/norms reduce over owned facets
with one all-reduce.  Global <-> strip layout conversion happens once at the API boundary.
"""

from __future__ import annotations

import numpy as np


def split_rows(ny, world, align=1):
    """Even split of element rows into `world` strips, boundaries multiples of `align`."""
    units = ny // align
    if units < world:
        raise ValueError(f"{ny} rows cannot be split into {world} strips of >= {align} rows")
    base, extra = divmod(units, world)
    counts = [(base + (1 if g < extra else 0)) * align for g in range(world)]
    counts[-1] += ny - sum(counts)
    starts = np.cumsum([0] + counts)
    return [(int(starts[g]), int(starts[g + 1])) for g in range(world)]


class StripLayout:
    """Index maps of one rank's strip (host, int64)."""

    def __init__(self, nx, ny, p, world, rank, align=1, rows=None):
        self.nx, self.ny, self.p, self.n1 = nx, ny, p, p + 1
        self.world, self.rank = world, rank
        self.r0, self.r1 = rows if rows is not None else split_rows(ny, world, align)[rank]
        self.lo, self.hi = max(self.r0 - 2, 0), min(self.r1 + 1, ny)
        self.nyl = self.hi - self.lo
        n1 = self.n1
        self.nh_l = nx * (self.nyl - 1)
        self.ndof_l = n1 * (self.nh_l + (nx - 1) * self.nyl)
        self.nh_g = nx * (ny - 1)
        self.ndof_g = n1 * (self.nh_g + (nx - 1) * ny)
        # local dof -> global dof
        jl = np.arange(1, self.nyl)
        hb_l = ((jl - 1)[:, None] * nx + np.arange(nx)[None, :]).ravel()
        hb_g = ((jl + self.lo - 1)[:, None] * nx + np.arange(nx)[None, :]).ravel()
        il = np.arange(1, nx)
        jv = np.arange(self.nyl)
        vb_l = (self.nh_l + (il - 1)[:, None] * self.nyl + jv[None, :]).ravel()
        vb_g = (self.nh_g + (il - 1)[:, None] * ny + (jv + self.lo)[None, :]).ravel()
        blk_l = np.concatenate([hb_l, vb_l])
        blk_g = np.concatenate([hb_g, vb_g])
        self.local_to_global = np.empty(self.ndof_l, np.int64)
        k = np.arange(n1)
        self.local_to_global[(blk_l[:, None] * n1 + k).ravel()] = (blk_g[:, None] * n1 + k).ravel()
        # owned local dofs: rows j in [r0, r1)
        hj = np.repeat(jl + self.lo, nx)
        vj = np.tile(jv + self.lo, nx - 1)
        own_blk = np.concatenate([(hj >= self.r0) & (hj < self.r1), (vj >= self.r0) & (vj < self.r1)])
        self.owned = np.repeat(own_blk[np.argsort(blk_l)], n1)
        # halo index lists (local dofs), ordered identically on both sides of each boundary
        self.send_down = self._h_row(self.r0) if rank > 0 else np.zeros(0, np.int64)
        self.recv_up = self._h_row(self.r1) if rank < world - 1 else np.zeros(0, np.int64)
        if rank < world - 1:
            self.send_up = np.concatenate([self._h_row(self.r1 - 1), self._v_row(self.r1 - 1)])
        else:
            self.send_up = np.zeros(0, np.int64)
        if rank > 0:
            self.recv_down = np.concatenate([self._h_row(self.r0 - 1), self._v_row(self.r0 - 1)])
        else:
            self.recv_down = np.zeros(0, np.int64)
        # residual halo for the h-restriction: the coarse facets of this strip's bottom coarse row
        # gather fine residuals of the two fine rows below it (cross facets, multigrid.py:276-281)
        empty = np.zeros(0, np.int64)
        self.rsend_up = np.concatenate([self._v_row(self.r1 - 2), self._v_row(self.r1 - 1),
                                        self._h_row(self.r1 - 1)]) if rank < world - 1 else empty
        self.rrecv_down = np.concatenate([self._v_row(self.r0 - 2), self._v_row(self.r0 - 1),
                                          self._h_row(self.r0 - 1)]) if rank > 0 else empty
        self.rsend_down = self.rrecv_up = empty

    def _h_row(self, j):
        """local dofs of h(0..nx-1, j) (empty on the Dirichlet rows j = 0, ny)."""
        if j < 1 or j > self.ny - 1:
            return np.zeros(0, np.int64)
        jl = j - self.lo
        assert 1 <= jl <= self.nyl - 1, (j, self.lo, self.hi)
        b = (jl - 1) * self.nx + np.arange(self.nx)
        return (b[:, None] * self.n1 + np.arange(self.n1)).ravel()

    def _v_row(self, j):
        jl = j - self.lo
        assert 0 <= jl < self.nyl
        b = self.nh_l + np.arange(self.nx - 1) * self.nyl + jl
        return (b[:, None] * self.n1 + np.arange(self.n1)).ravel()

    # -- layout conversion (API boundary, once per solve) ------------------------------------
    def scatter(self, x_global):
        """global vector -> this rank's local vector (owned + ghost values)."""
        return x_global[self.local_to_global]

    def owned_pairs(self):
        """(local indices, global indices) of the owned dofs."""
        loc = np.flatnonzero(self.owned)
        return loc, self.local_to_global[loc]


class StripOperator:
    """y = A x on the strip with halo exchange.  `local_apply(x_local) -> y_local` is the
    single-GPU operator of the local mesh (BlockOperator.apply on the GPU)."""

    def __init__(self, layout, local_apply, group=None):
        import torch
        import torch.distributed as dist
        self.L, self.apply_local, self.group = layout, local_apply, group
        self.dist = dist
        self.torch = torch
        self._idx = {}

    def _index(self, name, device):
        key = (name, str(device))
        if key not in self._idx:
            self._idx[key] = self.torch.as_tensor(getattr(self.L, name), device=device)
        return self._idx[key]

    def exchange(self, x, kind=""):
        """Refresh x's ghost rows from the neighbours (one send/recv pair per boundary).
        kind "" = operator halo (before an apply), "r" = residual halo (before an h-restriction)."""
        L, dist, torch = self.L, self.dist, self.torch
        if L.world == 1:
            return x
        ops, recvs = [], []
        dev = x.device
        names = {"sd": kind + "send_down" if kind else "send_down", "rd": kind + "recv_down" if kind else "recv_down",
                 "su": kind + "send_up" if kind else "send_up", "ru": kind + "recv_up" if kind else "recv_up"}
        for peer, snd, rcv in ((L.rank - 1, names["sd"], names["rd"]), (L.rank + 1, names["su"], names["ru"])):
            if not (0 <= peer < L.world):
                continue
            sidx, ridx = getattr(L, snd), getattr(L, rcv)
            if sidx.size:
                ops.append(dist.P2POp(dist.isend, x[self._index(snd, dev)].contiguous(), peer, self.group))
            if ridx.size:
                buf = torch.empty(ridx.size, dtype=x.dtype, device=dev)
                ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
                recvs.append((rcv, buf))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for name, buf in recvs:
            x[self._index(name, dev)] = buf
        return x

    def apply(self, x):
        self.exchange(x)
        return self.apply_local(x)

    def dot(self, a, b):
        """sum over OWNED dofs of a*b, all-reduced."""
        m = self._owned_mask(a.device, a.dtype)
        v = (a * b * m).sum().reshape(1)
        if self.L.world > 1:
            self.dist.all_reduce(v, group=self.group)
        return v

    def _owned_mask(self, device, dtype):
        key = ("owned_mask", str(device))
        if key not in self._idx:
            self._idx[key] = self.torch.as_tensor(self.L.owned.astype(np.float64), device=device, dtype=dtype)
        return self._idx[key]


# ------------------------------------------------------------------------ distributed V-cycle


def plan_strips(shapes, world, min_rows=4):
    """shapes: [(nx, ny, p, link_to_next)] of a hierarchy (link "p" / "h" / None).  Returns
    (d, rows): levels 0..d are strip-distributed (>= min_rows element rows per rank), levels
    d+1.. run replicated on every rank (agglomeration); rows[l] = (r0, r1) of this
    partition for every distributed level l and for level d+1 (the restriction target)."""
    d = -1
    for l, (nx, ny, p, link) in enumerate(shapes[:-1]):
        if ny // world >= min_rows:
            d = l
        else:
            break
    if d < 0:
        return -1, []
    base = shapes[d + 1][1]
    parts = split_rows(base, world)
    rows = []
    for l in range(d + 2):
        f = shapes[l][1] // base
        rows.append([(r0 * f, r1 * f) for r0, r1 in parts])
    return d, rows


class StripMG:
    """Multiplicative V/W cycle (multigrid.py:393-406) on strip-partitioned levels.

    Per distributed level: operator-halo exchange before every block-Jacobi sweep and residual,
    residual-halo exchange before an h-restriction, operator-halo exchange of the coarse
    correction before the prolongation; p-transfers are facet-local.  Below level d the
    restricted residual is all-gathered and the remaining levels run replicated.  The local
    operations come from `backend` (GPU: the sm_100a kernels on row windows; tests: CSR
    restrictions of the oracle), so the orchestration here is device-agnostic."""

    def __init__(self, backend, layouts, d, group=None):
        import torch
        import torch.distributed as dist
        self.B, self.layouts, self.d = backend, layouts, d
        self.ops = [StripOperator(L, None, group) for L in layouts]
        self.torch, self.dist, self.group = torch, dist, group

    def _gather_owned(self, l, v):
        """assemble the global vector of level l from every rank's owned values"""
        torch, dist = self.torch, self.dist
        L = self.layouts[l]
        loc, glob = L.owned_pairs()
        vals = v[torch.as_tensor(loc, device=v.device)]
        idx = torch.as_tensor(glob, device=v.device)
        if L.world == 1:
            out = torch.zeros(L.ndof_g, dtype=v.dtype, device=v.device)
            out[idx] = vals
            return out
        n = torch.tensor([vals.numel()], device=v.device)
        sizes = [torch.zeros_like(n) for _ in range(L.world)]
        dist.all_gather(sizes, n, group=self.group)
        m = int(max(s.item() for s in sizes))
        pv = torch.zeros(m, dtype=v.dtype, device=v.device)
        pi = torch.full((m,), -1, dtype=torch.int64, device=v.device)
        pv[:vals.numel()] = vals
        pi[:idx.numel()] = idx
        allv = [torch.empty_like(pv) for _ in range(L.world)]
        alli = [torch.empty_like(pi) for _ in range(L.world)]
        dist.all_gather(allv, pv, group=self.group)
        dist.all_gather(alli, pi, group=self.group)
        out = torch.zeros(L.ndof_g, dtype=v.dtype, device=v.device)
        for vv, ii in zip(allv, alli):
            k = ii >= 0
            out[ii[k]] = vv[k]
        return out

    def cycle(self, l, b, x, zero_init, nu1, nu2, visits):
        B = self.B
        op = self.ops[l]
        if zero_init:
            x = B.bj_zero(l, b, 1, nu1) if nu1 >= 1 else self.torch.zeros_like(b)
            start = 1 if nu1 >= 1 else 0
        else:
            start = 0
        for k in range(start, nu1):
            op.exchange(x)
            x = B.bj_sweep(l, b, x, k + 1, nu1)
        op.exchange(x)
        if B.link(l) == "p":
            bc = B.residual_restrict_p(l, b, x)
        else:
            r = B.residual(l, b, x)
            op.exchange(r, "r")
            bc = B.restrict_h(l, r)
        if l + 1 <= self.d:
            xc = None
            for v in range(visits):
                xc = self.cycle(l + 1, bc, xc, v == 0, nu1, nu2, visits)
            self.ops[l + 1].exchange(xc)
        else:
            bg = self._gather_owned(l + 1, bc)
            xg = None
            for v in range(visits):
                xg = B.global_cycle(bg, xg, nu1, nu2, visits)
            xc = xg[self.torch.as_tensor(self.layouts[l + 1].local_to_global, device=xg.device)]
        x = B.prolong_add(l, xc, x)
        for k in range(nu2):
            op.exchange(x)
            x = B.bj_sweep(l, b, x, k + 1, nu2)
        return x

    def v_cycle(self, b, x0=None, nu1=2, nu2=2, visits=1):
        """one cycle on the strip of level 0 (b, x0: this rank's local window vectors)"""
        if x0 is None:
            return self.cycle(0, b, None, True, nu1, nu2, visits)
        return self.cycle(0, b, x0.clone(), False, nu1, nu2, visits)


class DeviceStripBackend:
    """StripMG's local operations on this rank's row windows, all in the sm_100a kernels.

    Window level l is the reference-layout trace operator of element rows [lo, hi) of level l
    (its element classes sliced from the global level), so hdg_bj_sweep / hdg_residual apply
    unchanged: every window facet has both of its elements inside the window.  p-links use
    hdg_transfer_create_p on the two windows (facet-local); h-links use
    hdg_transfer_create_h_window with the windows' global row offsets, whose kernels drop
    contributions from outside the window (only ghost facets are affected).  Levels d+1.. run
    replicated through the single-GPU device cycle (hdg_mg_cycle)."""

    def __init__(self, levels, layouts, d, omega=0.8):
        import ctypes

        import torch
        from . import _device as dev
        from ._lib import check, lib
        from .mesh import build_cartesian
        from .multigrid import BlockJacobiSmoother, Prolongation
        from .trace import BlockOperator
        self.torch, self.dev, self.lib, self.check, self.ct = torch, dev, lib, check, ctypes
        self.levels, self.layouts, self.d, self.omega = levels, layouts, d, float(omega)
        self.ops, self.links, self.transfers, self._own = [], [], [], []
        for l in range(d + 2):
            L, g = layouts[l], levels[l].block_op
            nx = L.nx
            ec = g.elem_class[L.lo * nx:L.hi * nx]
            op = BlockOperator(build_cartesian(nx, L.nyl), L.p, g.S_cls, ec)
            if l <= d:
                op.set_blockjacobi(self.omega)
            self.ops.append(op)
        for l in range(d + 1):
            P = levels[l].prolong
            if P.kind == "p":
                self.links.append("p")
                self.transfers.append(Prolongation(self.ops[l], self.ops[l + 1], "p", V=P.V))
            else:
                self.links.append("h")
                Lc = layouts[l + 1]
                cross = np.ascontiguousarray(P.cross)
                if cross.shape[0] != 1:
                    cross = np.ascontiguousarray(cross[Lc.lo * Lc.nx:Lc.hi * Lc.nx])
                hv = np.ascontiguousarray(P.halves)
                h = ctypes.c_void_p()
                check(lib.hdg_transfer_create_h_window(self.ops[l].handle, self.ops[l + 1].handle, hv.ctypes.data,
                                                       cross.ctypes.data, cross.shape[0], layouts[l].lo, Lc.lo,
                                                       ctypes.byref(h)))
                t = Prolongation(self.ops[l], self.ops[l + 1], "h", halves=hv, cross=cross)
                t._handle = h
                self.transfers.append(t)
        self.sub = levels[d + 1:]
        for lev in self.sub[:-1]:
            if not isinstance(lev.smoother, BlockJacobiSmoother) or lev.smoother.omega != self.omega:
                lev.smoother = BlockJacobiSmoother(lev.block_op, self.omega)
        self._zero = {}

    def _empty(self, l):
        return self.dev.empty(self.ops[l].ndof)

    def link(self, l):
        return self.links[l]

    def bj_sweep(self, l, b, x, k, steps):
        out = self._empty(l)
        dev = self.dev
        self.check(self.lib.hdg_bj_sweep(self.ops[l].handle, dev.ptr(b), dev.ptr(x), dev.ptr(out), dev.stream()))
        return out

    def bj_zero(self, l, b, k, steps):
        if l not in self._zero:
            self._zero[l] = self.dev.zeros(self.ops[l].ndof)
        return self.bj_sweep(l, b, self._zero[l], k, steps)

    def residual(self, l, b, x):
        r = self._empty(l)
        dev = self.dev
        self.check(self.lib.hdg_residual(self.ops[l].handle, dev.ptr(b), dev.ptr(x), dev.ptr(r), None, dev.stream()))
        return r

    def restrict_h(self, l, r):
        out = self._empty(l + 1)
        dev = self.dev
        self.check(self.lib.hdg_restrict(self.transfers[l].handle, dev.ptr(r), dev.ptr(out), dev.stream()))
        return out

    def residual_restrict_p(self, l, b, x):
        return self.restrict_h(l, self.residual(l, b, x))

    def prolong_add(self, l, ec, x):
        dev = self.dev
        self.check(self.lib.hdg_prolong_add(self.transfers[l].handle, dev.ptr(ec), dev.ptr(x), dev.stream()))
        return x

    def global_cycle(self, bg, xg, nu1, nu2, visits):
        from .multigrid import _run_cycle
        return _run_cycle(self.sub, bg, xg, nu1, nu2, visits)


def strip_multigrid(levels, world=None, rank=None, group=None, omega=0.8, min_rows=4):
    """StripMG over a hierarchy from build_hierarchy(..., smoother=None): levels whose strips
    keep >= min_rows element rows per rank are distributed, the rest replicated."""
    import torch.distributed as dist
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    shapes = [(lev.mesh.n_x, lev.mesh.n_y, lev.p, None) for lev in levels]
    d, rows = plan_strips(shapes, world, min_rows)
    if d < 0:
        raise ValueError("mesh too small to distribute")
    layouts = [StripLayout(shapes[l][0], shapes[l][1], shapes[l][2], world, rank, rows=rows[l][rank])
               for l in range(d + 2)]
    return StripMG(DeviceStripBackend(levels, layouts, d, omega), layouts, d, group)
