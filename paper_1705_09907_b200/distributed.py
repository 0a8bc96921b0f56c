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

    def _gather_plan(self, l, device):
        """Static agglomeration plan of level l (sizes and global indices of every rank's owned
        values): exchanged once, so a cycle costs ONE all_gather of values and no host sync."""
        key = (l, str(device))
        if not hasattr(self, "_plans"):
            self._plans = {}
        if key not in self._plans:
            torch, dist = self.torch, self.dist
            L = self.layouts[l]
            loc, glob = L.owned_pairs()
            plan = {"loc": torch.as_tensor(loc, device=device)}
            if L.world == 1:
                plan["glob"] = torch.as_tensor(glob, device=device)
            else:
                n = torch.tensor([loc.size], device=device)
                sizes = [torch.zeros_like(n) for _ in range(L.world)]
                dist.all_gather(sizes, n, group=self.group)
                m = int(max(int(s.item()) for s in sizes))
                pi = torch.full((m,), -1, dtype=torch.int64, device=device)
                pi[:glob.size] = torch.as_tensor(glob, device=device)
                alli = [torch.empty_like(pi) for _ in range(L.world)]
                dist.all_gather(alli, pi, group=self.group)
                gi = torch.cat(alli)
                plan.update(m=m, keep=gi >= 0, glob=gi[gi >= 0])
            self._plans[key] = plan
        return self._plans[key]

    def _gather_owned(self, l, v):
        """assemble the global vector of level l from every rank's owned values"""
        torch, dist = self.torch, self.dist
        L = self.layouts[l]
        plan = self._gather_plan(l, v.device)
        vals = v[plan["loc"]]
        out = torch.zeros(L.ndof_g, dtype=v.dtype, device=v.device)
        if L.world == 1:
            out[plan["glob"]] = vals
            return out
        pv = torch.zeros(plan["m"], dtype=v.dtype, device=v.device)
        pv[:vals.numel()] = vals
        allv = [torch.empty_like(pv) for _ in range(L.world)]
        dist.all_gather(allv, pv, group=self.group)
        out[plan["glob"]] = torch.cat(allv)[plan["keep"]]
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

    @classmethod
    def from_local(cls, H, omega=0.8):
        """The same window kernels on a rank-local hierarchy (LocalStripHierarchy): no global
        operator is ever built."""
        import ctypes

        import torch
        from . import _device as dev
        from ._lib import check, lib
        from .multigrid import BlockJacobiSmoother, Prolongation
        self = cls.__new__(cls)
        self.torch, self.dev, self.lib, self.check, self.ct = torch, dev, lib, check, ctypes
        self.levels, self.layouts, self.d, self.omega = None, H.layouts, H.d, float(omega)
        self.ops, self.links, self.transfers = list(H.ops), list(H.links), []
        for l in range(H.d + 1):
            self.ops[l].set_blockjacobi(self.omega)
        for l in range(H.d + 1):
            if H.links[l] == "p":
                self.transfers.append(Prolongation(self.ops[l], self.ops[l + 1], "p", V=H.tspecs[l]))
            else:
                halves, cross = H.tspecs[l]
                hv, cr = np.ascontiguousarray(halves), np.ascontiguousarray(cross)
                h = ctypes.c_void_p()
                check(lib.hdg_transfer_create_h_window(self.ops[l].handle, self.ops[l + 1].handle, hv.ctypes.data,
                                                       cr.ctypes.data, cr.shape[0], H.layouts[l].lo,
                                                       H.layouts[l + 1].lo, ctypes.byref(h)))
                t = Prolongation(self.ops[l], self.ops[l + 1], "h", halves=hv, cross=cr)
                t._handle = h
                self.transfers.append(t)
        self.sub = H.sub
        for lev in self.sub[:-1]:
            lev.smoother = BlockJacobiSmoother(lev.block_op, self.omega)
        self._zero = {}
        return self

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


def local_strip_multigrid(mesh, p, spec, group=None, omega=0.8, min_rows=4):
    """StripMG over a rank-local hierarchy (LocalStripHierarchy): each rank condenses and
    coarsens only its own window.  Returns (mg, H)."""
    H = LocalStripHierarchy(mesh, p, spec, RowComm(group), min_rows=min_rows)
    return StripMG(DeviceStripBackend.from_local(H, omega), H.layouts, H.d, group), H


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
    from .multigrid import HierarchyError
    for l in range(d + 2):
        if getattr(levels[l].block_op, "S_cls", True) is None:
            raise HierarchyError("strip_multigrid slices the global levels' element blocks, released on large "
                                 "device-condensed hierarchies: use local_strip_multigrid (rank-local build)")
    layouts = [StripLayout(shapes[l][0], shapes[l][1], shapes[l][2], world, rank, rows=rows[l][rank])
               for l in range(d + 2)]
    return StripMG(DeviceStripBackend(levels, layouts, d, omega), layouts, d, group)


# ------------------------------------------------------------- rank-local strip hierarchies


class RowComm:
    """Neighbour exchange and all-gather over torch.distributed (NCCL between GPUs, gloo on CPU
    for the tests).  world 1 without an initialised process group is allowed."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if on else 1
        self.rank = dist.get_rank(group) if on else 0
        self.backend = dist.get_backend(group) if on else None
        self.device = "cuda" if self.backend == "nccl" else "cpu"

    def _t(self, a):
        import torch
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        return t.to(device=self.device, dtype=torch.float64).contiguous()

    def sendrecv(self, to_below, to_above, n_below, n_above):
        """Send flat arrays to rank-1 / rank+1 and receive n_below / n_above values from them
        (one grouped send/recv)."""
        import torch
        dist = self.dist
        if self.world == 1:
            return None, None
        ops, out = [], {}
        for peer, snd, nrc, key in ((self.rank - 1, to_below, n_below, "below"),
                                    (self.rank + 1, to_above, n_above, "above")):
            if not (0 <= peer < self.world):
                continue
            if snd is not None and np.prod(snd.shape) > 0:
                ops.append(dist.P2POp(dist.isend, self._t(snd).reshape(-1), peer, self.group))
            if nrc:
                buf = torch.empty(int(nrc), dtype=torch.float64, device=self.device)
                ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
                out[key] = buf
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return out.get("below"), out.get("above")

    def all_gather(self, a):
        """list (by rank) of every rank's flat array (lengths may differ)."""
        import torch
        t = self._t(a).reshape(-1)
        if self.world == 1:
            return [t]
        dist = self.dist
        n = torch.tensor([t.numel()], dtype=torch.int64, device=self.device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(ns, n, group=self.group)
        m = int(max(int(v.item()) for v in ns))
        pad = torch.zeros(m, dtype=torch.float64, device=self.device)
        pad[:t.numel()] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(outs, pad, group=self.group)
        return [o[:int(k.item())] for o, k in zip(outs, ns)]

    def all_max(self, v):
        import torch
        if self.world == 1:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def all_sum(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return t


def _window_mesh(gm, lo, nyl):
    from .mesh import Mesh
    return Mesh(gm.n_x, nyl, gm.x0, gm.y0 + lo * gm.dy, gm.dx, gm.dy)


class _RowsView:
    """Element rows [a, a + nrows) of a level operator, as _h_level reads it (mesh.n_x, S_cls,
    elem_class)."""

    def __init__(self, op, a, nrows):
        from .mesh import Mesh
        nx = op.mesh.n_x
        self.mesh = Mesh(nx, nrows, 0.0, 0.0, 1.0, 1.0)
        self.S_cls = op.S_cls
        self.elem_class = op.elem_class[a * nx:(a + nrows) * nx]


class LocalStripHierarchy:
    """The strip-partitioned hierarchy built RANK-LOCALLY: no rank ever holds the
    global operator.  Rank g owns element rows [r0, r1) of every distributed level and keeps the
    window [r0 - 2, r1 + 1) (StripLayout).  Per level:

      fine level   the window is condensed on its own (TraceSystem on the window mesh: element
                   blocks depend only on the element's data, local.py:133-237);
      p-link       Galerkin blocks are element-local (S_c = Q^T S Q, multigrid.py:328-334): the
                   coarse window is the fine window's rows;
      h-link       each rank forms the Galerkin blocks of the coarse elements it OWNS (their
                   children are owned fine rows) and the h-transfer cross maps of its coarse
                   window (rediscretised coarse K, multigrid.py:269-293, from the coefficient
                   callable); the three ghost coarse rows come from the neighbours (one grouped
                   send/recv of element blocks);
      tail         below the last distributed level d the owned blocks of level d + 1 are
                   all-gathered and the rest of the hierarchy is built replicated on every rank
                   (agglomeration).

    `ops[l]` are the window operators (BlockOperator), `links[l]` / `tspecs[l]` the transfer
    l -> l+1 (("p", V) or ("h", (halves, window cross maps))), `sub` the replicated tail (MGLevel
    list starting at level d + 1), `layouts` the StripLayouts."""

    def __init__(self, mesh, p, spec, comm=None, tau_per_facet=None, min_rows=4, release_ndof=4_000_000):
        from .discretization import galerkin_p, h_cross_maps, h_halves, p_transfer_matrix
        from .multigrid import _coarse_classes, _h_level, hierarchy_from_operator, level_schedule
        from .trace import BlockOperator, TraceSystem
        if tau_per_facet is not None:
            raise NotImplementedError("strip hierarchies with per-facet tau")
        comm = comm or RowComm()
        self.comm = comm
        world, rank = comm.world, comm.rank
        sched = level_schedule(mesh.n_x, mesh.n_y, p)
        shapes = [(nx, ny, q, None) for nx, ny, q in sched]
        d, rows = plan_strips(shapes, world, min_rows)
        if d < 0:
            raise ValueError("mesh too small to distribute")
        self.d, self.sched = d, sched
        self.layouts = [StripLayout(sched[l][0], sched[l][1], sched[l][2], world, rank, rows=rows[l][rank])
                        for l in range(d + 2)]
        # global geometry of every level l <= d + 1
        gms = [mesh]
        for l in range(1, d + 2):
            prev = gms[-1]
            if sched[l][0] == sched[l - 1][0]:
                gms.append(prev)
            else:
                from .mesh import Mesh
                gms.append(Mesh(sched[l][0], sched[l][1], prev.x0, prev.y0, 2 * prev.dx, 2 * prev.dy))
        self.gmeshes = gms
        L0 = self.layouts[0]
        op = TraceSystem(_window_mesh(mesh, L0.lo, L0.nyl), p, spec, with_rhs=False).operator
        self.ops, self.links, self.tspecs = [op], [], []
        for l in range(d + 1):
            Lf, Lc = self.layouts[l], self.layouts[l + 1]
            qf, qc = sched[l][2], sched[l + 1][2]
            if sched[l + 1][0] == sched[l][0]:                       # p-link (same mesh)
                assert (Lc.lo, Lc.hi) == (Lf.lo, Lf.hi)
                V = p_transfer_matrix(qf)
                cop = BlockOperator(_window_mesh(gms[l + 1], Lc.lo, Lc.nyl), qc, galerkin_p(op.S_cls, V),
                                    op.elem_class)
                self.links.append("p")
                self.tspecs.append(V)
            else:                                                     # h-link
                cop, cross = self._h_window(op, Lf, Lc, gms[l + 1], spec, _h_level, _coarse_classes,
                                            h_cross_maps)
                self.links.append("h")
                self.tspecs.append((h_halves(), cross))
            if op.ndof > release_ndof and not isinstance(op.S_cls, np.ndarray) and l > 0:
                op.release_blocks()
            self.ops.append(cop)
            op = cop
        # replicated tail: all-gather the owned blocks of level d + 1
        Lt = self.layouts[d + 1]
        nxt, qt = sched[d + 1][0], sched[d + 1][2]
        Lw = 4 * (qt + 1)
        tail_op = self.ops[d + 1]
        if self._is_shared(tail_op):
            S_g, ec_g = np.asarray(self._host(tail_op.S_cls[:1])), np.zeros(nxt * sched[d + 1][1], np.int64)
        else:
            a = (Lt.r0 - Lt.lo) * nxt
            own = self._elem_blocks(tail_op)[a:a + (Lt.r1 - Lt.r0) * nxt]
            parts = comm.all_gather(own)
            S_g = np.concatenate([np.asarray(self._host(t)) for t in parts]).reshape(-1, Lw, Lw)
            ec_g = np.arange(S_g.shape[0], dtype=np.int64)
        gop = BlockOperator(gms[d + 1], qt, S_g, ec_g)
        self.sub = hierarchy_from_operator(gms[d + 1], qt, gop, spec, None, smoother=None)

    # -- helpers --------------------------------------------------------------------------------
    @staticmethod
    def _host(t):
        return t if isinstance(t, np.ndarray) else t.detach().cpu().numpy()

    @staticmethod
    def _is_shared(op):
        return op.S_cls is not None and op.S_cls.shape[0] == 1

    @staticmethod
    def _elem_blocks(op):
        S = op.S_cls
        if isinstance(S, np.ndarray):
            return S[op.elem_class]
        import torch
        return S.index_select(0, torch.as_tensor(op.elem_class, device=S.device))

    def _h_window(self, op, Lf, Lc, gmc, spec, _h_level, _coarse_classes, h_cross_maps):
        from .trace import BlockOperator
        comm = self.comm
        nxc = gmc.n_x
        r0c, r1c = Lc.r0, Lc.r1
        a = 2 * r0c - Lf.lo                                   # first owned fine row, window-local
        view = _RowsView(op, a, 2 * (r1c - r0c))
        mco = _window_mesh(gmc, r0c, r1c - r0c)
        S_c, inv, _, _ = _h_level(view, mco, spec, None)      # Galerkin blocks of the owned coarse rows
        mcw = _window_mesh(gmc, Lc.lo, Lc.nyl)
        ucols, ucls = _coarse_classes(mcw, spec, None)        # h-transfer maps of the coarse window
        cross_u = h_cross_maps(ucols)
        cross = cross_u if cross_u.shape[0] == 1 else cross_u[ucls]
        shared = comm.all_max(S_c.shape[0]) == 1 and self._agree(S_c)
        if shared:
            return BlockOperator(mcw, 1, S_c, np.zeros(nxc * Lc.nyl, np.int64)), cross
        owned = S_c[inv] if isinstance(S_c, np.ndarray) else S_c.index_select(
            0, __import__("torch").as_tensor(inv, device=S_c.device))
        per_row = nxc * 64
        nb, na = (r0c - Lc.lo), (Lc.hi - r1c)                # ghost rows below / above
        to_below = owned[:nxc] if comm.rank > 0 else None                    # my first owned row
        to_above = owned[-2 * nxc:] if comm.rank < comm.world - 1 else None   # my last two owned rows
        rb, ra = comm.sendrecv(to_below, to_above, nb * per_row, na * per_row)
        parts = []
        tgt = owned
        as_np = isinstance(tgt, np.ndarray)
        conv = (lambda t: self._host(t)) if as_np else (lambda t: t.to(tgt.device))
        if rb is not None:
            parts.append(conv(rb).reshape(-1, 8, 8))
        parts.append(tgt)
        if ra is not None:
            parts.append(conv(ra).reshape(-1, 8, 8))
        if as_np:
            win = np.concatenate(parts)
        else:
            import torch
            win = torch.cat(parts).contiguous()
        assert win.shape[0] == nxc * Lc.nyl
        return BlockOperator(mcw, 1, win, np.arange(win.shape[0], dtype=np.int64)), cross

    def _agree(self, S_c):
        """every rank formed the same single coarse block (constant coefficients)"""
        if self.comm.world == 1:
            return True
        blk = np.asarray(self._host(S_c)).reshape(-1)
        ref = self.comm.all_gather(blk)
        r0 = np.asarray(self._host(ref[0]))
        return all(np.array_equal(np.asarray(self._host(t)), r0) for t in ref)
