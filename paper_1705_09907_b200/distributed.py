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

    def __init__(self, nx, ny, p, world, rank, align=1):
        self.nx, self.ny, self.p, self.n1 = nx, ny, p, p + 1
        self.world, self.rank = world, rank
        self.r0, self.r1 = split_rows(ny, world, align)[rank]
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

    def exchange(self, x):
        """Refresh x's ghost rows from the neighbours (one send/recv pair per boundary)."""
        L, dist, torch = self.L, self.dist, self.torch
        if L.world == 1:
            return x
        ops, recvs = [], []
        dev = x.device
        if L.rank > 0:
            sd = x[self._index("send_down", dev)].contiguous()
            rd = torch.empty(L.recv_down.size, dtype=x.dtype, device=dev)
            ops += [dist.P2POp(dist.isend, sd, L.rank - 1, self.group),
                    dist.P2POp(dist.irecv, rd, L.rank - 1, self.group)]
            recvs.append(("recv_down", rd))
        if L.rank < L.world - 1:
            su = x[self._index("send_up", dev)].contiguous()
            ru = torch.empty(L.recv_up.size, dtype=x.dtype, device=dev)
            ops += [dist.P2POp(dist.isend, su, L.rank + 1, self.group),
                    dist.P2POp(dist.irecv, ru, L.rank + 1, self.group)]
            recvs.append(("recv_up", ru))
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
