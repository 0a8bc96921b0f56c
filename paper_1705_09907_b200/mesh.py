"""Structured Cartesian meshes (reference: mesh.py).

The device never stores connectivity: kernels compute facet/element indices
arithmetically.  This host class keeps the reference's
numbering and attribute names (mesh.py:24-109) so reference-style callers work;
the connectivity arrays are built lazily and vectorised.  Any object with
n_x, n_y, x0, y0, dx, dy (e.g. a reference `hdgmg.mesh.Mesh`) is accepted by
TraceSystem / build_hierarchy.
"""

from __future__ import annotations

import numpy as np

SIDE_BOTTOM, SIDE_RIGHT, SIDE_TOP, SIDE_LEFT = 0, 1, 2, 3
NORMALS = np.array([[0.0, -1.0], [1.0, 0.0], [0.0, 1.0], [-1.0, 0.0]])


class MeshError(ValueError):
    pass


class Mesh:
    """n_x-by-n_y quad mesh of an axis-aligned rectangle (mesh.py:24-56)."""

    def __init__(self, n_x, n_y, x0, y0, dx, dy, child_elements=None):
        self.n_x, self.n_y = int(n_x), int(n_y)
        self.x0, self.y0, self.dx, self.dy = float(x0), float(y0), float(dx), float(dy)
        self.child_elements = child_elements
        self._cache = {}

    @property
    def n_elems(self):
        return self.n_x * self.n_y

    @property
    def n_h(self):
        return self.n_x * (self.n_y + 1)

    @property
    def n_facets(self):
        return self.n_h + self.n_y * (self.n_x + 1)

    def _arrays(self):
        if not self._cache:
            nx, ny, nh = self.n_x, self.n_y, self.n_h
            j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
            e = (j * nx + i).ravel()
            fb = (j * nx + i).ravel()
            ft = ((j + 1) * nx + i).ravel()
            fl = (nh + i * ny + j).ravel()
            fr = (nh + (i + 1) * ny + j).ravel()
            e2f = np.stack([fb, fr, ft, fl], axis=1).astype(np.int64)
            f2e = np.full((self.n_facets, 2, 2), -1, np.int64)
            f2e[ft, 0] = np.stack([e, np.full_like(e, SIDE_TOP)], 1)
            f2e[fb, 1] = np.stack([e, np.full_like(e, SIDE_BOTTOM)], 1)
            f2e[fr, 0] = np.stack([e, np.full_like(e, SIDE_RIGHT)], 1)
            f2e[fl, 1] = np.stack([e, np.full_like(e, SIDE_LEFT)], 1)
            axis = np.zeros(self.n_facets, np.int8)
            axis[nh:] = 1
            bnd = np.zeros(self.n_facets, bool)
            bnd[np.arange(nx)] = True
            bnd[ny * nx + np.arange(nx)] = True
            bnd[nh + np.arange(ny)] = True
            bnd[nh + nx * ny + np.arange(ny)] = True
            self._cache.update(elem_to_facets=e2f, facet_to_elems=f2e, facet_axis=axis, facet_boundary=bnd)
        return self._cache

    @property
    def elem_to_facets(self):
        return self._arrays()["elem_to_facets"]

    @property
    def facet_to_elems(self):
        return self._arrays()["facet_to_elems"]

    @property
    def facet_axis(self):
        return self._arrays()["facet_axis"]

    @property
    def facet_boundary(self):
        return self._arrays()["facet_boundary"]

    @property
    def interior_facets(self):
        return np.flatnonzero(~self.facet_boundary)

    def elem_cell(self, e):
        return e % self.n_x, e // self.n_x

    def elem_origin(self, e):
        i, j = self.elem_cell(e)
        return self.x0 + i * self.dx, self.y0 + j * self.dy

    def facet_length(self, f):
        return self.dx if f < self.n_h else self.dy

    def facet_geometry(self, f):
        """mesh.py:76-84."""
        if f < self.n_h:
            i, j = f % self.n_x, f // self.n_x
            return (self.x0 + i * self.dx, self.y0 + j * self.dy), (1.0, 0.0)
        k = f - self.n_h
        i, j = k // self.n_y, k % self.n_y
        return (self.x0 + i * self.dx, self.y0 + j * self.dy), (0.0, 1.0)

    def facet_points(self, f, t):
        (px, py), (tx, ty) = self.facet_geometry(f)
        s = self.facet_length(f) * (np.asarray(t) + 1.0) / 2.0
        return px + tx * s, py + ty * s

    def normal(self, e, side):
        return NORMALS[side]


def build_cartesian(n_x, n_y, domain=((0.0, 1.0), (0.0, 1.0))):
    """mesh.py:120-163."""
    if n_x < 1 or n_y < 1:
        raise MeshError(f"element counts must be positive, got ({n_x}, {n_y})")
    (xa, xb), (ya, yb) = domain
    if not (xb > xa and yb > ya):
        raise MeshError("domain must have positive area")
    return Mesh(n_x, n_y, xa, ya, (xb - xa) / n_x, (yb - ya) / n_y)


def coarsen(mesh):
    """mesh.py:166-196: halve each direction; children (SW, SE, NW, NE)."""
    if mesh.n_x % 2 or mesh.n_y % 2:
        raise MeshError(f"cannot coarsen a {mesh.n_x}x{mesh.n_y} mesh: element counts must be even")
    nx, ny = mesh.n_x // 2, mesh.n_y // 2
    cj, ci = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    base = (2 * cj * mesh.n_x + 2 * ci).ravel()
    kids = np.stack([base, base + 1, base + mesh.n_x, base + mesh.n_x + 1], axis=1).astype(np.int64)
    c = build_cartesian(nx, ny, ((mesh.x0, mesh.x0 + mesh.n_x * mesh.dx),
                                 (mesh.y0, mesh.y0 + mesh.n_y * mesh.dy)))
    return Mesh(c.n_x, c.n_y, c.x0, c.y0, c.dx, c.dy, child_elements=kids)
