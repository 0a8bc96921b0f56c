"""FSAI smoother: host setup, device application (reference: multigrid.py:38-173).

Setup (host, once per level) restates `fsai_build`: for every row i of the lower-triangular
pattern, solve the dense SPD principal system A[P_i, P_i] g = e_last and scale g by
1/sqrt(g_last) (multigrid.py:133-152) - here batched over all rows at once (rows padded to a
common length with identity blocks).  lambda_max of G'G A by the same 20-step power
iteration with seed 1234 (multigrid.py:162-173), Chebyshev sweep weights on
[frac lambda_max, lambda_max] (multigrid.py:76-81).

Application runs on the device: x <- x + w_k G'(G(b - A x)) is one residual kernel + two CSR
SpMV kernels (the second fused with the update) per sweep (hdg_fsai_sweeps).
"""

from __future__ import annotations

import ctypes
import warnings

import numpy as np
import scipy.sparse as sp

from . import _device as dev
from ._lib import check, lib

CHEB_LOWER_FRACTION = 0.15             # multigrid.py:43
CHEB_LOWER_FRACTION_AGGRESSIVE = 0.30  # multigrid.py:44


class NotSPDError(RuntimeError):
    """multigrid.py:34."""


def _aggressive_pattern(A, power, max_complexity):
    """multigrid.py:91-120: lower(|A|^power), the strongest extra couplings filling the budget."""
    absA = sp.csr_matrix((np.abs(A.data), A.indices, A.indptr), shape=A.shape)
    W = absA
    for _ in range(power - 1):
        W = (W @ absA).tocsr()
    lower = sp.tril(W, format="coo")
    base = sp.tril(A, format="coo")
    budget = int((max_complexity * A.nnz + A.shape[0]) // 2)
    if lower.nnz <= budget:
        return lower.tocsr()
    n = A.shape[0]
    key_low = lower.row.astype(np.int64) * n + lower.col
    in_base = np.isin(key_low, base.row.astype(np.int64) * n + base.col)
    extras = np.flatnonzero(~in_base)
    room = max(budget - int(in_base.sum()), 0)
    order = extras[np.argsort(-lower.data[extras], kind="stable")][:room]
    keep = np.concatenate([np.flatnonzero(in_base), order])
    return sp.coo_matrix((np.ones(keep.size), (lower.row[keep], lower.col[keep])), shape=A.shape).tocsr()


def _rows_solve(A, pattern):
    """All FSAI rows at once: (n, L, L) principal blocks, real entries at the end of each row."""
    n = A.shape[0]
    counts = np.diff(pattern.indptr)
    L = int(counts.max()) if n else 0
    cols = np.zeros((n, L), np.int64)
    valid = np.zeros((n, L), bool)
    rr = np.repeat(np.arange(n), counts)
    pos = np.arange(pattern.nnz) - np.repeat(pattern.indptr[:-1], counts) + np.repeat(L - counts, counts)
    cols[rr, pos] = pattern.indices
    valid[rr, pos] = True
    out = np.empty(pattern.nnz)
    chunk = max(1, (1 << 24) // max(L * L, 1))
    Acsr = A.tocsr()
    for s in range(0, n, chunk):
        c = cols[s:s + chunk]
        v = valid[s:s + chunk]
        m = c.shape[0]
        sub = np.asarray(Acsr[np.repeat(c, L, axis=1).ravel(), np.tile(c, (1, L)).ravel()]).reshape(m, L, L)
        mask2 = v[:, :, None] & v[:, None, :]
        sub = np.where(mask2, sub, 0.0)
        eye = np.broadcast_to(np.eye(L), sub.shape)
        sub = np.where((~v)[:, :, None] & (~v)[:, None, :], eye, sub)
        rhs = np.zeros((m, L))
        rhs[:, -1] = 1.0
        try:
            g = np.linalg.solve(sub, rhs[:, :, None])[:, :, 0]
        except np.linalg.LinAlgError as exc:
            raise NotSPDError("singular principal submatrix in FSAI") from exc
        if np.any(g[:, -1] <= 0.0):
            bad = s + int(np.flatnonzero(g[:, -1] <= 0.0)[0])
            raise NotSPDError(f"non-SPD principal submatrix in FSAI row {bad}")
        g = g / np.sqrt(g[:, -1:])
        out[pattern.indptr[s]:pattern.indptr[min(s + chunk, n)]] = g[v]
    return out


def _rows_solve_device(A, pattern):
    """_rows_solve on the GPU (hdg_fsai_rows: one thread per row, Cholesky of the gathered
    principal block); A and the pattern go up once as int32 CSR, G's values come back."""
    import torch
    n = A.shape[0]
    counts = np.diff(pattern.indptr)
    max_len = int(counts.max()) if n else 0
    if max_len > 96 or A.nnz >= 2 ** 31 or pattern.nnz >= 2 ** 31:
        # not silent: the device kernel holds one gathered block of <= 96 x 96 per thread
        warnings.warn(f"FSAI row solves on the host: pattern rows up to {max_len} entries "
                      f"(device kernel limit 96) or nnz >= 2^31", RuntimeWarning, stacklevel=2)
        return _rows_solve(A, pattern)
    Acsr = A.tocsr()
    Acsr.sort_indices()
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()
    a_ptr, a_col, a_val = t(Acsr.indptr, np.int32), t(Acsr.indices, np.int32), t(Acsr.data, np.float64)
    g_ptr, g_col = t(pattern.indptr, np.int32), t(pattern.indices, np.int32)
    g_val = torch.empty(pattern.nnz, dtype=torch.float64, device="cuda")
    bad = ctypes.c_int64(-1)
    check(lib.hdg_fsai_rows(n, a_ptr.data_ptr(), a_col.data_ptr(), a_val.data_ptr(), g_ptr.data_ptr(),
                            g_col.data_ptr(), g_val.data_ptr(), max_len, ctypes.byref(bad), dev.stream()))
    if bad.value >= 0:
        raise NotSPDError(f"non-SPD principal submatrix in FSAI row {bad.value}")
    return g_val.cpu().numpy()


class FSAISmoother:
    """multigrid.py:47-88 with device application.  Host attributes match the reference
    (G, Gt scipy CSR; omega, aggressiveness, complexity, lam_max, cheb_fraction)."""

    def __init__(self, G, omega, aggressiveness, complexity, lam_max, cheb_fraction):
        self.G = G
        self.Gt = G.T.tocsr()
        self.omega = omega
        self.aggressiveness = aggressiveness
        self.complexity = complexity
        self.lam_max = lam_max
        self.cheb_fraction = cheb_fraction
        self.block_op = None

    def sweep_weights(self, steps):
        lo, hi = self.cheb_fraction * self.lam_max, self.lam_max
        mid, half = 0.5 * (hi + lo), 0.5 * (hi - lo)
        k = np.arange(1, steps + 1)
        return self.omega / (mid + half * np.cos(np.pi * (2 * k - 1) / (2 * steps)))

    # -- device ------------------------------------------------------------------------------
    def bind(self, block_op):
        """Upload G and G' to the level's native handle (hdg_level_set_fsai)."""
        G, Gt = self.G.tocsr(), self.Gt
        G.sort_indices()
        Gt.sort_indices()
        arrs = [np.ascontiguousarray(a) for a in (G.indptr.astype(np.int32), G.indices.astype(np.int32), G.data,
                                                  Gt.indptr.astype(np.int32), Gt.indices.astype(np.int32), Gt.data)]
        check(lib.hdg_level_set_fsai(block_op.handle, G.shape[0], arrs[0].ctypes.data, arrs[1].ctypes.data,
                                     arrs[2].ctypes.data, G.nnz, arrs[3].ctypes.data, arrs[4].ctypes.data,
                                     arrs[5].ctypes.data, float(self.lam_max), float(self.cheb_fraction),
                                     float(self.omega)))
        self.block_op = block_op
        return self

    def apply_inverse(self, r):
        """G'(G r) on the device (multigrid.py:72-74)."""
        rd, was_np = dev.to_device(r)
        out = dev.empty(rd.numel())
        check(lib.hdg_fsai_apply(self.block_op.handle, dev.ptr(rd), dev.ptr(out), dev.stream()))
        return dev.back(out, was_np)

    def smooth(self, matvec, b, x, steps):
        """multigrid.py:83-88 on the device (the level's own operator is applied)."""
        if steps < 1:
            return x
        bd, was_np = dev.to_device(b)
        xd = dev.to_device(x)[0].clone()
        n = xd.numel()
        r, t = dev.empty(n), dev.empty(n)
        check(lib.hdg_fsai_sweeps(self.block_op.handle, dev.ptr(bd), dev.ptr(xd), dev.ptr(r), dev.ptr(t),
                                  int(steps), dev.stream()))
        return dev.back(xd, was_np)


class StructuredFSAI(FSAISmoother):
    """FSAISmoother with the baseline pattern lower(A) (multigrid.py:123-159) set up ENTIRELY on
    the device from the level's element blocks (hdg_level_set_fsai_struct, hdg_fsai.cuh): one
    Cholesky per facet gives the facet's n1 rows of G, stored per facet without column indices;
    lambda_max(G'GA) by the reference's 20 power steps from its seed-1234 start vector
    (multigrid.py:162-173).  No host CSR, no host pattern: this is the path for large levels.
    `.G` / `.Gt` assemble scipy CSR views on demand (small levels; tests and API parity)."""

    LAM_ITERS = 20

    def __init__(self, block_op, omega=1.0, seed=1234):
        import torch
        self.block_op = block_op
        self.omega = float(omega)
        self.aggressiveness = 1
        self.cheb_fraction = CHEB_LOWER_FRACTION
        self.complexity = 1.0          # (2 nnz(lower A) - n) / nnz(A) for a symmetric pattern
        self._G = None
        n = block_op.ndof
        S = block_op.S_cls
        if S is None:
            raise ValueError("structured FSAI needs the level's element blocks (build it before release_blocks)")
        S = S if isinstance(S, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(S))
        S = S.to(device="cuda", dtype=torch.float64).contiguous()
        cls = torch.from_numpy(np.ascontiguousarray(block_op.elem_class, dtype=np.int64)).cuda()
        v0 = torch.from_numpy(np.random.default_rng(seed).standard_normal(n)).cuda() if n else None
        lam = ctypes.c_double(1.0)
        bad = ctypes.c_int64(-1)
        import time
        t0 = time.perf_counter()
        rc = lib.hdg_level_set_fsai_struct(block_op.handle, S.data_ptr(), cls.data_ptr(),
                                           v0.data_ptr() if v0 is not None else None, self.LAM_ITERS,
                                           self.cheb_fraction, self.omega, ctypes.byref(lam), ctypes.byref(bad),
                                           dev.stream())
        if bad.value >= 0:
            raise NotSPDError(f"non-SPD principal submatrix in FSAI row {bad.value}")
        check(rc)
        self.lam_max = float(lam.value)
        self.setup_s = time.perf_counter() - t0        # factor + lambda_max (the call synchronises)

    def bind(self, block_op):
        if block_op is not self.block_op:
            raise ValueError("a structured FSAI factor belongs to the level it was built on")
        return self

    @property
    def G(self):
        if self._G is None:
            self._G = self._assemble()
        return self._G

    @property
    def Gt(self):
        return self.G.T.tocsr()

    def _assemble(self):
        """Host CSR of the device factor: rows (f, k), columns of the pattern lower(A)."""
        lay = self.block_op.layout
        nx, ny, n1, nh = lay.nx, lay.ny, lay.n1, lay.nh
        nv = (nx - 1) * ny
        gh = np.zeros(nh * n1 * 2 * n1)
        gv = np.zeros(max(nv, 0) * n1 * 6 * n1)
        check(lib.hdg_level_fsai_struct_get(self.block_op.handle, gh.ctypes.data, gv.ctypes.data))
        rows, cols, vals = [], [], []

        def hb(i, j):
            return np.where((j >= 1) & (j <= ny - 1) & (i >= 0) & (i < nx), (j - 1) * nx + i, -1)

        def vb(i, j):
            return np.where((i >= 1) & (i <= nx - 1) & (j >= 0) & (j < ny), nh + (i - 1) * ny + j, -1)

        def emit(G, nslot, own_blk, slot_blk, nf):
            G = G.reshape(n1, nslot * n1, nf)
            for k in range(n1):
                for s_ in range(nslot):
                    for m in range(n1):
                        if s_ == nslot - 1 and m > k:
                            continue
                        blk = slot_blk[s_]
                        ok = blk >= 0
                        rows.append(own_blk[ok] * n1 + k)
                        cols.append(blk[ok] * n1 + m)
                        vals.append(G[k, s_ * n1 + m, ok])

        if nh:
            f = np.arange(nh)
            j, i = f // nx + 1, f % nx
            emit(gh, 2, f, [hb(i, j - 1), f], nh)
        if nv > 0:
            fv = np.arange(nv)
            j, i = fv // (nx - 1), fv % (nx - 1) + 1
            own = vb(i, j)
            emit(gv, 6, own, [hb(i - 1, j), hb(i - 1, j + 1), hb(i, j), hb(i, j + 1), vb(i - 1, j), own], nv)
        n = lay.ndof
        if not rows:
            return sp.csr_matrix((n, n))
        G = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()
        G.sort_indices()
        return G


def structured_fsai_supported(block_op, aggressiveness=1):
    return aggressiveness == 1 and 1 <= block_op.layout.n1 <= 9 and getattr(block_op, "S_cls", None) is not None


def _estimate_lam_max(A, G, iters=20, seed=1234):
    """multigrid.py:162-173 (host, deterministic)."""
    Gt = G.T.tocsr()
    v = np.random.default_rng(seed).standard_normal(A.shape[0])
    lam = 1.0
    for _ in range(iters):
        w = Gt @ (G @ (A @ v))
        lam = np.linalg.norm(w)
        if lam == 0.0:
            return 1.0
        v = w / lam
    return lam


def _estimate_lam_max_device(A, G, iters=20, seed=1234):
    """_estimate_lam_max with the three sparse products per step on the GPU (setup only; the same
    seed-1234 start vector as multigrid.py:162-173)."""
    import torch

    import warnings

    def csr(M):
        M = M.tocsr()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)   # torch marks sparse CSR as beta
            return torch.sparse_csr_tensor(torch.from_numpy(M.indptr.astype(np.int64)),
                                           torch.from_numpy(M.indices.astype(np.int64)),
                                           torch.from_numpy(np.ascontiguousarray(M.data, dtype=np.float64)),
                                           size=M.shape).cuda()
    Ad, Gd, Gtd = csr(A), csr(G), csr(G.T)
    v = torch.from_numpy(np.random.default_rng(seed).standard_normal(A.shape[0])).cuda()
    lam = 1.0
    for _ in range(iters):
        w = Gtd @ (Gd @ (Ad @ v))
        lam = float(torch.linalg.vector_norm(w))
        if lam == 0.0:
            return 1.0
        v = w / lam
    return lam


def fsai_build(A, aggressiveness=1, omega=1.0, max_complexity=2.85, device=None):
    """multigrid.py:123-159.  The per-row SPD solves run on the GPU (hdg_fsai_rows) when one is
    present (device=None) — the host restatement is ~34 us/row (baseline) to ~250 us/row
    (aggressive), minutes at configs[1] sizes."""
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    if aggressiveness == 1:
        pattern = sp.tril(A, format="csr")
    else:
        pattern = _aggressive_pattern(A, aggressiveness, max_complexity)
    pattern.sort_indices()
    if device is None:
        device = dev.cuda_available()
    if not n:
        data = np.zeros(0)
    elif device:
        data = _rows_solve_device(A, pattern)
    else:
        data = _rows_solve(A, pattern)
    G = sp.csr_matrix((data, pattern.indices.astype(np.int64), pattern.indptr.astype(np.int64)), shape=(n, n))
    complexity = (2 * G.nnz - n) / A.nnz if A.nnz else 1.0
    if not n:
        lam_max = 1.0
    elif device:
        lam_max = _estimate_lam_max_device(A, G)
    else:
        lam_max = _estimate_lam_max(A, G)
    frac = CHEB_LOWER_FRACTION if aggressiveness == 1 else CHEB_LOWER_FRACTION_AGGRESSIVE
    return FSAISmoother(G, omega, aggressiveness, complexity, lam_max, frac)
