// hdg_fsai.cuh - facet-structured FSAI smoother (reference: multigrid.py:47-173) on the device.
//
// The baseline FSAI pattern is lower(A) (multigrid.py:127-131).  On the structured trace
// operator it is made of whole facet blocks: row (f, k) of facet f keeps the DOFs of the
// LOWER-numbered facets of f's 7-facet stencil (block_of order, trace.py:39-41: horizontal facets
// first, then vertical ones column by column) and its own DOFs m <= k.  Hence
//     h(i,j): { h(i,j-1) }                                   + own
//     v(i,j): { h(i-1,j), h(i-1,j+1), h(i,j), h(i,j+1), v(i-1,j) } + own
// (Dirichlet facets absent).  Row (f, k) solves A[P_k, P_k] g = e_last and scales g by
// 1/sqrt(g_last) (multigrid.py:133-152).  With Q = (neighbour blocks, own nodes 0..n1-1) and
// L = chol(A[Q, Q]), the leading blocks of L factor every A[P_k, P_k], and the scaled solution is
//     g_k = L_k^-T e_last  =  row (nb n1 + k) of L^-1 (first nb n1 + k + 1 entries),
// so ONE Cholesky per facet yields all n1 rows of G.  Absent neighbours enter as identity blocks
// with zero couplings, which leaves the other entries bit-identical and their G columns 0.
//
// G is stored per facet type without column indices: Gh[(k * 2n1 + c) * nhf + f],
// Gv[(k * 6n1 + c) * nvf + f], facets numbered row-major (h: (j-1) nx + i; v: j (nx-1) + i-1) so
// a thread per facet reads coalesced.  t = G r gathers r over Q; x += w G' t gathers, for facet g,
// the G columns that other facets' rows hold for g (h(i,j) appears in h(i,j+1) slot 0,
// v(i+1,j) slot 0, v(i+1,j-1) slot 1, v(i,j) slot 2, v(i,j-1) slot 3; v(i,j) in v(i+1,j) slot 4):
// no atomics, one writer per facet.
#pragma once
#include <cuda_runtime.h>

namespace hdg {

struct FsaiSetupArgs {
  const double* S;        // (C, 4 n1, 4 n1) element-class blocks, row-major, sides (B, R, T, L)
  const long long* cls;   // (E,) element -> class
  const double* Dg;       // (n_blocks, n1, n1) facet diagonal blocks of A (both owners), block_of order
  double* Gh;
  double* Gv;
  long long* bad;         // smallest failing DOF row (atomicMin; LLONG_MAX if none)
  int nx, ny;
  long long nh;           // interior horizontal facets = nx (ny - 1) = nhf
  long long nvf;          // interior vertical facets = (nx - 1) ny
};

// block_of index of the interior facets (trace.py:39-41); -1 for Dirichlet / outside
__device__ __forceinline__ long long fs_hb(int nx, int ny, int i, int j) {
  return (j >= 1 && j <= ny - 1 && i >= 0 && i < nx) ? (long long)(j - 1) * nx + i : -1;
}
__device__ __forceinline__ long long fs_vb(int nx, int ny, long long nh, int i, int j) {
  return (i >= 1 && i <= nx - 1 && j >= 0 && j < ny) ? nh + (long long)(i - 1) * ny + j : -1;
}

template <int N1>
struct FsaiCfg {
  static constexpr int MMAX = 6 * N1;             // v facets: 5 neighbour blocks + own
  static constexpr int MS = MMAX | 1;              // odd row stride: conflict-free column walks
  static constexpr int WARPS = 4;
  static constexpr int PER_WARP = MMAX * MS + N1 * MMAX * 2;   // A/L + R + acc
  static constexpr int SMEM = WARPS * PER_WARP * 8;
};

// facet diagonal blocks D_f = sum of the owners' own-side blocks (thread per entry)
template <int N1>
__global__ void fsai_diag_kernel(const double* __restrict__ S, const long long* __restrict__ cls, int nx, int ny,
                                 long long nh, long long nblocks, double* __restrict__ Dg) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nblocks * N1 * N1) return;
  const long long b = t / (N1 * N1);
  const int k = (int)(t % (N1 * N1)) / N1, m = (int)(t % N1);
  constexpr int L4 = 4 * N1;
  long long e1, e2;
  int s1, s2;
  if (b < nh) {
    const int j = (int)(b / nx) + 1, i = (int)(b % nx);
    e1 = (long long)(j - 1) * nx + i; s1 = 2;   // below: top side
    e2 = (long long)j * nx + i; s2 = 0;         // above: bottom side
  } else {
    const long long v = b - nh;
    const int i = (int)(v / ny) + 1, j = (int)(v % ny);
    e1 = (long long)j * nx + i - 1; s1 = 1;     // left: right side
    e2 = (long long)j * nx + i; s2 = 3;         // right: left side
  }
  const double* S1 = S + cls[e1] * L4 * L4;
  const double* S2 = S + cls[e2] * L4 * L4;
  Dg[t] = S1[(s1 * N1 + k) * L4 + s1 * N1 + m] + S2[(s2 * N1 + k) * L4 + s2 * N1 + m];
}

// one warp per facet: assemble A[Q,Q], Cholesky, last n1 rows of L^-1 -> n1 rows of G
template <int N1>
__global__ void __launch_bounds__(32 * FsaiCfg<N1>::WARPS) fsai_setup_kernel(const FsaiSetupArgs a) {
  using C = FsaiCfg<N1>;
  constexpr int L4 = 4 * N1, MS = C::MS;
  extern __shared__ __align__(16) double fs_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* A = fs_smem + wib * C::PER_WARP;
  double* R = A + C::MMAX * MS;
  double* acc = R + N1 * C::MMAX;
  const long long nf = a.nh + a.nvf;
  const long long nwarps = (long long)gridDim.x * C::WARPS;
  for (long long f = (long long)blockIdx.x * C::WARPS + wib; f < nf; f += nwarps) {
    const bool horiz = f < a.nh;
    int i, j;
    if (horiz) { j = (int)(f / a.nx) + 1; i = (int)(f % a.nx); }
    else { const long long v = f - a.nh; j = (int)(v / (a.nx - 1)); i = (int)(v % (a.nx - 1)) + 1; }
    const int nb = horiz ? 1 : 5;
    const int m = (nb + 1) * N1;
    // slots: global block, and side in the facet's two elements E1 (below / left), E2 (above / right)
    long long gb[6];
    int side1[6], side2[6];
    long long E1, E2;
    if (horiz) {
      E1 = (long long)(j - 1) * a.nx + i; E2 = (long long)j * a.nx + i;
      gb[0] = fs_hb(a.nx, a.ny, i, j - 1); side1[0] = 0; side2[0] = -1;       // bottom of E1
      gb[1] = fs_hb(a.nx, a.ny, i, j);     side1[1] = 2; side2[1] = 0;        // own
    } else {
      E1 = (long long)j * a.nx + i - 1; E2 = (long long)j * a.nx + i;
      gb[0] = fs_hb(a.nx, a.ny, i - 1, j);     side1[0] = 0; side2[0] = -1;   // E1 bottom
      gb[1] = fs_hb(a.nx, a.ny, i - 1, j + 1); side1[1] = 2; side2[1] = -1;   // E1 top
      gb[2] = fs_hb(a.nx, a.ny, i, j);         side1[2] = -1; side2[2] = 0;   // E2 bottom
      gb[3] = fs_hb(a.nx, a.ny, i, j + 1);     side1[3] = -1; side2[3] = 2;   // E2 top
      gb[4] = fs_vb(a.nx, a.ny, a.nh, i - 1, j); side1[4] = 3; side2[4] = -1; // E1 left
      gb[5] = fs_vb(a.nx, a.ny, a.nh, i, j);   side1[5] = 1; side2[5] = 3;    // own
    }
    const double* S1 = a.S + a.cls[E1] * L4 * L4;
    const double* S2 = a.S + a.cls[E2] * L4 * L4;
    // ---- assemble A[Q,Q] (lower triangle) into A[r * MS + c]
    for (int t = lane; t < m * m; t += 32) {
      const int r = t / m, c = t % m;
      if (c > r) continue;
      const int sr = r / N1, kr = r % N1, sc = c / N1, kc = c % N1;
      double v = 0.0;
      if (gb[sr] < 0 || gb[sc] < 0) {
        v = (r == c) ? 1.0 : 0.0;                        // absent facet: identity, no coupling
      } else if (sr == sc) {
        v = a.Dg[(gb[sr] * N1 + kr) * N1 + kc];
      } else {
        if (side1[sr] >= 0 && side1[sc] >= 0) v += S1[(side1[sr] * N1 + kr) * L4 + side1[sc] * N1 + kc];
        if (side2[sr] >= 0 && side2[sc] >= 0) v += S2[(side2[sr] * N1 + kr) * L4 + side2[sc] * N1 + kc];
      }
      A[r * MS + c] = v;
    }
    __syncwarp();
    // ---- right-looking Cholesky, lower triangle
    bool ok = true;
    int fail_col = -1;
    for (int q = 0; q < m; ++q) {
      double d = A[q * MS + q];
      if (!(d > 0.0)) { ok = false; if (fail_col < 0) fail_col = q; d = 1.0; }
      d = sqrt(d);
      for (int r = q + 1 + lane; r < m; r += 32) A[r * MS + q] /= d;
      __syncwarp();
      if (lane == 0) A[q * MS + q] = d;
      for (int r = q + 1 + lane; r < m; r += 32) {
        const double lrq = A[r * MS + q];
        for (int c = q + 1; c <= r; ++c) A[r * MS + c] = fma(-lrq, A[c * MS + q], A[r * MS + c]);
      }
      __syncwarp();
    }
    if (!ok && lane == 0) {
      // the reference reports the first row whose principal system is not SPD (multigrid.py:145)
      const long long own_row = gb[nb] * N1 + (fail_col >= nb * N1 ? fail_col - nb * N1 : 0);
      atomicMin(reinterpret_cast<unsigned long long*>(a.bad), (unsigned long long)own_row);
    }
    // ---- rows nb n1 + k of L^-1: R L = [0 | I], columns right to left
    for (int t = lane; t < N1 * C::MMAX; t += 32) acc[t] = 0.0;
    __syncwarp();
    for (int c = m - 1; c >= 0; --c) {
      if (lane < N1) {
        const double rhs = (c == nb * N1 + lane) ? 1.0 : 0.0;
        R[lane * C::MMAX + c] = (rhs - acc[lane * C::MMAX + c]) / A[c * MS + c];
      }
      __syncwarp();
      for (int t = lane; t < N1 * c; t += 32) {
        const int k = t / c, cc = t % c;
        acc[k * C::MMAX + cc] = fma(R[k * C::MMAX + c], A[c * MS + cc], acc[k * C::MMAX + cc]);
      }
      __syncwarp();
    }
    // ---- store: G[k][c] for the facet (absent slots are exact zeros)
    if (horiz) {
      for (int t = lane; t < N1 * m; t += 32) {
        const int k = t / m, c = t % m;
        a.Gh[((long long)k * 2 * N1 + c) * a.nh + f] = R[k * C::MMAX + c];
      }
    } else {
      const long long fv = f - a.nh;
      for (int t = lane; t < N1 * m; t += 32) {
        const int k = t / m, c = t % m;
        a.Gv[((long long)k * 6 * N1 + c) * a.nvf + fv] = R[k * C::MMAX + c];
      }
    }
    __syncwarp();
  }
}

struct FsaiApplyArgs {
  const double* Gh;
  const double* Gv;
  const double* x;     // input vector (reference layout)
  double* y;           // output
  const double* xin;   // AXPY: y = xin + w * (G' x)  (may alias y)
  double w;
  int nx, ny;
  long long nh, nvf;
};

// t = G r (thread per facet, row-major facet order)
template <int N1>
__global__ void fsai_g_kernel(const FsaiApplyArgs a) {
  const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= a.nh + a.nvf) return;
  if (f < a.nh) {
    const int j = (int)(f / a.nx) + 1, i = (int)(f % a.nx);
    const long long b0 = fs_hb(a.nx, a.ny, i, j - 1), own = f;
    double q[2 * N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      q[k] = b0 >= 0 ? a.x[b0 * N1 + k] : 0.0;
      q[N1 + k] = a.x[own * N1 + k];
    }
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < N1 + k + 1; ++c) s = fma(__ldg(a.Gh + ((long long)k * 2 * N1 + c) * a.nh + f), q[c], s);
      a.y[own * N1 + k] = s;
    }
  } else {
    const long long fv = f - a.nh;
    const int j = (int)(fv / (a.nx - 1)), i = (int)(fv % (a.nx - 1)) + 1;
    const long long bs[6] = {fs_hb(a.nx, a.ny, i - 1, j), fs_hb(a.nx, a.ny, i - 1, j + 1), fs_hb(a.nx, a.ny, i, j),
                             fs_hb(a.nx, a.ny, i, j + 1), fs_vb(a.nx, a.ny, a.nh, i - 1, j),
                             fs_vb(a.nx, a.ny, a.nh, i, j)};
    double q[6 * N1];
#pragma unroll
    for (int s = 0; s < 6; ++s)
#pragma unroll
      for (int k = 0; k < N1; ++k) q[s * N1 + k] = bs[s] >= 0 ? a.x[bs[s] * N1 + k] : 0.0;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 5 * N1 + k + 1; ++c) s = fma(__ldg(a.Gv + ((long long)k * 6 * N1 + c) * a.nvf + fv), q[c], s);
      a.y[bs[5] * N1 + k] = s;
    }
  }
}

// z = G' t, or x = xin + w G' t (thread per facet)
template <int N1, bool AXPY>
__global__ void fsai_gt_kernel(const FsaiApplyArgs a) {
  const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= a.nh + a.nvf) return;
  double z[N1];
#pragma unroll
  for (int m = 0; m < N1; ++m) z[m] = 0.0;
  // add  sum_k G_src[k][col0 + m] t_src[k]  over rows k of a source facet
  auto add_h = [&](long long hf, int col0, int kmin_off) {   // source: horizontal facet hf (its block index)
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const double tk = a.x[hf * N1 + k];
#pragma unroll
      for (int m = 0; m < N1; ++m)
        if (kmin_off == 0 || m <= k)
          z[m] = fma(__ldg(a.Gh + ((long long)k * 2 * N1 + col0 + m) * a.nh + hf), tk, z[m]);
    }
  };
  auto add_v = [&](int vi, int vj, int col0, int own) {      // source: vertical facet v(vi, vj)
    const long long fv = (long long)vj * (a.nx - 1) + (vi - 1);
    const long long vb = a.nh + (long long)(vi - 1) * a.ny + vj;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const double tk = a.x[vb * N1 + k];
#pragma unroll
      for (int m = 0; m < N1; ++m)
        if (!own || m <= k)
          z[m] = fma(__ldg(a.Gv + ((long long)k * 6 * N1 + col0 + m) * a.nvf + fv), tk, z[m]);
    }
  };
  long long ob;   // output block
  if (f < a.nh) {
    const int j = (int)(f / a.nx) + 1, i = (int)(f % a.nx);
    ob = f;
    add_h(f, N1, 1);                                                  // own rows (lower triangle)
    if (j + 1 <= a.ny - 1) add_h(f + a.nx, 0, 0);                     // h(i, j+1) slot 0
    if (i + 1 <= a.nx - 1) { add_v(i + 1, j, 0, 0); add_v(i + 1, j - 1, N1, 0); }   // slots 0, 1
    if (i >= 1) { add_v(i, j, 2 * N1, 0); add_v(i, j - 1, 3 * N1, 0); }             // slots 2, 3
  } else {
    const long long fv = f - a.nh;
    const int j = (int)(fv / (a.nx - 1)), i = (int)(fv % (a.nx - 1)) + 1;
    ob = a.nh + (long long)(i - 1) * a.ny + j;
    add_v(i, j, 5 * N1, 1);                                           // own
    if (i + 1 <= a.nx - 1) add_v(i + 1, j, 4 * N1, 0);                // v(i+1, j) slot 4
  }
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    if constexpr (AXPY) a.y[ob * N1 + m] = fma(a.w, z[m], a.xin[ob * N1 + m]);
    else a.y[ob * N1 + m] = z[m];
  }
}

// v <- w / ||w|| given the device norm^2 (power iteration step, multigrid.py:167-172)
static __global__ void fsai_scale_kernel(const double* __restrict__ w, const double* __restrict__ nrm2, double* __restrict__ v,
                                  double* __restrict__ lam_out, long long n) {
  const double lam = sqrt(*nrm2);
  if (blockIdx.x == 0 && threadIdx.x == 0) *lam_out = lam;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    v[t] = lam > 0.0 ? w[t] / lam : 0.0;
}

}  // namespace hdg
