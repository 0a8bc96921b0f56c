// hdg_kernels.cuh - sm_100a kernels for the HDG trace operator and its multigrid cycle.
//
// Reference path (pure numpy in /root/reference/pkg/src/hdgmg):
//   matvec_free            trace.py:87-94   gather -> per-element GEMV -> two-owner sum
//   block-Jacobi smoother  north star, plugs into multigrid.py:397-405
//   residual + restriction multigrid.py:399    prolongation multigrid.py:403
//   p/h transfers          multigrid.py:215-298
//   coarse solve           multigrid.py:209-212
//
// Design (DESIGN.md has the full story):
//  * Edge-centric, one writer per interior facet, no atomics, no grid sync.
//  * A CTA owns a TX x TY tile of elements and computes the facets h(i,j) (bottom of
//    element (i,j)) and v(i,j) (left of element (i,j)) of that tile: one thread = one
//    horizontal + one vertical facet.  The x values of the facet stencil (7 facet blocks
//    per facet) are staged once per CTA into shared memory with coalesced loads
//    (odd per-block stride => conflict-free 64-bit LDS).
//  * Operator per facet = the two owner elements' side rows merged into ONE n1 x 7n1
//    matrix over the 7 stencil blocks (the shared facet's two diagonal blocks are summed,
//    so the stencil is 7 n1^2 FMAs instead of 8 n1^2).
//      - shared mode (constant K and tau): the two merged matrices (h and v)
//        live in the kernel-parameter constant bank; DFMA reads them as c[][] operands.
//      - stored mode (per-element blocks): merged matrices are re-laid out once at
//        setup into a facet-interleaved SoA stream [warp group][entry][lane], so
//        a warp's 32 facets read 256 contiguous bytes per load instruction, streamed with
//        evict-first hints; 7 n1^2 doubles per facet (12.5% fewer bytes than the
//        reference's (E, 4n1, 4n1) layout, whose boundary-side rows are never needed).
//  * Epilogues fuse what follows the apply: residual, residual norm^2 partials, damped
//    block-Jacobi update, and residual + p-restriction.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hdg {

constexpr int TX = 32;   // tile width in elements (= warp width: lanes walk i)
constexpr int TY = 8;    // tile height in elements (= warps per CTA)
constexpr int NT = TX * TY;
constexpr int MAXN1 = 13;  // p <= 12

enum Epi { EPI_Y = 0, EPI_RES = 1, EPI_BJ = 2, EPI_RESPR = 3 };

template <int N1> struct Cfg {
  static constexpr int S = (N1 & 1) ? N1 : N1 + 1;  // odd smem stride per facet block
  static constexpr int WSZ = 7 * N1 * N1;           // merged facet operator entries
  static constexpr int DSZ = N1 * N1;               // block-Jacobi inverse entries
  static constexpr int QUNROLL = (N1 <= 8) ? 7 : 1; // keep registers bounded at high order
  static constexpr int HROWS = TY + 2, HCOLS = TX + 1;
  static constexpr int VCOLS = TX + 2, VROWS = TY + 1;
  static constexpr int SMEM_DOUBLES = (HROWS * HCOLS + VCOLS * VROWS) * S;
};

// Shared-mode operator: both merged facet matrices + block-Jacobi inverses.
// Passed by value => constant bank; fully unrolled indices become c[0x0][imm] operands.
template <int N1> struct SharedOp {
  double Wh[7 * N1 * N1];
  double Wv[7 * N1 * N1];
  double Dh[N1 * N1];
  double Dv[N1 * N1];
};

struct MvArgs {
  int nx, ny, nxp;          // mesh and padded interleave row length (multiple of 32)
  long long nh;             // interior horizontal facet blocks = nx * (ny - 1)
  const double* x;          // input trace vector
  const double* b;          // right-hand side (RES / BJ / RESPR)
  double* out;              // y | r | x_out | r_coarse
  const double* Wh;         // stored mode: interleaved merged operators [grp][idx][lane]
  const double* Wv;
  const double* Dh;         // stored mode: interleaved D^-1 [grp][idx][lane]
  const double* Dv;
  double omega;
  double* partials;         // per-CTA norm^2 partials (RES) or nullptr
  double V[MAXN1 * (MAXN1 - 1)];  // RESPR: fine x coarse p-transfer matrix, row-major
};

__device__ __forceinline__ long long hblk(int nx, int i, int j) { return (long long)(j - 1) * nx + i; }
__device__ __forceinline__ long long vblk(long long nh, int ny, int i, int j) {
  return nh + (long long)(i - 1) * ny + j;
}

// streaming load of operator data: read once per apply, so keep it out of L1 and mark it
// evict-first in L2 (x, which IS re-read by neighbouring tiles, keeps the L2)
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

template <int N1>
__device__ __forceinline__ void stage_tile(const MvArgs& a, double* Hs, double* Vs, int i0, int j0) {
  using C = Cfg<N1>;
  constexpr int HROW = C::HCOLS * N1;
  for (int t = threadIdx.x; t < C::HROWS * HROW; t += NT) {
    const int jj = t / HROW, r = t - jj * HROW;
    const int ii = r / N1, m = r - ii * N1;
    const int i = i0 - 1 + ii, j = j0 - 1 + jj;
    double v = 0.0;
    if (j >= 1 && j <= a.ny - 1 && i >= 0 && i < a.nx) v = __ldg(a.x + hblk(a.nx, i, j) * N1 + m);
    Hs[(jj * C::HCOLS + ii) * C::S + m] = v;
  }
  constexpr int VCOL = C::VROWS * N1;
  for (int t = threadIdx.x; t < C::VCOLS * VCOL; t += NT) {
    const int ii = t / VCOL, r = t - ii * VCOL;
    const int jj = r / N1, m = r - jj * N1;
    const int i = i0 - 1 + ii, j = j0 - 1 + jj;
    double v = 0.0;
    if (i >= 1 && i <= a.nx - 1 && j >= 0 && j < a.ny) v = __ldg(a.x + vblk(a.nh, a.ny, i, j) * N1 + m);
    Vs[(ii * C::VROWS + jj) * C::S + m] = v;
  }
}

// acc = W_f . [x of the 7 stencil blocks];  W from constant bank (shared) or streamed (stored)
template <int N1, bool STORED>
__device__ __forceinline__ void facet_apply(const double* const* nb, const double* Wc, const double* Ws,
                                            double (&acc)[N1]) {
  using C = Cfg<N1>;
#pragma unroll
  for (int k = 0; k < N1; ++k) acc[k] = 0.0;
  if constexpr (!STORED) {
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      double xv[N1];
#pragma unroll
      for (int m = 0; m < N1; ++m) xv[m] = nb[q][m];
#pragma unroll
      for (int k = 0; k < N1; ++k)
#pragma unroll
        for (int m = 0; m < N1; ++m) acc[k] = fma(Wc[(q * N1 + k) * N1 + m], xv[m], acc[k]);
    }
  } else {
    const uint64_t pol = evict_first_policy();
#pragma unroll (C::QUNROLL)
    for (int q = 0; q < 7; ++q) {
      double xv[N1];
#pragma unroll
      for (int m = 0; m < N1; ++m) xv[m] = nb[q][m];
      const double* Wq = Ws + (size_t)q * N1 * N1 * 32;
#pragma unroll
      for (int k = 0; k < N1; ++k)
#pragma unroll
        for (int m = 0; m < N1; ++m) acc[k] = fma(ld_stream(Wq + (k * N1 + m) * 32, pol), xv[m], acc[k]);
    }
  }
}

template <int N1, bool STORED, int EPI>
__device__ __forceinline__ void facet_epilogue(const MvArgs& a, long long blk, const double* xf,
                                               const double* Dc, const double* Ds, const double (&acc)[N1],
                                               double& nrm) {
  if constexpr (EPI == EPI_Y) {
#pragma unroll
    for (int k = 0; k < N1; ++k) a.out[blk * N1 + k] = acc[k];
  } else {
    double r[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) r[k] = __ldg(a.b + blk * N1 + k) - acc[k];
    if constexpr (EPI == EPI_RES) {
#pragma unroll
      for (int k = 0; k < N1; ++k) nrm = fma(r[k], r[k], nrm);
      if (a.out != nullptr) {
#pragma unroll
        for (int k = 0; k < N1; ++k) a.out[blk * N1 + k] = r[k];
      }
    } else if constexpr (EPI == EPI_BJ) {
      double dinv[N1 * N1];
      if constexpr (!STORED) {
#pragma unroll
        for (int t = 0; t < N1 * N1; ++t) dinv[t] = Dc[t];
      } else {
#pragma unroll
        const uint64_t pol = evict_first_policy();
#pragma unroll
        for (int t = 0; t < N1 * N1; ++t) dinv[t] = ld_stream(Ds + (size_t)t * 32, pol);
      }
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) s = fma(dinv[k * N1 + m], r[m], s);
        a.out[blk * N1 + k] = fma(a.omega, s, xf[k]);
      }
    } else {  // EPI_RESPR: r_coarse = V^T r  (multigrid.py:399, p-level)
      constexpr int NC = N1 - 1;
#pragma unroll
      for (int c = 0; c < (NC > 0 ? NC : 1); ++c) {
        if (c < NC) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < N1; ++k) s = fma(a.V[k * NC + c], r[k], s);
          a.out[blk * NC + c] = s;
        }
      }
    }
  }
}

template <int N1, bool STORED, int EPI>
__global__ void __launch_bounds__(NT)
trace_apply_kernel(const MvArgs a, const __grid_constant__ SharedOp<(STORED ? 1 : N1)> op) {
  using C = Cfg<N1>;
  extern __shared__ double smem[];
  double* Hs = smem;
  double* Vs = smem + C::HROWS * C::HCOLS * C::S;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  stage_tile<N1>(a, Hs, Vs, i0, j0);
  __syncthreads();

  const int tx = threadIdx.x & (TX - 1), ty = threadIdx.x / TX;
  const int i = i0 + tx, j = j0 + ty;
  const int ii = tx + 1, jj = ty + 1;
  auto H = [&](int r, int c) { return Hs + (r * C::HCOLS + c) * C::S; };
  auto V = [&](int c, int r) { return Vs + (c * C::VROWS + r) * C::S; };
  double nrm = 0.0;
  const double* Wc_h = nullptr; const double* Wc_v = nullptr;
  const double* Dc_h = nullptr; const double* Dc_v = nullptr;
  if constexpr (!STORED) { Wc_h = op.Wh; Wc_v = op.Wv; Dc_h = op.Dh; Dc_v = op.Dv; }
  const long long grp_off = (((long long)j * a.nxp + i0) >> 5);  // warp group of this row segment

  // horizontal facet h(i, j): owners (i, j-1) [TOP rows] and (i, j) [BOTTOM rows]
  if (i < a.nx && j >= 1 && j <= a.ny - 1) {
    const double* nb[7] = {H(jj - 1, ii), H(jj, ii), H(jj + 1, ii),
                           V(ii, jj - 1), V(ii + 1, jj - 1), V(ii, jj), V(ii + 1, jj)};
    double acc[N1];
    const double* Ws = nullptr; const double* Ds = nullptr;
    if constexpr (STORED) {
      Ws = a.Wh + (size_t)grp_off * C::WSZ * 32 + tx;
      if constexpr (EPI == EPI_BJ) Ds = a.Dh + (size_t)grp_off * C::DSZ * 32 + tx;
    }
    facet_apply<N1, STORED>(nb, Wc_h, Ws, acc);
    facet_epilogue<N1, STORED, EPI>(a, hblk(a.nx, i, j), H(jj, ii), Dc_h, Ds, acc, nrm);
  }
  // vertical facet v(i, j): owners (i-1, j) [RIGHT rows] and (i, j) [LEFT rows]
  if (i >= 1 && i <= a.nx - 1 && j < a.ny) {
    const double* nb[7] = {V(ii - 1, jj), V(ii, jj), V(ii + 1, jj),
                           H(jj, ii - 1), H(jj + 1, ii - 1), H(jj, ii), H(jj + 1, ii)};
    double acc[N1];
    const double* Ws = nullptr; const double* Ds = nullptr;
    if constexpr (STORED) {
      Ws = a.Wv + (size_t)grp_off * C::WSZ * 32 + tx;
      if constexpr (EPI == EPI_BJ) Ds = a.Dv + (size_t)grp_off * C::DSZ * 32 + tx;
    }
    facet_apply<N1, STORED>(nb, Wc_v, Ws, acc);
    facet_epilogue<N1, STORED, EPI>(a, vblk(a.nh, a.ny, i, j), V(ii, jj), Dc_v, Ds, acc, nrm);
  }

  if constexpr (EPI == EPI_RES) {
    if (a.partials != nullptr) {
      __shared__ double red[NT / 32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < NT / 32; ++w) s += red[w];
        a.partials[blockIdx.y * gridDim.x + blockIdx.x] = s;
      }
    }
  }
}

// ---------------------------------------------------------------------------------- setup
// Element blocks (E, 4n1, 4n1) [trace.py:54] -> facet-merged, facet-interleaved stream.
// Stencil order  h: [h(i,j-1), h(i,j), h(i,j+1), v(i,j-1), v(i+1,j-1), v(i,j), v(i+1,j)]
//                v: [v(i-1,j), v(i,j), v(i+1,j), h(i-1,j), h(i-1,j+1), h(i,j), h(i,j+1)]
__host__ __device__ inline void merged_entry_src(bool vert, int q, int k, int m, int n1, int& which,
                                                 int& row, int& col, int& which2, int& row2, int& col2) {
  // which: 0 = first owner, 1 = second owner; which2 = -1 unless the entry is a sum
  which2 = -1; row2 = col2 = 0;
  if (!vert) {
    const int r1 = 2 * n1 + k, r2 = k;  // TOP rows of (i,j-1), BOTTOM rows of (i,j)
    switch (q) {
      case 0: which = 0; row = r1; col = 0 * n1 + m; break;
      case 1: which = 0; row = r1; col = 2 * n1 + m; which2 = 1; row2 = r2; col2 = 0 * n1 + m; break;
      case 2: which = 1; row = r2; col = 2 * n1 + m; break;
      case 3: which = 0; row = r1; col = 3 * n1 + m; break;
      case 4: which = 0; row = r1; col = 1 * n1 + m; break;
      case 5: which = 1; row = r2; col = 3 * n1 + m; break;
      default: which = 1; row = r2; col = 1 * n1 + m; break;
    }
  } else {
    const int r1 = 1 * n1 + k, r2 = 3 * n1 + k;  // RIGHT rows of (i-1,j), LEFT rows of (i,j)
    switch (q) {
      case 0: which = 0; row = r1; col = 3 * n1 + m; break;
      case 1: which = 0; row = r1; col = 1 * n1 + m; which2 = 1; row2 = r2; col2 = 3 * n1 + m; break;
      case 2: which = 1; row = r2; col = 1 * n1 + m; break;
      case 3: which = 0; row = r1; col = 0 * n1 + m; break;
      case 4: which = 0; row = r1; col = 2 * n1 + m; break;
      case 5: which = 1; row = r2; col = 0 * n1 + m; break;
      default: which = 1; row = r2; col = 2 * n1 + m; break;
    }
  }
}

template <int N1>
__global__ void relayout_kernel(const double* __restrict__ S, int nx, int ny, int nxp, bool vert,
                                double* __restrict__ W) {
  using C = Cfg<N1>;
  const long long nslots = (long long)ny * nxp;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= nslots * C::WSZ) return;
  // thread -> (group, entry, lane): consecutive threads write consecutive addresses
  const int lane = tid & 31;
  const long long rest = tid >> 5;
  const int idx = (int)(rest % C::WSZ);
  const long long grp = rest / C::WSZ;
  const long long slot = grp * 32 + lane;
  const int j = (int)(slot / nxp), i = (int)(slot % nxp);
  const bool valid = vert ? (i >= 1 && i <= nx - 1 && j < ny) : (i < nx && j >= 1 && j <= ny - 1);
  long long e1 = 0, e2 = 0;
  if (valid) {
    e1 = vert ? ((long long)j * nx + (i - 1)) : ((long long)(j - 1) * nx + i);
    e2 = (long long)j * nx + i;
  }
  const int L = 4 * N1;
  const int q = idx / (N1 * N1), k = (idx / N1) % N1, m = idx % N1;
  double v = 0.0;
  if (valid) {
    int w1, r1, c1, w2, r2, c2;
    merged_entry_src(vert, q, k, m, N1, w1, r1, c1, w2, r2, c2);
    v = S[((w1 ? e2 : e1) * L + r1) * L + c1];
    if (w2 >= 0) v += S[((w2 ? e2 : e1) * L + r2) * L + c2];
  }
  W[(grp * C::WSZ + idx) * 32 + lane] = v;
}

// In-place inverse of SPD n1 x n1 blocks held in the interleaved layout (Gauss-Jordan, no
// pivoting: the blocks are principal submatrices of an SPD operator).  Padding slots hold
// zero blocks; they are replaced by the identity so no inf/NaN is ever stored.
template <int N1>
__global__ void invert_kernel(double* __restrict__ D, long long nslots) {
  using C = Cfg<N1>;
  const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nslots) return;
  const long long grp = slot >> 5;
  const int lane = slot & 31;
  double a[N1 * N1];
  auto at = [&](int idx) -> double& { return D[(grp * C::DSZ + idx) * 32 + lane]; };
  for (int t = 0; t < N1 * N1; ++t) a[t] = at(t);
  if (a[0] == 0.0) {
    for (int t = 0; t < N1 * N1; ++t) at(t) = (t / N1 == t % N1) ? 1.0 : 0.0;
    return;
  }
  for (int c = 0; c < N1; ++c) {
    const double piv = 1.0 / a[c * N1 + c];
    for (int m = 0; m < N1; ++m) a[c * N1 + m] *= piv;
    a[c * N1 + c] = piv;
    for (int r = 0; r < N1; ++r) {
      if (r == c) continue;
      const double f = a[r * N1 + c];
      a[r * N1 + c] = 0.0;
      for (int m = 0; m < N1; ++m) a[r * N1 + m] -= f * a[c * N1 + m];
      a[r * N1 + c] = -f * piv;
    }
  }
  for (int t = 0; t < N1 * N1; ++t) at(t) = a[t];
}

// ------------------------------------------------------------------------------ transfers
// p-transfer, facet-local (multigrid.py:215-219): x_f += V e_c ; r_c = V^T r_f
struct PArgs { double V[MAXN1 * (MAXN1 - 1)]; };

template <int N1>
__global__ void p_prolong_add_kernel(const double* __restrict__ ec, double* __restrict__ xf,
                                     long long nblocks, const PArgs a) {
  constexpr int NC = N1 - 1;
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  double e[NC > 0 ? NC : 1];
#pragma unroll
  for (int c = 0; c < NC; ++c) e[c] = __ldg(ec + b * NC + c);
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) s = fma(a.V[k * NC + c], e[c], s);
    xf[b * N1 + k] += s;
  }
}

template <int N1>
__global__ void p_restrict_kernel(const double* __restrict__ rf, double* __restrict__ rc,
                                  long long nblocks, const PArgs a) {
  constexpr int NC = N1 - 1;
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  double r[N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) r[k] = __ldg(rf + b * N1 + k);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N1; ++k) s = fma(a.V[k * NC + c], r[k], s);
    rc[b * NC + c] = s;
  }
}

// h-transfer at p = 1 (multigrid.py:229-298).  halves[h][k][c]; cross[set][cf][k][s*2+c]
struct HArgs {
  int nxc, nyc;           // coarse mesh
  long long nhf, nhc;     // interior horizontal block counts (fine, coarse)
  double halves[8];
  const double* cross;    // device, (nsets, 4, 2, 8)
  int shared_cross;       // 1 => one set for every coarse element
};

__device__ __forceinline__ const double* hcross(const HArgs& h, int I, int J, int cf) {
  const long long set = h.shared_cross ? 0 : ((long long)J * h.nxc + I);
  return h.cross + (set * 4 + cf) * 16;
}

// coarse side value (2 doubles) of coarse element (I, J), side s; zero when Dirichlet
__device__ __forceinline__ void coarse_side(const HArgs& h, const double* ec, int I, int J, int s, double* v) {
  long long blk = -1;
  if (s == 0 && J >= 1) blk = (long long)(J - 1) * h.nxc + I;
  if (s == 2 && J + 1 <= h.nyc - 1) blk = (long long)J * h.nxc + I;
  if (s == 3 && I >= 1) blk = h.nhc + (long long)(I - 1) * h.nyc + J;
  if (s == 1 && I + 1 <= h.nxc - 1) blk = h.nhc + (long long)I * h.nyc + J;
  if (blk >= 0) { v[0] = __ldg(ec + 2 * blk); v[1] = __ldg(ec + 2 * blk + 1); }
  else { v[0] = 0.0; v[1] = 0.0; }
}

__global__ void h_prolong_add_kernel(const HArgs h, const double* __restrict__ ec, double* __restrict__ xf) {
  const int nxf = 2 * h.nxc, nyf = 2 * h.nyc;
  const long long nvf = (long long)(nxf - 1) * nyf;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= h.nhf + nvf) return;
  double add[2] = {0.0, 0.0};
  if (t < h.nhf) {  // fine h(i, j), block (j-1)*nxf + i
    const int j = (int)(t / nxf) + 1, i = (int)(t % nxf);
    const int I = i >> 1;
    if ((j & 1) == 0) {
      const int J = j >> 1, hf = i & 1;
      const long long cb = (long long)(J - 1) * h.nxc + I;
      const double e0 = __ldg(ec + 2 * cb), e1 = __ldg(ec + 2 * cb + 1);
      for (int k = 0; k < 2; ++k) add[k] = h.halves[hf * 4 + k * 2] * e0 + h.halves[hf * 4 + k * 2 + 1] * e1;
    } else {
      const int J = (j - 1) >> 1, cf = (i & 1) ? 3 : 2;
      const double* tm = hcross(h, I, J, cf);
      for (int s = 0; s < 4; ++s) {
        double v[2];
        coarse_side(h, ec, I, J, s, v);
        for (int k = 0; k < 2; ++k) add[k] += tm[k * 8 + s * 2] * v[0] + tm[k * 8 + s * 2 + 1] * v[1];
      }
    }
  } else {  // fine v(i, j), block nhf + (i-1)*nyf + j
    const long long u = t - h.nhf;
    const int i = (int)(u / nyf) + 1, j = (int)(u % nyf);
    const int J = j >> 1;
    if ((i & 1) == 0) {
      const int I = i >> 1, hf = j & 1;
      const long long cb = h.nhc + (long long)(I - 1) * h.nyc + J;
      const double e0 = __ldg(ec + 2 * cb), e1 = __ldg(ec + 2 * cb + 1);
      for (int k = 0; k < 2; ++k) add[k] = h.halves[hf * 4 + k * 2] * e0 + h.halves[hf * 4 + k * 2 + 1] * e1;
    } else {
      const int I = (i - 1) >> 1, cf = (j & 1) ? 1 : 0;
      const double* tm = hcross(h, I, J, cf);
      for (int s = 0; s < 4; ++s) {
        double v[2];
        coarse_side(h, ec, I, J, s, v);
        for (int k = 0; k < 2; ++k) add[k] += tm[k * 8 + s * 2] * v[0] + tm[k * 8 + s * 2 + 1] * v[1];
      }
    }
  }
  xf[2 * t] += add[0];
  xf[2 * t + 1] += add[1];
}

// contribution of coarse element (I, J)'s 4 cross facets to its side-s coarse dofs
__device__ __forceinline__ void cross_restrict(const HArgs& h, const double* rf, int I, int J, int s, double* acc) {
  const int nxf = 2 * h.nxc, nyf = 2 * h.nyc;
  const long long cfb[4] = {
      h.nhf + (long long)(2 * I + 1 - 1) * nyf + 2 * J,       // right of SW = v(2I+1, 2J)
      h.nhf + (long long)(2 * I + 1 - 1) * nyf + 2 * J + 1,   // right of NW = v(2I+1, 2J+1)
      (long long)(2 * J + 1 - 1) * nxf + 2 * I,               // top of SW   = h(2I, 2J+1)
      (long long)(2 * J + 1 - 1) * nxf + 2 * I + 1};          // top of SE   = h(2I+1, 2J+1)
  for (int cf = 0; cf < 4; ++cf) {
    const double* tm = hcross(h, I, J, cf);
    const double r0 = __ldg(rf + 2 * cfb[cf]), r1 = __ldg(rf + 2 * cfb[cf] + 1);
    for (int c = 0; c < 2; ++c) acc[c] += tm[0 * 8 + s * 2 + c] * r0 + tm[1 * 8 + s * 2 + c] * r1;
  }
}

__global__ void h_restrict_kernel(const HArgs h, const double* __restrict__ rf, double* __restrict__ rc) {
  const int nxf = 2 * h.nxc, nyf = 2 * h.nyc;
  const long long nvc = (long long)(h.nxc - 1) * h.nyc;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= h.nhc + nvc) return;
  double acc[2] = {0.0, 0.0};
  long long k0;
  if (t < h.nhc) {  // coarse h(I, J)
    const int J = (int)(t / h.nxc) + 1, I = (int)(t % h.nxc);
    k0 = (long long)(2 * J - 1) * nxf + 2 * I;  // fine h(2I, 2J); +1 is h(2I+1, 2J)
    for (int hf = 0; hf < 2; ++hf) {
      const double r0 = __ldg(rf + 2 * (k0 + hf)), r1 = __ldg(rf + 2 * (k0 + hf) + 1);
      for (int c = 0; c < 2; ++c) acc[c] += h.halves[hf * 4 + 0 * 2 + c] * r0 + h.halves[hf * 4 + 1 * 2 + c] * r1;
    }
    cross_restrict(h, rf, I, J - 1, 2, acc);  // element below: this facet is its TOP side
    cross_restrict(h, rf, I, J, 0, acc);      // element above: BOTTOM side
  } else {          // coarse v(I, J)
    const long long u = t - h.nhc;
    const int I = (int)(u / h.nyc) + 1, J = (int)(u % h.nyc);
    k0 = h.nhf + (long long)(2 * I - 1) * nyf + 2 * J;  // fine v(2I, 2J); +1 is v(2I, 2J+1)
    for (int hf = 0; hf < 2; ++hf) {
      const double r0 = __ldg(rf + 2 * (k0 + hf)), r1 = __ldg(rf + 2 * (k0 + hf) + 1);
      for (int c = 0; c < 2; ++c) acc[c] += h.halves[hf * 4 + 0 * 2 + c] * r0 + h.halves[hf * 4 + 1 * 2 + c] * r1;
    }
    cross_restrict(h, rf, I - 1, J, 1, acc);  // element left: RIGHT side
    cross_restrict(h, rf, I, J, 3, acc);      // element right: LEFT side
  }
  rc[2 * t] = acc[0];
  rc[2 * t + 1] = acc[1];
}

// ---------------------------------------------------------------------------- small kernels
// dense y = M b, warp per row (coarsest level, multigrid.py:209-212)
__global__ void dense_gemv_kernel(const double* __restrict__ M, const double* __restrict__ b,
                                  double* __restrict__ y, int n) {
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s = fma(__ldg(M + (size_t)row * n + c), __ldg(b + c), s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

// deterministic dot: fixed grid, per-CTA partials, then one CTA sums them in order
__global__ void dot_partials_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
                                    double* __restrict__ partials) {
  double s = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    s = fma(__ldg(a + t), __ldg(b + t), s);
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    partials[blockIdx.x] = t;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ partials, int n, double* __restrict__ out) {
  // one warp; fixed order => bitwise deterministic
  double s = 0.0;
  for (int t = threadIdx.x; t < n; t += 32) s += partials[t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *out = s;
}

// CG vector updates (trace.py:156-161): x += a d, r -= a ad ;  d = z + beta d
__global__ void cg_update_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ d,
                                 const double* __restrict__ ad, double alpha, long long n) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    x[t] = fma(alpha, d[t], x[t]);
    r[t] = fma(-alpha, ad[t], r[t]);
  }
}

__global__ void xpby_kernel(const double* __restrict__ z, double beta, double* __restrict__ d, long long n) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    d[t] = fma(beta, d[t], z[t]);
}

}  // namespace hdg
