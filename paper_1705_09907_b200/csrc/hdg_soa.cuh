// hdg_soa.cuh - element-column streaming trace apply in the facet-plane (SoA) device layout.
//
// Same operator as trace_apply_kernel (TraceSystem.matvec_free, trace.py:87-94: gather the 4
// facets of each element, y_e = S x_e, sum the two owners of every facet), organised for the
// B200 memory system instead of for the reference's [facet][node] layout:
//
//   Device layout ("facet planes"): node k of every horizontal facet line r (r = 0..ny, the
//   boundary lines 0 and ny included as zeros) is one contiguous run over the element columns,
//   H[k][r][slot], slot = column + 1; vertical facets are stored by element row,
//   V[k][r][slot], slot = line + 1 (line 0 and nx are boundary zeros).  The pitch
//   P = even(31 W + 4) (W = column warps) keeps zero pad slots on both sides, so every load is
//   one unpredicated 16-byte-aligned bulk copy (TMA) of 34 doubles per node plane and row.
//
//   One warp walks a vertical segment of 32 element columns (lane = column); warps overlap by one
//   column (31 owned).  Per element row the warp's lanes 0 .. 2 N1 - 1 issue one bulk copy each
//   (node k of the H line above and of the V facets of the row: 34 consecutive slots) into a
//   per-warp ring of RING entries completed on mbarriers, RING - 2 rows ahead; each lane then
//   reads its four facets from the ring (bottom = the previous entry's H run).  The element product
//   runs in the symmetry-adapted basis of the square element (mirrors x -> 1-x and y -> 1-y
//   commute with S for a constant coefficient on a uniform mesh): sum/difference butterflies
//   split the 4 n1 element values into four classes and S becomes four dense blocks
//   (2h)^2 + 2 n1^2 + (2l)^2 FMAs, h = ceil(n1/2), l = floor(n1/2): 102 instead of 400 at p = 4.
//   Facet sums: the top part of row r-1 stays in registers for the bottom part of row r; the
//   right part of a lane meets the left part of lane+1 by shuffle.  Every slot of y is written
//   exactly once (boundary and pad slots as zeros), so y is a valid input of the next apply.
//   No shared memory, no atomics, no grid synchronisation: one writer per facet (trace.py:3-7).
//
//   A segment of J element rows starts with one ghost row (its top part feeds the first
//   horizontal line the segment owns): (J+1)/J compute, the extra loads are L2 hits.
#pragma once
#include <cuda_runtime.h>

#include "hdg_kernels.cuh"   // cp_async8 / cp_async_commit / cp_async_wait

#ifndef HDG_SOA_EXP
#define HDG_SOA_EXP 0          // experiment flags (tools/build_variants.sh), 0 in the product
#endif
#ifndef HDG_SOA_ALT
#define HDG_SOA_ALT 0          // experiment: alternate the walk direction of neighbouring segments
#endif
#ifndef HDG_SOA_STCS
#define HDG_SOA_STCS 0         // experiment: streaming (evict-first) stores of y
#endif
#ifndef HDG_SOA_VW
#define HDG_SOA_VW 34          // V row width of a facet record (36: 32-byte aligned records)
#endif
#ifndef HDG_SOA_RING
#define HDG_SOA_RING 3
#endif
#ifndef HDG_SOA_MCONST
#define HDG_SOA_MCONST -1      // blocks from the constant bank (1) or shared memory (0); -1: by order
                               // (constant bank for p <= 4: 36.7 vs 37.3 us at 1024^2; at p = 8
                               // the 326 entries overflow the uniform registers: 264 vs 220 us)
#endif
#ifndef HDG_SOA_MINB_HI
#define HDG_SOA_MINB_HI 3      // CTAs per SM for p >= 3 (154 registers at p = 4 without a cap)
#endif

namespace hdg {

template <int N1>
struct SoaCfg {
  static constexpr int H = (N1 + 1) / 2, L = N1 / 2;
  static constexpr int A0 = 2 * H, A1 = N1, A2 = N1, A3 = 2 * L;   // class sizes
  static constexpr int MSZ = A0 * A0 + A1 * A1 + A2 * A2 + A3 * A3;
  static constexpr int NTH = 128;
  static constexpr int MINB = N1 <= 3 ? 4 : HDG_SOA_MINB_HI;
  static constexpr int RING = HDG_SOA_RING;              // ring entries per warp (RING-2 rows in flight)
  static constexpr int VW = HDG_SOA_VW;                  // V row width (34: slots 0..33)
  static constexpr int ENT = N1 * (32 + VW);             // record: H[N1][32] + V[N1][VW] doubles
  static constexpr int WSTRIDE = (RING * ENT + RING + 1) & ~1;   // doubles per warp (16-byte multiple)
  static constexpr int SMEM_RING = (NTH / 32) * WSTRIDE * 8;
};

template <int N1>
struct SoaArgs {
  const double* x;
  double* y;
  int nx, ny, W, J, nseg;
  double M[SoaCfg<N1>::MSZ];        // symmetry-adapted blocks, row-major, classes 0..3
};

// forward butterflies: local values (B, R, T, L) -> class vectors t0 | t1 | t2 | t3
template <int N1>
__host__ __device__ __forceinline__ void soa_forward(const double* xB, const double* xR, const double* xT,
                                                     const double* xL, double* t) {
  using C = SoaCfg<N1>;
  constexpr int H = C::H, L = C::L;
  double* t0 = t;
  double* t1 = t + C::A0;
  double* t2 = t1 + C::A1;
  double* t3 = t2 + C::A2;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const int q = N1 - 1 - k;
    const double ak = xL[k] + xR[k], aq = xL[q] + xR[q];
    const double bk = xL[k] - xR[k], bq = xL[q] - xR[q];
    const double ck = xB[k] + xT[k], cq = xB[q] + xT[q];
    const double dk = xB[k] - xT[k], dq = xB[q] - xT[q];
    t0[k] = ak + aq;      // a+
    t0[H + k] = ck + cq;  // c+
    t1[k] = ak - aq;      // a-
    t1[L + k] = dk + dq;  // d+
    t2[k] = bk + bq;      // b+
    t2[H + k] = ck - cq;  // c-
    t3[k] = bk - bq;      // b-
    t3[L + k] = dk - dq;  // d-
  }
  if (N1 & 1) {
    t0[L] = xL[L] + xR[L];
    t0[H + L] = xB[L] + xT[L];
    t1[L + L] = xB[L] - xT[L];
    t2[L] = xL[L] - xR[L];
  }
}

// inverse (transposed) butterflies: class vectors -> local values (B, R, T, L)
template <int N1>
__host__ __device__ __forceinline__ void soa_backward(const double* t, double* yB, double* yR, double* yT,
                                                      double* yL) {
  using C = SoaCfg<N1>;
  constexpr int H = C::H, L = C::L;
  const double* t0 = t;
  const double* t1 = t + C::A0;
  const double* t2 = t1 + C::A1;
  const double* t3 = t2 + C::A2;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const int q = N1 - 1 - k;
    const double ak = t0[k] + t1[k], aq = t0[k] - t1[k];
    const double bk = t2[k] + t3[k], bq = t2[k] - t3[k];
    const double ck = t0[H + k] + t2[H + k], cq = t0[H + k] - t2[H + k];
    const double dk = t1[L + k] + t3[L + k], dq = t1[L + k] - t3[L + k];
    yL[k] = ak + bk; yR[k] = ak - bk; yL[q] = aq + bq; yR[q] = aq - bq;
    yB[k] = ck + dk; yT[k] = ck - dk; yB[q] = cq + dq; yT[q] = cq - dq;
  }
  if (N1 & 1) {
    const double a = t0[L], b = t2[L], c = t0[H + L], d = t1[L + L];
    yL[L] = a + b; yR[L] = a - b; yB[L] = c + d; yT[L] = c - d;
  }
}

// The blocks live in shared memory as packed upper triangles (M is symmetric: S is, and the
// butterflies are scaled symmetrically), each block padded to an even length and read as LDS.128
// broadcasts; every stored entry feeds two FMAs.  Held in registers they would pin ~200
// registers per thread for the whole loop.
template <int SZ>
struct SoaTri { static constexpr int N = SZ * (SZ + 1) / 2, NP = (N + 1) & ~1; };

template <int N1>
struct SoaSmem {
  using C = SoaCfg<N1>;
  static constexpr int O0 = 0;
  static constexpr int O1 = O0 + SoaTri<C::A0>::NP;
  static constexpr int O2 = O1 + SoaTri<C::A1>::NP;
  static constexpr int O3 = O2 + SoaTri<C::A2>::NP;
  static constexpr int TOTAL = O3 + SoaTri<C::A3>::NP;   // doubles (even)
};

template <int N1>
constexpr int soa_smem_bytes() { return SoaSmem<N1>::TOTAL * 8 + SoaCfg<N1>::SMEM_RING; }

// packed index of (i, j), i <= j, row-major upper triangle
template <int SZ>
__host__ __device__ constexpr int soa_tri(int i, int j) { return i * SZ - i * (i - 1) / 2 + (j - i); }

template <int SZ, int SOFF, int TOFF>
__device__ __forceinline__ void soa_block(const double* __restrict__ Ms, const double* t, double* z) {
  constexpr int NP = SoaTri<SZ>::NP;
  double m[NP];
#pragma unroll
  for (int q = 0; q < NP / 2; ++q) {
    const double2 v = reinterpret_cast<const double2*>(Ms + SOFF)[q];
    m[2 * q] = v.x;
    m[2 * q + 1] = v.y;
  }
#pragma unroll
  for (int i = 0; i < SZ; ++i) z[TOFF + i] = m[soa_tri<SZ>(i, i)] * t[TOFF + i];
#pragma unroll
  for (int i = 0; i < SZ; ++i)
#pragma unroll
    for (int j = i + 1; j < SZ; ++j) {
      const double v = m[soa_tri<SZ>(i, j)];
      z[TOFF + i] = fma(v, t[TOFF + j], z[TOFF + i]);
      z[TOFF + j] = fma(v, t[TOFF + i], z[TOFF + j]);
    }
}

template <int N1>
__device__ __forceinline__ void soa_blocks(const double* __restrict__ Ms, const double* t, double* z) {
  using C = SoaCfg<N1>;
  using M = SoaSmem<N1>;
  soa_block<C::A0, M::O0, 0>(Ms, t, z);
  soa_block<C::A1, M::O1, C::A0>(Ms, t, z);
  soa_block<C::A2, M::O2, C::A0 + C::A1>(Ms, t, z);
  soa_block<C::A3, M::O3, C::A0 + C::A1 + C::A2>(Ms, t, z);
}

// The same product with the blocks read from the kernel-parameter (constant) bank: every lane
// uses the same entry at the same time, so DFMA takes it as a uniform c[][] operand and the
// shared-memory pipe carries only the ring.
template <int SZ, int MOFF, int TOFF>
__device__ __forceinline__ void soa_block_c(const double* M, const double* t, double* z) {
#pragma unroll
  for (int i = 0; i < SZ; ++i) z[TOFF + i] = M[MOFF + i * SZ + i] * t[TOFF + i];
#pragma unroll
  for (int i = 0; i < SZ; ++i)
#pragma unroll
    for (int j = i + 1; j < SZ; ++j) {
      const double v = M[MOFF + i * SZ + j];
      z[TOFF + i] = fma(v, t[TOFF + j], z[TOFF + i]);
      z[TOFF + j] = fma(v, t[TOFF + i], z[TOFF + j]);
    }
}

template <int N1>
__device__ __forceinline__ void soa_blocks_c(const double* M, const double* t, double* z) {
  using C = SoaCfg<N1>;
  constexpr int M1 = C::A0 * C::A0, M2 = M1 + C::A1 * C::A1, M3 = M2 + C::A2 * C::A2;
  soa_block_c<C::A0, 0, 0>(M, t, z);
  soa_block_c<C::A1, M1, C::A0>(M, t, z);
  soa_block_c<C::A2, M2, C::A0 + C::A1>(M, t, z);
  soa_block_c<C::A3, M3, C::A0 + C::A1 + C::A2>(M, t, z);
}

// a.M (dense class blocks, row-major, symmetric) -> packed upper triangles in shared memory
template <int N1>
__device__ __forceinline__ void soa_load_blocks(const SoaArgs<N1>& a, double* Ms) {
  using C = SoaCfg<N1>;
  using M = SoaSmem<N1>;
  constexpr int sz[4] = {C::A0, C::A1, C::A2, C::A3};
  constexpr int so[5] = {M::O0, M::O1, M::O2, M::O3, M::TOTAL};
  for (int idx = threadIdx.x; idx < M::TOTAL; idx += blockDim.x) {
    int c = 0;
    while (c < 3 && idx >= so[c + 1]) ++c;
    const int n = sz[c], q = idx - so[c];
    int mo = 0;
    for (int u = 0; u < c; ++u) mo += sz[u] * sz[u];
    double v = 0.0;
    if (q < n * (n + 1) / 2) {
      int i = 0, rem = q;
      while (rem >= n - i) { rem -= n - i; ++i; }
      v = a.M[mo + i * n + i + rem];
    }
    Ms[idx] = v;
  }
}

template <int N1, int MCONST = (HDG_SOA_MCONST < 0 ? (N1 <= 5) : HDG_SOA_MCONST)>
__global__ void __launch_bounds__(SoaCfg<N1>::NTH, SoaCfg<N1>::MINB)
    soa_apply_kernel(const __grid_constant__ SoaArgs<N1> a) {
  constexpr int NT = 4 * N1, RING = SoaCfg<N1>::RING, D = RING - 1;
  constexpr int ENT = SoaCfg<N1>::ENT;                 // doubles per record: H[N1][32] | V[N1][VW]
  constexpr int VW = SoaCfg<N1>::VW;
  constexpr int VOFF = N1 * 32;
  extern __shared__ __align__(16) double smem_soa[];
  double* Ms = smem_soa;
  if (!MCONST) {
    soa_load_blocks<N1>(a, Ms);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (SoaCfg<N1>::NTH / 32) + (threadIdx.x >> 5);
  if (gw >= a.W * a.nseg) return;                      // whole warps only
  double* ring = smem_soa + SoaSmem<N1>::TOTAL + (threadIdx.x >> 5) * SoaCfg<N1>::WSTRIDE;
  const int w = gw % a.W, seg = gw / a.W;
  const int c = 31 * w - 1 + lane;                     // element column of this lane
  const int r0 = seg * a.J;
  const int r1 = min(r0 + a.J, a.ny);
  const int rs = r0 > 0 ? r0 - 1 : 0;                  // ghost row feeds the first owned line
  const int nrows = r1 - rs;                           // element rows walked; records rs .. r1
  // odd segments walk down: both rows a segment shares with a neighbour (its ghost row and the
  // neighbour's ghost) are then read by the two warps at the same time (L2 hits, not DRAM)
  const bool down = HDG_SOA_ALT && (seg & 1);
  const double* __restrict__ X = a.x;
  double* __restrict__ Y = a.y;
  const long long W = a.W;
  auto rec = [&](int R, long long tile) { return (R * W + tile) * ENT; };   // record R, tile

  // ring entry t = record rs + t of this warp's tile (H line rs+t, V of element row rs+t-1): one
  // contiguous bulk copy (TMA) issued by lane 0, completion counted on the entry's mbarrier
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + RING * ENT);
  if (lane == 0) {
#pragma unroll
    for (int e = 0; e < RING; ++e) mbar_init(bars + e, 1);
  }
  fence_proxy_async();
  __syncwarp();
  auto issue = [&](int t) {
    if (t > nrows || lane != 0) return;
    uint64_t* bar = bars + (t % RING);
    mbar_arrive_expect_tx(bar, ENT * 8u);
    tma_load_1d(ring + (t % RING) * ENT, X + rec(down ? r1 - t : rs + t, w), ENT * 8u, bar);
  };
#pragma unroll
  for (int t = 0; t < D; ++t) issue(t);

  const bool hcol = c >= 0 && c < a.nx;
  const bool vline = c + 1 >= 1 && c + 1 <= a.nx - 1;
  // tp: the facet-sum partner carried between rows (walking up: T of the row below; down: B of
  // the row above); xC: the shared H line carried (up: next bottom; down: next top)
  double tp[N1], xC[N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) tp[k] = 0.0;

#pragma unroll 1
  for (int t = 0; t < nrows; ++t) {
    const int r = down ? r1 - 1 - t : rs + t;
    fence_proxy_async();                               // generic reads of entry t-1 before its async refill
    issue(t + D);                                      // entry t+D (slot of entry t-1: read last iteration)
    if (t == 0) mbar_wait(bars, 0);
    mbar_wait(bars + (t + 1) % RING, ((t + 1) / RING) & 1);
    // lower entry = record r (H line r), upper entry = record r + 1 (H line r+1, V of row r)
    const double* e0 = ring + ((down ? t + 1 : t) % RING) * ENT + lane;
    const double* e1 = ring + ((down ? t : t + 1) % RING) * ENT + lane;
    double xB[N1], xT[N1], xR[N1], xL[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      if (down) {
        xT[k] = t == 0 ? e1[k * 32] : xC[k];
        xB[k] = e0[k * 32];
      } else {
        xB[k] = t == 0 ? e0[k * 32] : xC[k];
        xT[k] = e1[k * 32];
      }
      xL[k] = e1[VOFF + k * VW];
      xR[k] = e1[VOFF + k * VW + 1];
    }
    double yB[N1], yR[N1], yT[N1], yL[N1];
#if HDG_SOA_EXP == 1   // experiment: no element product (memory path only)
#pragma unroll
    for (int k = 0; k < N1; ++k) { yB[k] = xB[k]; yR[k] = xR[k]; yT[k] = xT[k]; yL[k] = xL[k]; }
#else
    double tv[NT], z[NT];
    soa_forward<N1>(xB, xR, xT, xL, tv);
    if (MCONST) soa_blocks_c<N1>(a.M, tv, z);
    else soa_blocks<N1>(Ms, tv, z);
    soa_backward<N1>(z, yB, yR, yT, yL);
#endif
#if HDG_SOA_EXP == 2   // experiment: no stores unless the result is NaN (compute + loads only)
    if (yB[0] != yB[0] || yR[N1 - 1] != yR[N1 - 1])
#endif
    // H line written this row: up: line r = T(r-1) + B(r) (rows >= r0); down: line r+1 =
    // T(r) + B(r+1) (from the second row on; the ghost row r0 - 1 comes last and closes line r0)
    const int hl = down ? r + 1 : r;
    const bool hwr = down ? t >= 1 : r >= r0;
    if (hwr) {
      const bool hint = hcol && hl >= 1;
      double* hrec = Y + rec(hl, w);
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        const double hv = hint ? (down ? yT[k] + tp[k] : tp[k] + yB[k]) : 0.0;
#if HDG_SOA_STCS
        __stcs(hrec + k * 32 + lane, hv);
#else
        hrec[k * 32 + lane] = hv;                      // lane 0 duplicates the left tile's slot 31
#endif
      }
    }
    if (r >= r0) {
      double* vrec = Y + rec(r + 1, w) + VOFF;         // V of element row r
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        const double fromR = __shfl_down_sync(0xffffffffu, yL[k], 1);
        const double vv = (vline && lane != 31) ? yR[k] + fromR : 0.0;
#if HDG_SOA_STCS
        __stcs(vrec + k * VW + lane + 1 + (lane == 31), vv);
#else
        vrec[k * VW + lane + 1 + (lane == 31)] = vv;   // slots 1..31; lane 31 zeroes pad slot 33
#endif
        if (VW > 34 && lane == 31)
#pragma unroll
          for (int q = 34; q < VW; ++q) vrec[k * VW + q] = 0.0;
        if (lane == 30 && w + 1 < W) vrec[ENT + k * VW] = vv;         // duplicate: right tile slot 0
        if (lane == 0 && w > 0) vrec[-ENT + k * VW + 32] = vv;        // duplicate: left tile slot 32
        if (lane == 0 && w == 0) vrec[k * VW] = 0.0;                  // line -1 (pad)
        if (lane == 31 && w + 1 == W) vrec[k * VW + 32] = 0.0;        // line 31 W >= nx (pad)
      }
    }
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      tp[k] = down ? yB[k] : yT[k];
      xC[k] = down ? xB[k] : xT[k];
    }
    __syncwarp();                                      // entry t is free for issue(t + RING)
  }
  if (down && r0 == 0) {                               // bottom boundary line (down walk)
    double* hrec = Y + rec(0, w);
#pragma unroll
    for (int k = 0; k < N1; ++k) hrec[k * 32 + lane] = 0.0;
  }
  if (r1 == a.ny) {                                    // top boundary line
    double* hrec = Y + rec(a.ny, w);
#pragma unroll
    for (int k = 0; k < N1; ++k) hrec[k * 32 + lane] = 0.0;
  }
  if (r0 == 0) {                                       // V of element row -1 (pad record 0)
    double* vrec = Y + rec(0, w) + VOFF;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      vrec[k * VW + lane] = 0.0;
      if (lane < VW - 32) vrec[k * VW + 32 + lane] = 0.0;
    }
  }
}

// Record layout: record R (R = 0..ny) of tile w holds H line R (slot j = column 31 w - 1 + j,
// j < 32) and V of element row R - 1 (slot j = line 31 w - 1 + j, j < 34; slot 33 unused).
template <int N1>
__global__ void soa_pack_kernel(const double* __restrict__ x, double* __restrict__ xs, int nx, int ny, int W,
                                long long nh, long long total) {
  constexpr int ENT = SoaCfg<N1>::ENT, VOFF = N1 * 32;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const long long rw = t / ENT;
  const int o = (int)(t % ENT);
  const int R = (int)(rw / W), w = (int)(rw % W);
  double v = 0.0;
  if (o < VOFF) {
    const int k = o / 32, col = 31 * w - 1 + o % 32;
    if (R >= 1 && R <= ny - 1 && col >= 0 && col < nx) v = x[((long long)(R - 1) * nx + col) * N1 + k];
  } else {
    constexpr int VW = SoaCfg<N1>::VW;
    const int k = (o - VOFF) / VW, j = (o - VOFF) % VW, line = 31 * w - 1 + j, r = R - 1;
    if (j < 33 && r >= 0 && line >= 1 && line <= nx - 1) v = x[(nh + (long long)(line - 1) * ny + r) * N1 + k];
  }
  xs[t] = v;
}

template <int N1>
__global__ void soa_unpack_kernel(const double* __restrict__ xs, double* __restrict__ x, int nx, int ny, int W,
                                  long long nh, long long ndof) {
  constexpr int ENT = SoaCfg<N1>::ENT, VOFF = N1 * 32;
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= ndof) return;
  const long long blk = u / N1;
  const int k = (int)(u % N1);
  long long src;
  if (blk < nh) {
    const int R = (int)(blk / nx) + 1, col = (int)(blk % nx), w = col / 31;
    src = ((long long)R * W + w) * ENT + k * 32 + (col - 31 * w + 1);
  } else {
    const long long b = blk - nh;
    const int line = (int)(b / ny) + 1, r = (int)(b % ny), w = line / 31;
    src = ((long long)(r + 1) * W + w) * ENT + VOFF + k * SoaCfg<N1>::VW + (line - 31 * w + 1);
  }
  x[u] = xs[src];
}

}  // namespace hdg
