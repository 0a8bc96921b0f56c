// hdg_soa.cuh - element-column streaming trace apply in the facet-plane (SoA) device layout.
//
// Same operator as trace_apply_kernel (TraceSystem.matvec_free, trace.py:87-94: gather the 4
// facets of each element, y_e = S x_e, sum the two owners of every facet), organised for the
// B200 memory system instead of for the reference's [facet][node] layout:
//
//   Device layout ("facet records", see soa_pack_kernel): the mesh is cut into tiles of 32
//   element columns that overlap by one (tile w = columns 31 w .. 31 w + 31).  Record (R, w) is one
//   contiguous, 32-byte-aligned run
//       H[N1][32] | V[N1][31] (+ pad to a sector) | Ein[2][EB]
//   H: node k of horizontal line R over the tile's 32 columns; V: node k of the 31 vertical
//   lines 31 w + 1 .. 31 w + 31 of element row R - 1 that the tile owns; Ein: the two
//   lines the tile needs from its neighbours (left-in = line 31 w, right-in = line 31 w + 32),
//   EB = N1 rounded up to 4 doubles each.  Boundary facets and pads are stored zeros.  Every 32-byte
//   sector of a record has exactly one writer and is written whole: H rows by 256-byte warp
//   stores, the packed V block by 32-byte vector stores staged through the ring, the edge blocks
//   of the neighbouring tiles by 32-byte vector stores of lanes 0 / 30
//   (partial sectors that meet late in L2 cost ~10% of the kernel at 1024^2, p = 4).
//
//   One warp walks a segment of element rows of one tile (lane = column); the four warps of a CTA
//   take four consecutive segments of the same tile.  Per element row lane 0 issues ONE bulk copy
//   (TMA) of the next record into a per-warp ring of RING entries completed on mbarriers,
//   RING - 1 rows ahead; each lane then reads its four facets from the ring (the bottom H values
//   stay in registers from the previous row).  The element product runs in the symmetry-adapted
//   basis of the square element (mirrors x -> 1-x and y -> 1-y commute with S for a constant
//   coefficient on a uniform mesh): sum/difference butterflies split the 4 n1 element values into
//   four classes and S becomes four dense blocks, (2h)^2 + 2 n1^2 + (2l)^2 FMAs, h = ceil(n1/2),
//   l = floor(n1/2): 102 instead of 400 at p = 4.  Facet sums: the top part of row r-1 stays in
//   registers for the bottom part of row r; the right part of a lane meets the left part of
//   lane+1 by shuffle.  Every slot of y is written exactly once (boundary and pad slots as
//   zeros), so y is a valid input of the next apply.  No atomics, no grid synchronisation: one
//   writer per facet (trace.py:3-7).
//
//   Segment boundaries: the first horizontal line of a segment also needs the top part of the
//   element row below it.  Inside a CTA the upper warp keeps its bottom part in registers and
//   closes the line after the loop with the lower warp's last top part (handed over through the
//   lower warp's idle ring, one __syncthreads per kernel); only the first warp of a CTA walks a
//   ghost row.  The first record of a segment is read for its H part only.
#pragma once
#include <cuda_runtime.h>

#include "hdg_kernels.cuh"   // cp_async8 / cp_async_commit / cp_async_wait

#ifndef HDG_SOA_EXP
#define HDG_SOA_EXP 0          // experiment flags (tools/build_variants.sh), 0 in the product
#endif
#ifndef HDG_SOA_BAL
#define HDG_SOA_BAL 1          // the ghost-row warp of a CTA owns one row fewer
#endif
#ifndef HDG_SOA_PDL
#define HDG_SOA_PDL 1          // programmatic dependent launch: the prologue overlaps the previous kernel's
                               // tail; griddepcontrol.wait before the first global access (32.7 vs 35.1 us)
#endif
#ifndef HDG_SOA_RING
#define HDG_SOA_RING 3
#endif
#ifndef HDG_SOA_RING_P1
#define HDG_SOA_RING_P1 8
#endif
#ifndef HDG_SOA_RING_P2
#define HDG_SOA_RING_P2 3
#endif
#ifndef HDG_SOA_MCONST
#define HDG_SOA_MCONST -1      // blocks from the constant bank (1) or shared memory (0); -1: by order
                               // (constant bank for p <= 4: 36.7 vs 37.3 us at 1024^2; at p = 8
                               // the 326 entries overflow the uniform registers: 264 vs 220 us)
#endif
#ifndef HDG_SOA_MINB3_MAXN1
#define HDG_SOA_MINB3_MAXN1 9   // 3 CTAs/SM (168 registers) up to this n1
#endif
#ifndef HDG_SOA_HOLD_SMEM_MIN_N1
#define HDG_SOA_HOLD_SMEM_MIN_N1 8
#endif
#ifndef HDG_SOA_MINB_HI
#define HDG_SOA_MINB_HI 3      // CTAs per SM for p >= 3 (154 registers at p = 4 without a cap)
#endif

namespace hdg {

// sweeps of the record-layout cycle (hdg_soa_cycle.cuh)
enum { SOA_EPI_BJ = 1, SOA_EPI_BJ0 = 2, SOA_EPI_RES = 3, SOA_EPI_RESPR = 4, SOA_EPI_BJ0F = 5 };

template <int N1>
struct SoaCfg {
  static constexpr int H = (N1 + 1) / 2, L = N1 / 2;
  static constexpr int A0 = 2 * H, A1 = N1, A2 = N1, A3 = 2 * L;   // class sizes
  static constexpr int MSZ = A0 * A0 + A1 * A1 + A2 * A2 + A3 * A3;
  static constexpr int NTH = 128;
  static constexpr int WPB = NTH / 32;                   // warps (= stacked segments) per CTA
  static constexpr int MINB = N1 <= 3 ? 4 : (N1 <= HDG_SOA_MINB3_MAXN1 ? HDG_SOA_MINB_HI : 2);   // high orders: 255 registers, 2 CTAs/SM (no spills)
  // ring entries per warp (RING-1 rows in flight): the short records of the lowest orders need more
  // rows in flight to cover the HBM latency (p = 1: 1088-byte records, 16 warps/SM)
  static constexpr int RING = N1 == 2 ? HDG_SOA_RING_P1 : (N1 == 3 ? HDG_SOA_RING_P2 : HDG_SOA_RING);
  static constexpr int VOFF = N1 * 32;                   // V rows, 31 slots each, packed
  static constexpr int VB = (N1 * 31 + 3) & ~3;          // doubles of the V block (whole sectors)
  static constexpr int EOFF = VOFF + VB;                 // edge-in blocks: left-in | right-in
  static constexpr int EB = (N1 + 3) & ~3;               // doubles per edge block (whole sectors)
  static constexpr int ENT = EOFF + 2 * EB;              // doubles per record (multiple of 4)
  // high orders keep the deferred first line's bottom part in shared memory (18 registers at n1 = 9)
  static constexpr bool HOLD_SMEM = N1 >= HDG_SOA_HOLD_SMEM_MIN_N1;
  static constexpr int HOLD = HOLD_SMEM ? N1 * 32 : 0;
  static constexpr int WSTRIDE = (RING * ENT + RING + HOLD + 3) & ~3;   // doubles per warp (32-byte multiple)
  static constexpr int SMEM_RING = WPB * WSTRIDE * 8;
};

template <int N1>
struct SoaArgs {
  const double* x;
  double* y;
  int nx, ny, W, nss;                // tiles, super-segments (CTAs per tile)
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
  static constexpr int TOTAL = (O3 + SoaTri<C::A3>::NP + 3) & ~3;   // doubles (32-byte multiple)
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

// general (non-symmetric) class blocks from the constant bank: z = M t, every entry one FMA
template <int SZ, int MOFF, int TOFF>
__device__ __forceinline__ void soa_block_cg(const double* M, const double* t, double* z) {
#pragma unroll
  for (int i = 0; i < SZ; ++i) {
    double s = M[MOFF + i * SZ] * t[TOFF];
#pragma unroll
    for (int j = 1; j < SZ; ++j) s = fma(M[MOFF + i * SZ + j], t[TOFF + j], s);
    z[TOFF + i] = s;
  }
}

template <int N1>
__device__ __forceinline__ void soa_blocks_cg(const double* M, const double* t, double* z) {
  using C = SoaCfg<N1>;
  constexpr int M1 = C::A0 * C::A0, M2 = M1 + C::A1 * C::A1, M3 = M2 + C::A2 * C::A2;
  soa_block_cg<C::A0, 0, 0>(M, t, z);
  soa_block_cg<C::A1, M1, C::A0>(M, t, z);
  soa_block_cg<C::A2, M2, C::A0 + C::A1>(M, t, z);
  soa_block_cg<C::A3, M3, C::A0 + C::A1 + C::A2>(M, t, z);
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

// one whole 32-byte sector per store (sm_100: 256-bit global stores)
__device__ __forceinline__ void st_sector(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// N1 values (+ zero pad) -> an edge block of EB doubles
template <int N1>
__device__ __forceinline__ void soa_store_edge(double* p, const double* v) {
  constexpr int EB = SoaCfg<N1>::EB;
#pragma unroll
  for (int q = 0; q < EB; q += 4)
    st_sector(p + q, q < N1 ? v[q] : 0.0, q + 1 < N1 ? v[q + 1] : 0.0, q + 2 < N1 ? v[q + 2] : 0.0,
              q + 3 < N1 ? v[q + 3] : 0.0);
}

template <int N1, int MCONST = (HDG_SOA_MCONST < 0 ? (N1 <= 5) : HDG_SOA_MCONST)>
__global__ void __launch_bounds__(SoaCfg<N1>::NTH, SoaCfg<N1>::MINB)
    soa_apply_kernel(const __grid_constant__ SoaArgs<N1> a) {
  using C = SoaCfg<N1>;
  constexpr int NT = 4 * N1, RING = C::RING, D = RING - 1, WPB = C::WPB;
  constexpr int ENT = C::ENT, VOFF = C::VOFF, VB = C::VB, EOFF = C::EOFF, EB = C::EB;
  extern __shared__ __align__(32) double smem_soa[];
  double* Ms = smem_soa;
  if (!MCONST) {
    soa_load_blocks<N1>(a, Ms);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  double* ring0 = smem_soa + SoaSmem<N1>::TOTAL;
  double* ring = ring0 + q * C::WSTRIDE;
  const int w = blockIdx.x % a.W, ss = blockIdx.x / a.W;
  const int c = 31 * w + lane;                         // element column of this lane
  // the CTA's rows [c0, c1) (balanced over the tile's CTAs) split over its warps; the first warp of
  // a CTA with rows below it also walks a ghost row, so it owns one row fewer
  const int c0 = (int)((long long)ss * a.ny / a.nss), c1 = (int)((long long)(ss + 1) * a.ny / a.nss);
  const int g = (HDG_SOA_BAL && c0 > 0) ? 1 : 0;
  auto lo = [&](int u) { return u <= 0 ? c0 : min(c1, c0 + max(0, (c1 - c0 + g) * u / WPB - g)); };
  const int r0 = lo(q), r1 = lo(q + 1);
  const bool active = r1 > r0;
  int below = -1;                                      // nearest non-empty segment below, same CTA
  for (int u = q - 1; u >= 0 && below < 0; --u)
    if (lo(u + 1) > lo(u)) below = u;
  const bool defer = active && below >= 0;             // first line closed after the loop
  const int rs = (active && below < 0 && r0 > 0) ? r0 - 1 : r0;   // ghost row (first warp of a CTA)
  const int nrows = r1 - rs;                           // element rows walked; records rs .. r1
  const double* __restrict__ X = a.x;
  double* __restrict__ Y = a.y;
  const long long W = a.W;
  auto rec = [&](int R, long long tile) { return (R * W + tile) * ENT; };   // record R, tile

  // ring entry t = record rs + t of this warp's tile (H line rs+t, V of element row rs+t-1): one
  // contiguous bulk copy (TMA) issued by lane 0, completion counted on the entry's mbarrier.
  // The first record of a segment is needed for its H line only: a short copy.
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + RING * ENT);
  if (lane == 0) {
#pragma unroll
    for (int e = 0; e < RING; ++e) mbar_init(bars + e, 1);
  }
  fence_proxy_async();
  __syncwarp();
#if HDG_SOA_PDL
#if HDG_SOA_PDL == 2
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");   // x may be the previous apply's y
#endif
  auto issue = [&](int t) {
    if (t > nrows || lane != 0 || !active) return;
    uint64_t* bar = bars + (t % RING);
    const unsigned bytes = t == 0 ? VOFF * 8u : ENT * 8u;
    mbar_arrive_expect_tx(bar, bytes);
    tma_load_1d(ring + (t % RING) * ENT, X + rec(rs + t, w), bytes, bar);
  };
#pragma unroll
  for (int t = 0; t < D; ++t) issue(t);

  const bool hcol = c < a.nx;
  const bool vline = lane < 31 && c + 1 <= a.nx - 1;   // V line c + 1 (slot = lane) is a DOF
  // per-lane V reads: right line = slot lane (lane 31: right-in), left line = slot lane - 1
  // (lane 0: left-in); edge blocks are [k] contiguous, V rows 32 apart
  const int oL = lane == 0 ? EOFF : VOFF + lane - 1, sL = lane == 0 ? 1 : 31;
  const int oR = lane == 31 ? EOFF + EB : VOFF + lane, sR = lane == 31 ? 1 : 31;
  // tp: the T part of the row below (facet-sum partner); xC: its top H line = this row's bottom
  double tp[N1], xC[N1], hold[C::HOLD_SMEM ? 1 : N1];
  double* holds = ring + RING * ENT + RING + lane;     // HOLD_SMEM: [k * 32 + lane], behind the barriers
#pragma unroll
  for (int k = 0; k < N1; ++k) tp[k] = 0.0;
#pragma unroll
  for (int k = 0; k < (C::HOLD_SMEM ? 1 : N1); ++k) hold[k] = 0.0;

  if (active) {
#pragma unroll 1
    for (int t = 0; t < nrows; ++t) {
      const int r = rs + t;
      fence_proxy_async();                             // generic reads of entry t-1 before its async refill
      issue(t + D);                                    // entry t+D (slot of entry t-1: read last iteration)
      if (t == 0) mbar_wait(bars, 0);
      mbar_wait(bars + (t + 1) % RING, ((t + 1) / RING) & 1);
      // lower entry = record r (H line r), upper entry = record r + 1 (H line r+1, V of row r)
      const double* e0 = ring + (t % RING) * ENT;
      const double* e1 = ring + ((t + 1) % RING) * ENT;
      double xB[N1], xT[N1], xR[N1], xL[N1];
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        xB[k] = t == 0 ? e0[k * 32 + lane] : xC[k];
        xT[k] = e1[k * 32 + lane];
        xL[k] = e1[oL + k * sL];
        xR[k] = e1[oR + k * sR];
      }
      double yB[N1], yR[N1], yT[N1], yL[N1];
#if HDG_SOA_EXP == 1 || HDG_SOA_EXP == 4   // experiment: no element product (memory path only)
#pragma unroll
      for (int k = 0; k < N1; ++k) { yB[k] = xB[k]; yR[k] = xR[k]; yT[k] = xT[k]; yL[k] = xL[k]; }
#else
      double tv[NT], z[NT];
      soa_forward<N1>(xB, xR, xT, xL, tv);
      if (MCONST) soa_blocks_c<N1>(a.M, tv, z);
      else soa_blocks<N1>(Ms, tv, z);
      soa_backward<N1>(z, yB, yR, yT, yL);
#endif
#if HDG_SOA_EXP == 2 || HDG_SOA_EXP == 4   // experiment: no stores unless the result is NaN (compute + loads only)
      if (yB[0] != yB[0] || yR[N1 - 1] != yR[N1 - 1])
#endif
      if (r >= r0) {
        if (t == 0 && defer) {                         // line r0 waits for the warp below
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            if constexpr (C::HOLD_SMEM) holds[k * 32] = yB[k];
            else hold[k] = yB[k];
          }
        } else {                                       // H line r = T(r-1) + B(r)
          const bool hint = hcol && r >= 1;
          double* hrec = Y + rec(r, w);
#pragma unroll
          for (int k = 0; k < N1; ++k) hrec[k * 32 + lane] = hint ? tp[k] + yB[k] : 0.0;
        }
        double* vrec = Y + rec(r + 1, w);              // V of element row r
        double vv[N1];
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          const double fromR = __shfl_down_sync(0xffffffffu, yL[k], 1);
          vv[k] = vline ? yR[k] + fromR : 0.0;
        }
        // the packed V block leaves as whole sectors through ring entry t (dead: its H line is in
        // registers, it is refilled next iteration after the proxy fence)
        double* stg = ring + (t % RING) * ENT;
        __syncwarp();                                  // t == 0: every lane has read its xB
#pragma unroll
        for (int k = 0; k < N1; ++k)
          if (lane < 31) stg[k * 31 + lane] = vv[k];
        if (lane < VB - N1 * 31) stg[N1 * 31 + lane] = 0.0;
        __syncwarp();
#pragma unroll
        for (int o = 0; o < VB / 4; o += 32)
          if (o + lane < VB / 4) {
            const double2 v0 = reinterpret_cast<const double2*>(stg)[2 * (o + lane)];
            const double2 v1 = reinterpret_cast<const double2*>(stg)[2 * (o + lane) + 1];
            st_sector(vrec + VOFF + 4 * (o + lane), v0.x, v0.y, v1.x, v1.y);
          }
        // edge-in blocks: line 31w+31 is the right tile's left-in, line 31w+1 the left tile's
        // right-in; the mesh boundary tiles zero their own outer blocks
        if (lane == 30) {
          if (w + 1 < W) soa_store_edge<N1>(vrec + ENT + EOFF, vv);
          else {
#pragma unroll
            for (int k = 0; k < N1; ++k) vv[k] = 0.0;
            soa_store_edge<N1>(vrec + EOFF + EB, vv);
          }
        }
        if (lane == 0) {
          if (w > 0) soa_store_edge<N1>(vrec - ENT + EOFF + EB, vv);
          else {
#pragma unroll
            for (int k = 0; k < N1; ++k) vv[k] = 0.0;
            soa_store_edge<N1>(vrec + EOFF, vv);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        tp[k] = yT[k];
        xC[k] = xT[k];
      }
      __syncwarp();                                    // entry t is free for issue(t + RING)
    }
#if HDG_SOA_PDL == 3
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    // hand the last top part to the warp above (this warp's ring is idle now)
#pragma unroll
    for (int k = 0; k < N1; ++k) ring[k * 32 + lane] = tp[k];
  }
  __syncthreads();
  if (defer) {
    const double* src = ring0 + below * C::WSTRIDE;
    const bool hint = hcol && r0 >= 1;
    double* hrec = Y + rec(r0, w);
#pragma unroll
    for (int k = 0; k < N1; ++k)
      hrec[k * 32 + lane] = hint ? src[k * 32 + lane] + (C::HOLD_SMEM ? holds[k * 32] : hold[C::HOLD_SMEM ? 0 : k]) : 0.0;
  }
  if (active && r1 == a.ny) {                          // top boundary line
    double* hrec = Y + rec(a.ny, w);
#pragma unroll
    for (int k = 0; k < N1; ++k) hrec[k * 32 + lane] = 0.0;
  }
  if (active && r0 == 0) {                             // V, edges of element row -1 (pad part of record 0)
    double* vrec = Y + rec(0, w) + VOFF;
    for (int o = lane; o < VB + 2 * EB; o += 32) vrec[o] = 0.0;
  }
}

// Record layout: record (R, w), R = 0..ny, w < W = ceil((nx - 1) / 31):
//   H[k][j] (j < 32)  = node k of horizontal line R, column 31 w + j
//   V[k][j] (j < 31)  = node k of vertical line 31 w + 1 + j, element row R - 1 (rows packed)
//   Ein[0][k], Ein[1][k] = node k of vertical lines 31 w and 31 w + 32, element row R - 1
template <int N1>
__global__ void soa_pack_kernel(const double* __restrict__ x, double* __restrict__ xs, int nx, int ny, int W,
                                long long nh, long long total) {
  using C = SoaCfg<N1>;
  constexpr int ENT = C::ENT, VOFF = C::VOFF, EOFF = C::EOFF, EB = C::EB;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const long long rw = t / ENT;
  const int o = (int)(t % ENT);
  const int R = (int)(rw / W), w = (int)(rw % W);
  double v = 0.0;
  if (o < VOFF) {
    const int k = o / 32, col = 31 * w + o % 32;
    if (R >= 1 && R <= ny - 1 && col < nx) v = x[((long long)(R - 1) * nx + col) * N1 + k];
  } else {
    int k, line;
    if (o < EOFF) {
      k = (o - VOFF) / 31;
      line = k < N1 ? 31 * w + 1 + (o - VOFF) % 31 : 0;
      k = min(k, N1 - 1);
    } else {
      k = (o - EOFF) % EB;
      line = k < N1 ? 31 * w + ((o - EOFF) / EB ? 32 : 0) : 0;
    }
    const int r = R - 1;
    if (r >= 0 && line >= 1 && line <= nx - 1) v = x[(nh + (long long)(line - 1) * ny + r) * N1 + k];
  }
  xs[t] = v;
}

template <int N1>
__global__ void soa_unpack_kernel(const double* __restrict__ xs, double* __restrict__ x, int nx, int ny, int W,
                                  long long nh, long long ndof) {
  using C = SoaCfg<N1>;
  constexpr int ENT = C::ENT, VOFF = C::VOFF;
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= ndof) return;
  const long long blk = u / N1;
  const int k = (int)(u % N1);
  long long src;
  if (blk < nh) {
    const int R = (int)(blk / nx) + 1, col = (int)(blk % nx), w = min(col / 31, W - 1);
    src = ((long long)R * W + w) * ENT + k * 32 + (col - 31 * w);
  } else {
    const long long b = blk - nh;
    const int line = (int)(b / ny) + 1, r = (int)(b % ny), w = (line - 1) / 31;
    src = ((long long)(r + 1) * W + w) * ENT + VOFF + k * 31 + (line - 31 * w - 1);
  }
  x[u] = xs[src];
}

// Blocked pack / unpack: one CTA moves SOA_PB consecutive records of one tile through shared
// memory, so the reference-layout side is read / written as contiguous runs (a horizontal line
// segment of 32 columns = 32 N1 doubles; SOA_PB rows of one vertical line = SOA_PB N1 doubles) and
// the record side as whole records.
__host__ __device__ constexpr int soa_pb(int n1) { return n1 <= 9 ? 8 : 4; }   // records per CTA (48 KB of static shared memory)

template <int N1>
__global__ void __launch_bounds__(256) soa_pack_blocked_kernel(const double* __restrict__ x, double* __restrict__ xs,
                                                               int nx, int ny, int W, long long nh) {
  using C = SoaCfg<N1>;
  constexpr int ENT = C::ENT, VOFF = C::VOFF, EOFF = C::EOFF, EB = C::EB;
  constexpr int SOA_PB = soa_pb(N1);
  __shared__ __align__(16) double S[SOA_PB * ENT];
  // row blocks fastest: CTAs running together read neighbouring pieces of the same vertical lines
  const int nrb = (ny + SOA_PB) / SOA_PB;
  const int w = blockIdx.x / nrb, R0 = (blockIdx.x % nrb) * SOA_PB;
  const int nr = min(SOA_PB, ny + 1 - R0);
  for (int t = threadIdx.x; t < SOA_PB * ENT; t += blockDim.x) S[t] = 0.0;
  __syncthreads();
  // H: record R0 + rr holds line R0 + rr, columns 31 w .. 31 w + 31: one contiguous source run per line
  const int ncol = min(32, nx - 31 * w), hl = ncol * N1;
  for (int t = threadIdx.x; t < nr * hl; t += blockDim.x) {
    const int rr = t / hl, u = t - rr * hl, R = R0 + rr;
    if (R < 1 || R > ny - 1) continue;
    S[rr * ENT + (u % N1) * 32 + u / N1] = __ldg(x + ((long long)(R - 1) * nx + 31 * w) * N1 + u);
  }
  // V: lines 31 w .. 31 w + 32 (first / last are the edge-in lines), element rows [ra, rb): one
  // contiguous source run of (rb - ra) N1 doubles per line
  const int ra = max(R0 - 1, 0), rb = R0 + nr - 1;
  const int len = max(rb - ra, 0) * N1;
  for (int t = threadIdx.x; t < 33 * len; t += blockDim.x) {
    const int l = t / len, u = t - l * len, line = 31 * w + l;
    if (line < 1 || line > nx - 1) continue;
    const int rr = ra + u / N1 + 1 - R0, k = u % N1;
    const int o = l == 0 ? EOFF + k : (l == 32 ? EOFF + EB + k : VOFF + k * 31 + (l - 1));
    S[rr * ENT + o] = __ldg(x + (nh + (long long)(line - 1) * ny + ra) * N1 + u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nr * ENT; t += blockDim.x) {
    const int rr = t / ENT, o = t - rr * ENT;
    xs[((long long)(R0 + rr) * W + w) * ENT + o] = S[t];
  }
}

template <int N1>
__global__ void __launch_bounds__(256) soa_unpack_blocked_kernel(const double* __restrict__ xs, double* __restrict__ x,
                                                                 int nx, int ny, int W, long long nh) {
  using C = SoaCfg<N1>;
  constexpr int ENT = C::ENT, VOFF = C::VOFF;
  constexpr int SOA_PB = soa_pb(N1);
  __shared__ __align__(16) double S[SOA_PB * ENT];
  // row blocks fastest: CTAs running together read neighbouring pieces of the same vertical lines
  const int nrb = (ny + SOA_PB) / SOA_PB;
  const int w = blockIdx.x / nrb, R0 = (blockIdx.x % nrb) * SOA_PB;
  const int nr = min(SOA_PB, ny + 1 - R0);
  for (int t = threadIdx.x; t < nr * ENT; t += blockDim.x) {
    const int rr = t / ENT, o = t - rr * ENT;
    S[t] = __ldg(xs + ((long long)(R0 + rr) * W + w) * ENT + o);
  }
  __syncthreads();
  // H columns 31 w .. 31 w + 30 (the last tile also its 32nd column)
  const int ncol = min(w == W - 1 ? 32 : 31, nx - 31 * w), hl = ncol * N1;
  for (int t = threadIdx.x; t < nr * hl; t += blockDim.x) {
    const int rr = t / hl, u = t - rr * hl, R = R0 + rr;
    if (R < 1 || R > ny - 1) continue;
    x[((long long)(R - 1) * nx + 31 * w) * N1 + u] = S[rr * ENT + (u % N1) * 32 + u / N1];
  }
  const int ra = max(R0 - 1, 0), rb = R0 + nr - 1;
  const int len = max(rb - ra, 0) * N1;
  for (int t = threadIdx.x; t < 31 * len; t += blockDim.x) {
    const int l = t / len + 1, u = t - (l - 1) * len, line = 31 * w + l;
    if (line > nx - 1) continue;
    const int rr = ra + u / N1 + 1 - R0, k = u % N1;
    x[(nh + (long long)(line - 1) * ny + ra) * N1 + u] = S[rr * ENT + VOFF + k * 31 + (l - 1)];
  }
}

}  // namespace hdg
