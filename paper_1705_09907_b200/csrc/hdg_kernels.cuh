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
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

namespace hdg {

namespace cg = cooperative_groups;

#ifndef HDG_NBUF
#define HDG_NBUF 0         // stage buffers per CTA; 0 = per-order default (measured, see Cfg)
#endif
#ifndef HDG_F_MAXN1
#define HDG_F_MAXN1 13     // cap on the two-facets-per-thread rule (tuning knob)
#endif
#ifndef HDG_F_SHARED
#define HDG_F_SHARED 3     // facet rows per thread in shared mode for n1 <= HDG_F3_MAXN1
#endif
#ifndef HDG_F3_MAXN1
#define HDG_F3_MAXN1 5     // shared mode: HDG_F_SHARED facets per thread up to this n1 (measured: p<=4)
#endif
#ifndef HDG_F_MAXN1_STORED
#define HDG_F_MAXN1_STORED 2   // stored mode: two facet rows per thread up to this n1 (smaller tiles keep the
                               // half-stored partner reads in L2: p=4 105 -> 90 us; p=1 prefers 2 rows)
#endif
#ifndef HDG_F_MAXN1_SHARED
#define HDG_F_MAXN1_SHARED 9
#endif
#ifndef HDG_MINB
#define HDG_MINB 2         // __launch_bounds__ min blocks per SM for the trace kernel
#endif
#ifndef HDG_DMMA
#define HDG_DMMA 0         // shared mode: FP64 tensor-core (DMMA m8n8k4) stencil GEMM for n1 <= 8
#endif
#ifndef HDG_NWARP
#define HDG_NWARP 0        // warps per CTA; 0 = per-configuration default (Cfg::NW, measured)
#endif
#ifndef HDG_SYMSTORE
#define HDG_SYMSTORE 1     // stored mode: each facet-pair coupling block stored once (4 of 7 blocks per facet)
#endif
#ifndef HDG_SYMSTORE_EF_MIN_N1
#ifndef HDG_PAIR_PREFETCH
#define HDG_PAIR_PREFETCH 0     // L2 prefetch of the next block of the merged stored pass (measured slower: 0.61 -> 0.58 at p = 8)
#endif
#ifndef HDG_PAIR_RING
#define HDG_PAIR_RING 1         // merged stored pass streams its blocks through a per-warp TMA ring
#endif
#ifndef HDG_PAIR_RING_MAX_N1
#define HDG_PAIR_RING_MAX_N1 10
#endif
#ifndef HDG_PAIR_AHEAD_MAX_N1
#define HDG_PAIR_AHEAD_MAX_N1 7
#endif
#ifndef HDG_PAIR_STAGES
#define HDG_PAIR_STAGES 4       // ring stages per warp of the merged stored pass (3 block rows in flight)
#endif
#ifndef HDG_PAIR_MIN_N1
#define HDG_PAIR_MIN_N1 6      // merged h/v pass over the half-stored stream from this n1 (apply_stored_pair; at n1 = 5 it loses: 0.88 -> 0.77)
#endif
#define HDG_SYMSTORE_EF_MIN_N1 7   // half-stored stream: evict-first hint on the owner's read from this n1
#endif                             // (measured: p=8 192 vs 207 us, p=4 118 vs 105 us, p=1 69 vs 62 us)
#ifndef HDG_SHARED_SYM
#define HDG_SHARED_SYM 1   // shared mode: mirror-reduced stencil (apply_shared_sym); 0 = full n1 x 7n1
#endif
#if HDG_DMMA
#undef HDG_SHARED_SYM
#define HDG_SHARED_SYM 0
#endif

constexpr int TX = 32;     // tile width in elements (= warp width: lanes walk i)
constexpr int MAXN1 = 13;  // p <= 12
constexpr int MAX_CTAS_PER_SM = 8;

enum Epi { EPI_Y = 0, EPI_RES = 1, EPI_BJ = 2, EPI_RESPR = 3 };

template <int N1, bool ST = false> struct Cfg {
  // warps per CTA (measured on B200, tools/tune_matvec.py): 8 for the low-order shared and the
  // p <= 2 stored kernels; 4-warp CTAs (3 per SM) for high orders and stored p >= 3, where
  // shorter tiles shorten the stencil/partner reuse distances (shared p=8 59.7 -> 48.2 us,
  // p=12 53.3 -> 49.2 us, stored p=8 192 -> 182 us; shared p=4 44.5 vs 45.1 us with 4)
  static constexpr int NW = HDG_NWARP ? HDG_NWARP : ((N1 <= 3 || (!ST && N1 <= 5)) ? 8 : 4);
  static constexpr int NTH = 32 * NW;
  static constexpr int MINB = (NW >= 8) ? (ST ? 2 : (N1 <= 9 ? HDG_MINB : 1)) : 3;
  static constexpr int S = N1;                      // facet blocks contiguous in a staged run
  // facets per thread per orientation (measured: 2 pays up to p=8 when W is in the constant
  // bank, up to p=4 when W streams from HBM)
  static constexpr int F = (N1 <= (ST ? HDG_F_MAXN1_STORED : HDG_F_MAXN1_SHARED)) && (N1 <= HDG_F_MAXN1)
                               ? ((!ST && N1 <= HDG_F3_MAXN1) ? HDG_F_SHARED : 2) : 1;
  static constexpr int TY = NW * F;                 // tile height in elements
  // stored stream entries per facet: the merged n1 x 7n1 row (7 blocks), or with HDG_SYMSTORE
  // only the blocks this facet owns (diagonal + 3 couplings); the other 3 are read transposed from
  // the neighbour that owns the pair (the operator is symmetric)
  static constexpr int WSZ = (HDG_SYMSTORE ? 4 : 7) * N1 * N1;
  static constexpr int DSZ = N1 * N1;               // block-Jacobi inverse entries
  static constexpr int QUNROLL = (N1 <= 8) ? 7 : 1; // keep registers bounded at high order
  static constexpr int HROWS = TY + 2, HCOLS = TX + 1;
  static constexpr int VCOLS = TX + 2, VROWS = TY + 1;
  // H rows are exact copies of contiguous global runs (TMA bulk copies); each run has one
  // slack double so its start can be shifted to the global 16-byte parity.  V columns are
  // contiguous along j in HBM but lanes walk i, so they are TRANSPOSED while staging (8-byte
  // LDGSTS scatter) into [row][column] with an odd block stride: conflict-free 64-bit LDS.
  static constexpr bool CONTIG = true;
  static constexpr int RS = (HCOLS * S + 2) & ~1;                         // H row stride (even)
  static constexpr int HSZ = HROWS * RS;                                  // even
  static constexpr int SV = (N1 & 1) ? N1 : N1 + 1;                       // V block stride (odd)
  static constexpr int BUF_X = HSZ + VROWS * VCOLS * SV;
  // output staging (reuses the consumed x buffer): h rows of TX facets, v columns of TY facets
  static constexpr int NOUT = N1;                                         // max outputs per facet
  static constexpr int YCS = (TY * NOUT) | 1;                             // odd column stride
  static constexpr int BUF_Y = TX * YCS + TY * TX * NOUT;
  static constexpr int BUF = ((BUF_X > BUF_Y ? BUF_X : BUF_Y) + 1) & ~1;  // doubles per stage buffer
  // measured on B200 (tools/tune_matvec.py): double buffering pays for p <= 2 (little compute
  // per byte); for p >= 3 a single buffer (more L1, two CTAs per SM overlap each other) wins
  static constexpr int NBUF = HDG_NBUF ? HDG_NBUF : (N1 <= 3 ? 2 : 1);
  static constexpr bool DMMA = HDG_DMMA && N1 <= 8;
  static constexpr int KS = (7 * N1 + 3) / 4;                             // DMMA k-steps (K = 7 n1)
  static constexpr int WSCR = DMMA ? 32 * 9 : 32 * NOUT;                  // per-warp output transpose
  // shared mode adds the per-warp transpose scratch; stored mode stages h outputs in BUF
  // Residual / Jacobi / restriction epilogues need b of the tile's own facets.  h-facet rows are
  // contiguous runs (loaded coalesced through the warp scratch); the v-facet columns would be
  // one scattered 40-byte piece per lane, so they are staged with the tile, transposed like x
  // ([row][column], odd block stride), when two CTAs per SM still fit.
  static constexpr int SB = (N1 & 1) ? N1 : N1 + 1;
  static constexpr int BSZ = ((TY * TX * SB) + 1) & ~1;
  __host__ __device__ static constexpr int base_doubles(bool stored) { return NBUF * BUF + (stored ? 0 : (NW + 1) * WSCR); }
  template <int EPI> __host__ __device__ static constexpr bool stage_b() {
    return EPI != 0 && (base_doubles(ST) + NBUF * BSZ) * 8 <= 113 * 1024;
  }
  template <int EPI> __host__ __device__ static constexpr int bufs() { return BUF + (stage_b<EPI>() ? BSZ : 0); }   // stage stride
  // merged h/v pass over the half-stored stream (apply_stored_pair): every warp streams its block
  // rows (n1 entries x 32 lanes = n1 * 256 contiguous bytes each) through a private TMA ring
  static constexpr bool PAIR = ST && HDG_SYMSTORE && F == 1 && N1 >= HDG_PAIR_MIN_N1;
  static constexpr int RSTAGES = HDG_PAIR_STAGES;
  static constexpr int RROW = N1 * 32;                                    // doubles per ring stage
  // the ring version's fully unrolled block rows outgrow the instruction cache above n1 = 10
  // (p = 12: 0.43 of HBM with the ring, 0.65 with per-thread loads)
  static constexpr bool PRING = PAIR && HDG_PAIR_RING && N1 <= HDG_PAIR_RING_MAX_N1;
  static constexpr int RING = PRING ? NW * RSTAGES * RROW : 0;
  template <int EPI> __host__ __device__ static constexpr int tile_doubles_epi() {
    return NBUF * bufs<EPI>() + (ST ? 0 : (NW + 1) * WSCR);
  }
  template <int EPI> __host__ __device__ static constexpr int smem_doubles_epi() {
    return ((tile_doubles_epi<EPI>() + 3) & ~3) + RING;
  }
  static constexpr int smem_doubles(bool stored) { return base_doubles(stored); }
};

// Shared-mode operator: both merged facet matrices + block-Jacobi inverses, passed by value
// (kernel-parameter constant bank -> LDCU.128 into uniform registers, shared by all lanes).
template <int N1> struct SharedOp {
  double Wh[7 * N1 * N1];
  double Wv[7 * N1 * N1];
  double Dh[N1 * N1];
  double Dv[N1 * N1];
};

struct MvArgs {
  int nx, ny, nxp;          // mesh and padded interleave row length (multiple of 32)
  int nh;                   // interior horizontal facet blocks = nx * (ny - 1)
  const double* x;          // input trace vector
  const double* b;          // right-hand side (RES / BJ / RESPR)
  double* out;              // y | r | x_out | r_coarse
  const double* Wh;         // stored mode: interleaved merged operators [grp][idx][lane]
  const double* Wv;
  const double* Dh;         // stored mode: interleaved D^-1 [grp][idx][lane]
  const double* Dv;
  double omega;
  double w_first;           // EPI_BJ, shared mode: staged x holds b; x1 = w_first D^-1 b first (0: off)
  const double* pec;        // EPI_BJ: coarse p-level vector; staged x becomes x + V ec first (null: off)
  double* partials;         // per-CTA norm^2 partials (RES) or nullptr
  double V[MAXN1 * (MAXN1 - 1)];  // RESPR: fine x coarse p-transfer matrix, row-major
};

// reference block numbering (trace.py:39-41, mesh.py:112-117); ndof < 2^31 per level
__device__ __forceinline__ int hblk(int nx, int i, int j) { return (j - 1) * nx + i; }
__device__ __forceinline__ int vblk(int nh, int ny, int i, int j) { return nh + (i - 1) * ny + j; }

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

// async global->shared copy of one double; src_size 0 zero-fills (boundary / outside the mesh)
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NPEND> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND));
}

// global start (element index) of H row r / V column c of the tile staged at (i0, j0)
template <int N1> __device__ __forceinline__ int h_run_start(const MvArgs& a, int i0, int j0, int r) {
  return ((j0 - 2 + r) * a.nx + i0 - 1) * N1;
}
template <int N1> __device__ __forceinline__ int v_run_start(const MvArgs& a, int i0, int j0, int c) {
  return (a.nh + (i0 - 2 + c) * a.ny + j0 - 1) * N1;
}

// programmatic dependent launch: wait for the kernel before this one in the stream (hdg_internal.h:
// launch_pdl); a no-op for a normally launched grid
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------- mbarrier / TMA (bulk)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// arrive on `bar` once this thread's prior cp.async (LDGSTS) complete; counts as one arrival
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// bounded wait: a lost arrival must surface as an error (trap), never as a hung GPU.  The limit is
// wall-clock (%globaltimer, 20 s), so profiler replay, sanitizers or heavy contention cannot trip it.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
  unsigned done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return done != 0;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  if (mbar_try(bar, parity)) return;
  const unsigned long long t0 = global_ns();
#pragma unroll 1
  while (!mbar_try(bar, parity))
    if (global_ns() - t0 > 20000000000ull) __trap();
}
__device__ __forceinline__ void fence_proxy_async() {
#ifndef HDG_EXP_NOFENCE
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
#endif
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// smem index of element e of a staged run = base + o + e, with o = parity shift so that the
// smem index has the parity of the global index (16-byte alignment of the bulk copy)
__device__ __forceinline__ int run_shift(int g0, int base) { return (g0 - base) & 1; }

// A run: global elements [g0, g0 + len) of x; elements [elo, ehi) are real facets, the rest
// (Dirichlet facets / outside the mesh) must read as 0.  Returns the TMA bytes it will load.
struct Run {
  int g0, base, elo, ehi, len;
  bool valid;
};

__device__ __forceinline__ unsigned run_bytes(const Run& r) {
  if (!r.valid || r.ehi <= r.elo) return 0u;
  int gs = r.g0 + r.elo, ge = r.g0 + r.ehi;
  gs += gs & 1;
  if (gs < ge) ge -= ge & 1;
  return ge > gs ? (unsigned)(ge - gs) * 8u : 0u;
}

// issued by one lane: head/tail doubles by LDGSTS, the aligned body by one bulk copy
__device__ __forceinline__ void run_issue(const double* __restrict__ x, double* buf, const Run& r, uint64_t* bar) {
  if (!r.valid || r.ehi <= r.elo) return;
  double* d = buf + r.base + run_shift(r.g0, r.base) - r.g0;  // d[g] = smem slot of global element g
  int gs = r.g0 + r.elo, ge = r.g0 + r.ehi;
  if (gs & 1) { cp_async8(d + gs, x + gs, true); ++gs; }
  if (gs < ge && (ge & 1)) { cp_async8(d + ge - 1, x + ge - 1, true); --ge; }
  if (ge > gs) tma_load_1d(d + gs, x + gs, (unsigned)(ge - gs) * 8u, bar);
}

// zero the non-facet part of a run (all lanes of the owning warp)
__device__ __forceinline__ void run_zero(double* buf, const Run& r, int lane) {
  double* d = buf + r.base + run_shift(r.g0, r.base);
  if (!r.valid || r.ehi <= r.elo) {
    for (int e = lane; e < r.len; e += 32) d[e] = 0.0;
    return;
  }
  for (int e = lane; e < r.elo; e += 32) d[e] = 0.0;
  for (int e = r.ehi + lane; e < r.len; e += 32) d[e] = 0.0;
}

template <int N1, bool ST> __device__ __forceinline__ Run h_run(const MvArgs& a, int i0, int j0, int r) {
  using C = Cfg<N1, ST>;
  const int j = j0 - 1 + r;
  Run q;
  q.g0 = h_run_start<N1>(a, i0, j0, r);
  q.base = r * C::RS;
  q.len = C::HCOLS * N1;
  q.elo = (i0 == 0) ? N1 : 0;                        // column i = -1
  q.ehi = min(C::HCOLS, a.nx - (i0 - 1)) * N1;       // columns i < nx
  q.valid = (j >= 1 && j <= a.ny - 1);
  return q;
}
// V columns c = c0, c0 + cstep, ... of the tile: lane-constant element offsets hoisted out of
// the column loop, so each copy is a pointer add, a predicate and the LDGSTS.
template <int N1, bool ST>
__device__ __forceinline__ void stage_v_columns(const MvArgs& a, double* Vs, int i0, int j0, int c0, int cstep,
                                                int lane) {
  using C = Cfg<N1, ST>;
  constexpr int LEN = C::VROWS * N1;
  constexpr int NQ = (LEN + 31) / 32;
  const int elo = (j0 == 0) ? N1 : 0;                          // row j = -1
  const int ehi = min(C::VROWS, a.ny - (j0 - 1)) * N1;         // rows j < ny
  int soffq[NQ];
  bool okq[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int e = lane + 32 * q;
    const int r = e / N1, m = e - r * N1;
    soffq[q] = (r * C::VCOLS) * C::SV + m;
    okq[q] = (e < LEN) && e >= elo && e < ehi;
  }
  const long long cstride = (long long)a.ny * N1;
  const double* src = a.x + (long long)v_run_start<N1>(a, i0, j0, c0);
  for (int c = c0; c < C::VCOLS; c += cstep, src += cstep * cstride) {
    const int i = i0 - 1 + c;
    const bool colok = (i >= 1 && i <= a.nx - 1);
    double* dst = Vs + c * C::SV;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (lane + 32 * q < LEN) {
        const bool ok = colok && okq[q];
        cp_async8(dst + soffq[q], ok ? src + lane + 32 * q : a.x, ok);
      }
    }
  }
}

// Stage the x blocks of one tile's facet stencils into shared memory.  H rows
// h(i0-1 .. i0+TX-1, j) and V columns v(i, j0-1 .. j0+TY-1) are contiguous runs of the
// reference layout, so each is ONE bulk (TMA) copy issued by the owning warp's lane 0, plus at
// most two 8-byte LDGSTS for a misaligned head/tail.  Completion: `bar` (2 arrivals per warp).
//   H region: h(i, j), i in [i0-1, i0+TX), j in [j0-1, j0+TY]      ((TY+2) x (TX+1) blocks)
//   V region: v(i, j), i in [i0-1, i0+TX], j in [j0-1, j0+TY)      ((TX+2) x (TY+1) blocks)
// b of the tile's own v facets v(i0 + c, j0 .. j0 + TY - 1), c < TX: one contiguous run per
// column, copied by coalesced 8-byte LDGSTS and transposed into [row][column] (stride SB, odd)
template <int N1, bool ST>
__device__ __forceinline__ void stage_b_columns(const MvArgs& a, double* Bs, int i0, int j0, int warp, int lane) {
  using C = Cfg<N1, ST>;
  constexpr int LEN = C::TY * N1;
  constexpr int NQ = (LEN + 31) / 32;
  const int ehi = min(C::TY, a.ny - j0) * N1;
  for (int c = warp; c < TX; c += C::NW) {
    const int i = i0 + c;
    if (i < 1 || i > a.nx - 1) continue;   // warp-uniform; never read for these columns
    const double* src = a.b + (long long)vblk(a.nh, a.ny, i, j0) * N1;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int e = lane + 32 * q;
      if (e < ehi) {
        const int r = e / N1, m = e - r * N1;
        cp_async8(Bs + (r * TX + c) * C::SB + m, src + e, true);
      }
    }
  }
}

template <int N1, bool ST, bool SBV = false>
__device__ __forceinline__ void stage_tile(const MvArgs& a, double* buf, int i0, int j0, uint64_t* bar) {
  using C = Cfg<N1, ST>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool edge = (i0 == 0) || (j0 == 0) || (i0 + TX >= a.nx) || (j0 + C::TY >= a.ny);
#ifdef HDG_EXP_NOSTAGE
  if (lane == 0) mbar_arrive_expect_tx(bar, 0);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)));
  return;
#endif
#ifdef HDG_EXP_BIGH
  // experiment: the same H bytes as ONE contiguous bulk copy (wrong data; measures per-copy cost)
  if (threadIdx.x == 0) {
    const unsigned hb = (unsigned)((C::HROWS * C::HCOLS * N1 * 8) & ~15);
    const long long tiles = (long long)((a.nx + TX - 1) / TX) * ((a.ny + C::TY - 1) / C::TY);
    const long long t = (long long)(j0 / C::TY) * ((a.nx + TX - 1) / TX) + i0 / TX;
    const long long maxoff = ((long long)a.nh * N1 * 8 - hb) & ~15LL;
    const long long off = (maxoff * t / (tiles > 1 ? tiles - 1 : 1)) & ~15LL;
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, hb);
    tma_load_1d(buf, reinterpret_cast<const char*>(a.x) + off, hb, bar);
  } else if (lane == 0) {
    mbar_arrive_expect_tx(bar, 0);
  }
  if (false) {
#else
  if (lane == 0) {
#endif
    unsigned bytes = 0;
#ifndef HDG_EXP_NOH
    for (int r = warp; r < C::HROWS; r += C::NW) bytes += run_bytes(h_run<N1, ST>(a, i0, j0, r));
#endif
    fence_proxy_async();               // prior generic reads/writes of this buffer -> async proxy
    mbar_arrive_expect_tx(bar, bytes);
#ifndef HDG_EXP_NOH
    for (int r = warp; r < C::HROWS; r += C::NW) run_issue(a.x, buf, h_run<N1, ST>(a, i0, j0, r), bar);
#endif
  }
  if (edge) {  // zero Dirichlet / out-of-mesh parts of H rows (interior tiles skip this)
    for (int r = warp; r < C::HROWS; r += C::NW) run_zero(buf, h_run<N1, ST>(a, i0, j0, r), lane);
  }
  // V columns: coalesced 8-byte LDGSTS from the contiguous run, transposed into [row][col];
  // src-size 0 zero-fills Dirichlet / out-of-mesh blocks
#ifndef HDG_EXP_NOV
  stage_v_columns<N1, ST>(a, buf + C::HSZ, i0, j0, warp, C::NW, lane);
#endif
  if constexpr (SBV) stage_b_columns<N1, ST>(a, buf + C::BUF, i0, j0, warp, lane);
  cp_async_mbar_arrive(bar);           // every thread: one arrival when its LDGSTS land
}

// CTA-wide barrier of the NTH compute threads (named barrier 1)
template <int NTH> __device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(NTH) : "memory");
}

// acc_f = W . [x of facet f's 7 stencil blocks] for FF facets of one orientation.
// Shared mode: W is uniform (constant bank), each W value feeds FF facets.
template <int N1, int FF>
__device__ __forceinline__ void apply_shared(const double* const (&nb)[FF][7], const double* W,
                                             double (&acc)[FF][N1]) {
#pragma unroll
  for (int f = 0; f < FF; ++f)
#pragma unroll
    for (int k = 0; k < N1; ++k) acc[f][k] = 0.0;
#ifdef HDG_EXP_NOCOMPUTE
#pragma unroll
  for (int f = 0; f < FF; ++f)
#pragma unroll
    for (int k = 0; k < N1; ++k) acc[f][k] = nb[f][1][k] + nb[f][4][k];
  return;
#endif
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double xv[FF][N1];
#pragma unroll
    for (int f = 0; f < FF; ++f)
#pragma unroll
      for (int m = 0; m < N1; ++m) xv[f][m] = nb[f][q][m];
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        const double w = W[(q * N1 + k) * N1 + m];
#pragma unroll
        for (int f = 0; f < FF; ++f) acc[f][k] = fma(w, xv[f][m], acc[f][k]);
      }
  }
}

// Shared mode, mirror-reduced form (default).  A constant-coefficient block on a uniform
// Cartesian mesh is invariant under the two mirrors of a facet's stencil (hdg_capi.cu checks
// this at setup to 1e-11 and falls back to stored blocks otherwise):
//   normal mirror      q0 <-> q2, q3 <-> R q5, q4 <-> R q6          (output unchanged)
//   tangential mirror  q0, q1, q2 reversed, q3 <-> q4, q5 <-> q6     (output reversed)
// (R = reversal of a facet's n1 nodes; GLL nodes are symmetric).  Folding the stencil with
// them, a = q0 + q2, c = q3 + R q5, d = q4 + R q6, and splitting a, q1 and c +/- d into their
// even / odd halves, the n1 x 7n1 stencil becomes two small dense blocks:
//   ye (H x KE) . [a_e, q1_e, c + d],   yo (L x KO) . [a_o, q1_o, c - d],
//   y[k] = ye[k] + yo[k],  y[n1-1-k] = ye[k] - yo[k]
// i.e. H KE + L KO FMAs (51 at n1 = 5) instead of 7 n1^2 (175), plus ~7 n1 adds.
template <int N1> struct Sym {
  static constexpr int H = (N1 + 1) / 2, L = N1 / 2;
  static constexpr int KE = 2 * H + N1, KO = 2 * L + N1;
  static constexpr int SIZE = H * KE + L * KO;   // <= 7 n1^2: lives in SharedOp::Wh / Wv
};

template <int N1, int FF>
__device__ __forceinline__ void apply_shared_sym(const double* const (&nb)[FF][7], const double* G,
                                                 double (&acc)[FF][N1]) {
  using Y = Sym<N1>;
  constexpr int H = Y::H, L = Y::L, KE = Y::KE, KO = Y::KO;
  const double* Ge = G;
  const double* Go = G + H * KE;
#ifdef HDG_EXP_NOCOMPUTE
#pragma unroll
  for (int f = 0; f < FF; ++f)
#pragma unroll
    for (int k = 0; k < N1; ++k) acc[f][k] = nb[f][1][k] + nb[f][4][k];
  return;
#endif
  double ze[FF][KE], zo[FF][KO > 0 ? KO : 1];
#pragma unroll
  for (int f = 0; f < FF; ++f) {
    const double* x0 = nb[f][0]; const double* x1 = nb[f][1]; const double* x2 = nb[f][2];
#pragma unroll
    for (int m = 0; m < L; ++m) {
      const double am = x0[m] + x2[m], ar = x0[N1 - 1 - m] + x2[N1 - 1 - m];
      ze[f][m] = am + ar;
      zo[f][m] = am - ar;
      const double om = x1[m], orr = x1[N1 - 1 - m];
      ze[f][H + m] = om + orr;
      zo[f][L + m] = om - orr;
    }
    if constexpr (N1 & 1) {
      ze[f][H - 1] = x0[H - 1] + x2[H - 1];
      ze[f][2 * H - 1] = x1[H - 1];
    }
#pragma unroll
    for (int m = 0; m < N1; ++m) {
      const double c = nb[f][3][m] + nb[f][5][N1 - 1 - m];
      const double d = nb[f][4][m] + nb[f][6][N1 - 1 - m];
      ze[f][2 * H + m] = c + d;
      zo[f][2 * L + m] = c - d;
    }
  }
#pragma unroll
  for (int k = 0; k < H; ++k) {
    double ye[FF], yo[FF];
#pragma unroll
    for (int f = 0; f < FF; ++f) ye[f] = 0.0, yo[f] = 0.0;
#pragma unroll
    for (int t = 0; t < KE; ++t) {
      const double g = Ge[k * KE + t];
#pragma unroll
      for (int f = 0; f < FF; ++f) ye[f] = fma(g, ze[f][t], ye[f]);
    }
    if (k < L) {
#pragma unroll
      for (int t = 0; t < KO; ++t) {
        const double g = Go[k * KO + t];
#pragma unroll
        for (int f = 0; f < FF; ++f) yo[f] = fma(g, zo[f][t], yo[f]);
      }
#pragma unroll
      for (int f = 0; f < FF; ++f) {
        acc[f][k] = ye[f] + yo[f];
        acc[f][N1 - 1 - k] = ye[f] - yo[f];
      }
    } else {
#pragma unroll
      for (int f = 0; f < FF; ++f) acc[f][k] = ye[f];
    }
  }
}

// ------------------------------------------------------------------ FP64 tensor-core core
// y (n1 x 32 facets of one warp row) = W (n1 x 7n1) . X (7n1 x 32) as 4 groups of
// mma.sync.m8n8k4.f64 (DMMA): A = W padded to 8 rows (per-lane fragment in registers), B = the
// facets' stencil values straight from the staged tile, D (8 x 8 facets) -> warp scratch.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// per-lane A fragments: wa[s] = W[row = lane/4][stencil 4s + lane%4] (0 outside n1 x 7n1)
template <int N1>
__device__ __forceinline__ void dmma_wfrag(const double* W, double (&wa)[Cfg<N1>::KS], int lane) {
  const int k = lane >> 2, t = lane & 3;
#pragma unroll
  for (int s = 0; s < Cfg<N1>::KS; ++s) {
    const int st = 4 * s + t;
    const int q = st / N1, m = st - q * N1;
    wa[s] = (k < N1 && st < 7 * N1) ? W[(q * N1 + k) * N1 + m] : 0.0;
  }
}

// stencil block q of facet (ii, jj): base pointer for lane's facet ii and stride along ii
template <int N1, bool VERT>
__device__ __forceinline__ const double* dmma_block(const double* Hs, const double* Vs, int hshift0, int hstep,
                                                    int jj, int ii, int q, int& stride) {
  using C = Cfg<N1>;
  auto H = [&](int r, int c) { return Hs + r * C::RS + ((hshift0 + r * hstep) & 1) + c * C::S; };
  auto V = [&](int c, int r) { return Vs + (r * C::VCOLS + c) * C::SV; };
  if (!VERT) {
    if (q < 3) { stride = C::S; return H(jj - 1 + q, ii); }
    stride = C::SV;
    const int dq = q - 3;
    return V(ii + (dq & 1), jj - 1 + (dq >> 1));
  }
  if (q < 3) { stride = C::SV; return V(ii - 1 + q, jj); }
  stride = C::S;
  const int dq = q - 3;
  return H(jj + (dq & 1), ii - 1 + (dq >> 1));
}

template <int N1, bool VERT>
__device__ __forceinline__ void apply_dmma_row(const double* Hs, const double* Vs, int hshift0, int hstep, int jj,
                                               const double (&wa)[Cfg<N1>::KS], double* scr, double (&acc)[N1],
                                               int lane) {
  using C = Cfg<N1>;
  const int t = lane & 3, fl = lane >> 2;   // k-slot and facet-in-group of this lane's B element
  const double* ptr[C::KS];
  int inc[C::KS];
#pragma unroll
  for (int s = 0; s < C::KS; ++s) {
    int st = 4 * s + t;
    if (st >= 7 * N1) st = 0;                // padding column: any finite value (W is 0 there)
    const int q = st / N1, m = st - q * N1;
    int stride;
    ptr[s] = dmma_block<N1, VERT>(Hs, Vs, hshift0, hstep, jj, fl + 1, q, stride) + m;
    inc[s] = 8 * stride;
  }
  double d[4][2];
#pragma unroll
  for (int g = 0; g < 4; ++g) { d[g][0] = 0.0; d[g][1] = 0.0; }
#pragma unroll
  for (int s = 0; s < C::KS; ++s) {
#pragma unroll
    for (int g = 0; g < 4; ++g) dmma_8x8x4(d[g][0], d[g][1], wa[s], ptr[s][g * inc[s]]);
  }
  // D[row = output k][col = facet 2t + c] -> scratch [facet][9], then each lane takes its facet
  const int k = lane >> 2;
  if (k < N1) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      scr[(8 * g + 2 * t) * 9 + k] = d[g][0];
      scr[(8 * g + 2 * t + 1) * 9 + k] = d[g][1];
    }
  }
  __syncwarp();
#pragma unroll
  for (int kk = 0; kk < N1; ++kk) acc[kk] = scr[lane * 9 + kk];
  __syncwarp();
}

// Stored mode: this facet's merged matrix streams from HBM (coalesced across the warp).
template <int N1>
__device__ __forceinline__ void apply_stored(const double* const (&nb)[7], const double* Ws, double (&acc)[N1]) {
  using C = Cfg<N1>;
  const uint64_t pol = evict_first_policy();
#pragma unroll
  for (int k = 0; k < N1; ++k) acc[k] = 0.0;
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

// Stored mode with each coupling block stored once (HDG_SYMSTORE).  Owned blocks per facet, in
// stream order:  h(i,j): q1 (diagonal), q2 = h(i,j+1), q5 = v(i,j), q6 = v(i+1,j)
//                v(i,j): q1, q2 = v(i+1,j), q4 = h(i-1,j+1), q6 = h(i,j+1)
// and the other three come transposed from their owners:
//   h(i,j): q0 <- h(i,j-1).q2,  q3 <- v(i,j-1).q6,  q4 <- v(i+1,j-1).q4
//   v(i,j): q0 <- v(i-1,j).q2,  q3 <- h(i-1,j).q6,  q5 <- h(i,j).q5
// (same lane or the neighbouring lane of the interleaved stream, so the reads stay coalesced;
// the owner's copy is read in the same tile, so the second read is an L2 hit).
template <int N1> __device__ __forceinline__ const double* wslot(const double* W, long long slot) {
  return W + (size_t)(slot >> 5) * Cfg<N1>::WSZ * 32 + (slot & 31);
}

template <int N1, bool VERT>
__device__ __forceinline__ void apply_stored_half(const double* const (&nb)[7], const double* own, const double* t0,
                                                  const double* t1, const double* t2, double (&acc)[N1]) {
  const uint64_t pol = evict_first_policy();
  constexpr int B = N1 * N1 * 32;   // one block of the interleaved stream
  constexpr int QO[4] = {1, 2, VERT ? 4 : 5, 6};
  constexpr int QT[3] = {0, 3, VERT ? 5 : 4};
#pragma unroll
  for (int k = 0; k < N1; ++k) acc[k] = 0.0;
#pragma unroll
  for (int qs = 0; qs < 4; ++qs) {
    double xv[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) xv[m] = nb[QO[qs]][m];
    const double* Wq = own + qs * B;
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        // the partner reads this block again (transposed) within the same tile: keep it in L2
        const double w = (N1 >= HDG_SYMSTORE_EF_MIN_N1) ? ld_stream(Wq + (k * N1 + m) * 32, pol)
                                                          : __ldg(Wq + (k * N1 + m) * 32);
        acc[k] = fma(w, xv[m], acc[k]);
      }
  }
  const double* tp[3] = {t0, t1, t2};
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    double xv[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) xv[m] = nb[QT[t]][m];
#pragma unroll
    for (int mm = 0; mm < N1; ++mm)       // owner's row mm = our input mm; its column k = our output k
#pragma unroll
      for (int k = 0; k < N1; ++k) acc[k] = fma(__ldg(tp[t] + (mm * N1 + k) * 32), xv[mm], acc[k]);
  }
}

// A horizontal facet h(i,j) and the vertical facet v(i,j) of the same thread in one pass over the
// half-stored stream, ordered so that both reads of every coupling block are close in time:
//   * h.q5 = v.q5^T is loaded once and feeds both accumulators;
//   * h.q6 / v.q2 are read again, transposed, by lane i+1 in the same loop iteration (one 8-byte
//     shift inside the same 256-byte line: an L1 hit, no second L2 / DRAM read);
//   * the three blocks owned by row j-1 (h.q2, v.q6, v.q4 of the row below) are read right after
//     this thread's own copies of the same three, so the warp of row j-1 and this warp touch them
//     one block apart (at p = 8 the separate h / v passes put ~100 MB of other traffic between
//     the two reads GPU-wide and the second read missed the L2: 1.55x DRAM bytes).
// Blocks nobody reads again (diagonals, q5, and the lane-shifted ones) carry the evict-first hint.
template <int N1>
__device__ __forceinline__ void apply_stored_pair(const double* const (&nh)[7], const double* const (&nv)[7],
                                                  const double* hown, const double* vown, const double* hd,
                                                  const double* vd, const double* vd1, const double* hw,
                                                  const double* vw, double (&ah)[N1], double (&av)[N1]) {
  const uint64_t pol = evict_first_policy();
  constexpr int B = N1 * N1 * 32;
#pragma unroll
  for (int k = 0; k < N1; ++k) ah[k] = av[k] = 0.0;
  // the warp's copy of one block is N1^2 * 256 contiguous bytes: pull the next step's own block into
  // L2 while this step computes (the loads then cost an L2 hit instead of a DRAM round trip)
  auto prefetch_block = [&](const double* W) {
#if HDG_PAIR_PREFETCH
    const char* base = reinterpret_cast<const char*>(W - (threadIdx.x & 31));
    constexpr int LINES = (N1 * N1 * 256 + 127) / 128;
#pragma unroll
    for (int l = 0; l < LINES; l += 32)
      if (l + (int)(threadIdx.x & 31) < LINES)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)(l + (threadIdx.x & 31)) * 128));
#endif
  };
  // own block W (acc += W x) followed by a transposed partner block P (acc2 += P^T x2)
  auto own_then_partner = [&](const double* W, const double* xo, double (&ao)[N1], const double* Pp, const double* xp,
                              double (&ap)[N1]) {
    double xa[N1], xb[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) { xa[m] = xo[m]; xb[m] = xp[m]; }
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int m = 0; m < N1; ++m) ao[k] = fma(__ldg(W + (k * N1 + m) * 32), xa[m], ao[k]);
#pragma unroll
    for (int mm = 0; mm < N1; ++mm)
#pragma unroll
      for (int k = 0; k < N1; ++k) ap[k] = fma(__ldg(Pp + (mm * N1 + k) * 32), xb[mm], ap[k]);
  };
  // own block and the neighbouring lane's copy of the same entries in one loop (L1 hit)
  auto own_and_shifted = [&](const double* W, const double* xo, double (&ao)[N1], const double* Ws, const double* xs,
                             double (&as)[N1]) {
    double xa[N1], xb[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) { xa[m] = xo[m]; xb[m] = xs[m]; }
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        const double w = __ldg(W + (k * N1 + m) * 32);
        const double ws = __ldg(Ws + (k * N1 + m) * 32);
        ao[k] = fma(w, xa[m], ao[k]);
        as[m] = fma(ws, xb[k], as[m]);
      }
  };
  prefetch_block(vown + 3 * B);
  own_then_partner(hown + 1 * B, nh[2], ah, hd + 1 * B, nh[0], ah);      // h.q2 ; h.q0 <- h(i,j-1).q2
  prefetch_block(vown + 2 * B);
  own_then_partner(vown + 3 * B, nv[6], av, vd + 3 * B, nh[3], ah);      // v.q6 ; h.q3 <- v(i,j-1).q6
  prefetch_block(hown + 2 * B);
  own_then_partner(vown + 2 * B, nv[4], av, vd1 + 2 * B, nh[4], ah);     // v.q4 ; h.q4 <- v(i+1,j-1).q4
  prefetch_block(hown + 3 * B);
  {                                                                      // h.q5 = v.q5^T: one load, two uses
    double xa[N1], xb[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) { xa[m] = nh[5][m]; xb[m] = nv[5][m]; }
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        const double w = ld_stream(hown + 2 * B + (k * N1 + m) * 32, pol);
        ah[k] = fma(w, xa[m], ah[k]);
        av[m] = fma(w, xb[k], av[m]);
      }
  }
  prefetch_block(vown + 1 * B);
  own_and_shifted(hown + 3 * B, nh[6], ah, hw + 3 * B, nv[3], av);       // h.q6 ; v.q3 <- h(i-1,j).q6
  prefetch_block(hown);
  prefetch_block(vown);
  own_and_shifted(vown + 1 * B, nv[2], av, vw + 1 * B, nv[0], av);       // v.q2 ; v.q0 <- v(i-1,j).q2
  {                                                                      // diagonal blocks
    double xa[N1], xb[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) { xa[m] = nh[1][m]; xb[m] = nv[1][m]; }
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        ah[k] = fma(ld_stream(hown + (k * N1 + m) * 32, pol), xa[m], ah[k]);
        av[k] = fma(ld_stream(vown + (k * N1 + m) * 32, pol), xb[m], av[k]);
      }
  }
}

// Per-warp ring of the merged stored pass.  `count` (chunks issued / consumed so far by this warp)
// runs on across the tiles of the persistent CTA and gives every chunk its stage and mbarrier parity.
struct PairRing {
  double* ring;
  uint64_t* bars;
  unsigned count;
};

// apply_stored_pair with the block rows streamed through the warp's TMA ring instead of per-thread
// register loads: the bytes in flight no longer depend on the registers left over by the two
// accumulators (the register version ran at 12 warps/SM with too few loads in flight: 59% of DRAM
// throughput although its traffic was down to 1.06x the stream).  Chunk sequence (block, row):
// the 11 blocks in the order of apply_stored_pair, N1 rows each; lane 0 issues chunk c + STAGES - 1
// when the warp has finished chunk c - 1.  Lane-shifted partner values come from the same staged
// row at lane - 1 / lane + 1; the one lane whose neighbour sits in the next slot group reads global
// memory directly.
template <int N1, int STAGES>
__device__ __forceinline__ void apply_stored_pair_ring(PairRing& pr, const double* const (&nh)[7],
                                                       const double* const (&nv)[7], const double* hown,
                                                       const double* vown, const double* hd, const double* vd,
                                                       const double* vd1, const double* hw, const double* vw,
                                                       double (&ah)[N1], double (&av)[N1]) {
  constexpr int B = N1 * N1 * 32, ROW = N1 * 32, NBLK = 11, NCH = NBLK * N1;
  // edge-lane values one row ahead, loaded by that lane only (n1 <= 7: p = 5 0.80 -> 0.85 of HBM), or
  // loaded in place by every lane (n1 >= 8, where the extra registers cost more: p = 8 0.76 vs 0.55)
  constexpr bool AHEAD = N1 <= HDG_PAIR_AHEAD_MAX_N1;
  const int lane = threadIdx.x & 31;
  // warp-uniform block bases (lane 0's slot of the group), in processing order
  const double* const blk[NBLK] = {hown - lane + 1 * B, hd - lane + 1 * B, vown - lane + 3 * B, vd - lane + 3 * B,
                                   vown - lane + 2 * B, vd - lane + 2 * B, hown - lane + 2 * B, hown - lane + 3 * B,
                                   vown - lane + 1 * B, hown - lane, vown - lane};
  const unsigned c0 = pr.count;
  auto issue = [&](int c) {
    if (c >= NCH || lane != 0) return;
    const unsigned g = c0 + c;
    uint64_t* bar = pr.bars + g % STAGES;
    mbar_arrive_expect_tx(bar, ROW * 8u);
    tma_load_1d(pr.ring + (g % STAGES) * ROW, blk[c / N1] + (c % N1) * ROW, ROW * 8u, bar);
  };
  auto wait = [&](int c) -> const double* {
    __syncwarp();                       // every lane has finished the stage that is refilled now
    fence_proxy_async();
    issue(c + STAGES - 1);
    const unsigned g = c0 + c;
    mbar_wait(pr.bars + g % STAGES, (g / STAGES) & 1u);
    return pr.ring + (g % STAGES) * ROW + lane;
  };
  __syncwarp();
  fence_proxy_async();
#pragma unroll
  for (int c = 0; c < STAGES - 1; ++c) issue(c);
#pragma unroll
  for (int k = 0; k < N1; ++k) ah[k] = av[k] = 0.0;
  int c = 0;
  // own block: acc[r] += row_r . x
  auto own = [&](const double* xo, double (&ao)[N1]) {
    double xa[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) xa[m] = xo[m];
#pragma unroll
    for (int r = 0; r < N1; ++r) {
      const double* q = wait(c++);
      double sacc = ao[r];
#pragma unroll
      for (int m = 0; m < N1; ++m) sacc = fma(q[m * 32], xa[m], sacc);
      ao[r] = sacc;
    }
  };
  // partner block (transposed): acc[k] += P[r][k] x[r]; shift = lane offset of the owner's slot.
  // The one lane whose owner sits in the next slot group loads its row from global memory, one row
  // ahead of its use (only that lane executes the loads).
  auto partner = [&](const double* xp, double (&ap)[N1], int shift, const double* edge) {
    double xb[N1], ev[AHEAD ? N1 : 1];
#pragma unroll
    for (int m = 0; m < N1; ++m) xb[m] = xp[m];
    const bool direct = (shift > 0 && lane == 31);
    if constexpr (!AHEAD) {
#pragma unroll
      for (int r = 0; r < N1; ++r) {
        const double* q = wait(c++);
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          const double v = direct ? __ldg(edge + (r * N1 + k) * 32) : q[k * 32 + shift];
          ap[k] = fma(v, xb[r], ap[k]);
        }
      }
      return;
    }
#pragma unroll
    for (int m = 0; m < (AHEAD ? N1 : 1); ++m) ev[m] = 0.0;
    if (direct) {
#pragma unroll
      for (int k = 0; k < (AHEAD ? N1 : 1); ++k) ev[k] = __ldg(edge + k * 32);
    }
#pragma unroll
    for (int r = 0; r < N1; ++r) {
      const double* q = wait(c++);
      double cur[N1];
#pragma unroll
      for (int k = 0; k < N1; ++k) cur[k] = ev[AHEAD ? k : 0];
      if (direct && r + 1 < N1) {
#pragma unroll
        for (int k = 0; k < (AHEAD ? N1 : 1); ++k) ev[k] = __ldg(edge + ((r + 1) * N1 + k) * 32);
      }
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        const double v = direct ? cur[k] : q[k * 32 + shift];
        ap[k] = fma(v, xb[r], ap[k]);
      }
    }
  };
  // own block whose rows the neighbouring lane also needs transposed: ao[r] += row_r . xo and
  // as[m] += W(lane - 1)[r][m] xs[r]; lane 0's neighbour is in the previous slot group (global loads,
  // one row ahead)
  auto own_and_shifted = [&](const double* xo, double (&ao)[N1], const double* xs, double (&as)[N1],
                             const double* edge) {
    double xa[N1], xb[N1], ev[AHEAD ? N1 : 1];
#pragma unroll
    for (int m = 0; m < N1; ++m) { xa[m] = xo[m]; xb[m] = xs[m]; }
    const bool direct = lane == 0;
    if constexpr (!AHEAD) {
#pragma unroll
      for (int r = 0; r < N1; ++r) {
        const double* q = wait(c++);
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          ao[r] = fma(q[m * 32], xa[m], ao[r]);
          const double ws = direct ? __ldg(edge + (r * N1 + m) * 32) : q[m * 32 - 1];
          as[m] = fma(ws, xb[r], as[m]);
        }
      }
      return;
    }
#pragma unroll
    for (int m = 0; m < (AHEAD ? N1 : 1); ++m) ev[m] = 0.0;
    if (direct) {
#pragma unroll
      for (int m = 0; m < (AHEAD ? N1 : 1); ++m) ev[m] = __ldg(edge + m * 32);
    }
#pragma unroll
    for (int r = 0; r < N1; ++r) {
      const double* q = wait(c++);
      double cur[N1];
#pragma unroll
      for (int m = 0; m < N1; ++m) cur[m] = ev[AHEAD ? m : 0];
      if (direct && r + 1 < N1) {
#pragma unroll
        for (int m = 0; m < (AHEAD ? N1 : 1); ++m) ev[m] = __ldg(edge + ((r + 1) * N1 + m) * 32);
      }
#pragma unroll
      for (int m = 0; m < N1; ++m) {      // ao and as may be the same accumulator (v.q2 / v.q0): no cached partial sums
        ao[r] = fma(q[m * 32], xa[m], ao[r]);
        const double ws = direct ? cur[m] : q[m * 32 - (direct ? 0 : 1)];
        as[m] = fma(ws, xb[r], as[m]);
      }
    }
  };
  own(nh[2], ah);                               // h.q2
  partner(nh[0], ah, 0, nullptr);               // h.q0 <- h(i,j-1).q2
  own(nv[6], av);                               // v.q6
  partner(nh[3], ah, 0, nullptr);               // h.q3 <- v(i,j-1).q6
  own(nv[4], av);                               // v.q4
  partner(nh[4], ah, 1, vd1 + 2 * B);           // h.q4 <- v(i+1,j-1).q4 (owner = lane + 1)
  {                                             // h.q5 = v.q5^T: one staged row, two uses
    double xa[N1], xb[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) { xa[m] = nh[5][m]; xb[m] = nv[5][m]; }
#pragma unroll
    for (int r = 0; r < N1; ++r) {
      const double* q = wait(c++);
      double sacc = ah[r];
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        const double w = q[m * 32];
        sacc = fma(w, xa[m], sacc);
        av[m] = fma(w, xb[r], av[m]);
      }
      ah[r] = sacc;
    }
  }
  own_and_shifted(nh[6], ah, nv[3], av, hw + 3 * B);   // h.q6 ; v.q3 <- h(i-1,j).q6
  own_and_shifted(nv[2], av, nv[0], av, vw + 1 * B);   // v.q2 ; v.q0 <- v(i-1,j).q2
  own(nh[1], ah);                               // diagonal blocks
  own(nv[1], av);
  pr.count = c0 + NCH;
}

template <int EPI, int N1> struct NOutOf { static constexpr int v = (EPI == EPI_RESPR) ? N1 - 1 : N1; };

// Per-facet epilogue: the facet's output values (y | r | x_out | r_coarse) into `o`.
template <int N1, bool STORED, int EPI>
__device__ __forceinline__ void facet_epilogue(const MvArgs& a, int blk, const double* xf, const double* Dc,
                                               const double* Ds, const double (&acc)[N1], double (&o)[N1],
                                               double& nrm, const double* bsm = nullptr) {
  if constexpr (EPI == EPI_Y) {
#pragma unroll
    for (int k = 0; k < N1; ++k) o[k] = acc[k];
  } else {
    double r[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) r[k] = (bsm ? bsm[k] : __ldg(a.b + blk * N1 + k)) - acc[k];
    if constexpr (EPI == EPI_RES) {
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        nrm = fma(r[k], r[k], nrm);
        o[k] = r[k];
      }
    } else if constexpr (EPI == EPI_BJ) {
      double dinv[N1 * N1];
      if constexpr (!STORED) {
#pragma unroll
        for (int t = 0; t < N1 * N1; ++t) dinv[t] = Dc[t];
      } else {
        const uint64_t pol = evict_first_policy();
#pragma unroll
        for (int t = 0; t < N1 * N1; ++t) dinv[t] = ld_stream(Ds + (size_t)t * 32, pol);
      }
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) s = fma(dinv[k * N1 + m], r[m], s);
        o[k] = fma(a.omega, s, xf[k]);
      }
    } else {  // EPI_RESPR: r_coarse = V^T r  (multigrid.py:399, p-level)
      constexpr int NC = N1 - 1;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < N1; ++k) s = fma(a.V[k * NC + c], r[k], s);
        o[c] = s;
      }
      o[N1 - 1] = 0.0;
    }
  }
}

// One tile: thread (tx, w) owns, for f < F, horizontal facet h(i0+tx, j0+F w+f) (bottom of that
// element) and vertical facet v(i0+tx, j0+F w+f) (its left side); consecutive rows share
// stencil blocks (the compiler CSEs the repeated shared-memory loads).  Outputs are staged through
// shared memory (the consumed x buffer) and written back as contiguous runs.
// h-facet outputs of one warp row (32 consecutive facets = one contiguous run in HBM):
// transposed through the warp's private scratch and stored coalesced, right after compute
template <int N1, int NO>
__device__ __forceinline__ void store_h_row(const MvArgs& a, double* scr, int i0, int j, const double (&o)[N1],
                                            int lane) {
  if (a.out == nullptr || j < 1 || j > a.ny - 1) return;  // warp-uniform
#ifdef HDG_EXP_NOHSTORE
  if (a.nx > 0) return;
#endif
#pragma unroll
  for (int k = 0; k < NO; ++k) scr[lane * NO + k] = o[k];
  __syncwarp();
  const int count = min(TX, a.nx - i0) * NO;
  double* dst = a.out + hblk(a.nx, i0, j) * NO;
#pragma unroll
  for (int q = 0; q < NO; ++q)
    if (lane + 32 * q < count) dst[lane + 32 * q] = scr[lane + 32 * q];
  __syncwarp();
}

template <int N1, bool STORED, int EPI>
__device__ __forceinline__ void compute_tile(PairRing& pring, const MvArgs& a, const SharedOp<(STORED ? 1 : N1)>& op,
                                             double* buf, double* scr, int i0, int j0, double& nrm) {
  using C = Cfg<N1, STORED>;
  constexpr int F = C::F;
  constexpr int NO = NOutOf<EPI, N1>::v;
  const int tx = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = i0 + tx, ii = tx + 1;
  const double* Hs = buf;
  const double* Vs = buf + C::HSZ;
  // run shifts: H row r starts at parity of ((j0-2+r) nx + i0-1) N1, V column c likewise
  const int hpar0 = h_run_start<N1>(a, i0, j0, 0), hstep = a.nx * N1;
  auto H = [&](int r, int c) { return Hs + r * C::RS + ((hpar0 + r * hstep) & 1) + c * C::S; };
  auto V = [&](int c, int r) { return Vs + (r * C::VCOLS + c) * C::SV; };
  if constexpr (!STORED && EPI == EPI_BJ) {
    if (a.w_first != 0.0) {
      // Two Jacobi steps from x = 0 in one pass (multigrid.py:400 then the first sweep): the
      // tile was staged from b, so every staged block becomes x1 = w1 D^-1 b in place
      // (Dirichlet / outside blocks are 0 and stay 0), then the sweep below runs on x1.
      auto dmul = [&](double* blk, const double* D) {
        double r[N1];
#pragma unroll
        for (int k = 0; k < N1; ++k) r[k] = blk[k];
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) s = fma(D[k * N1 + m], r[m], s);
          blk[k] = a.w_first * s;
        }
      };
      for (int t = threadIdx.x; t < C::HROWS * C::HCOLS; t += C::NTH) {
        const int r = t / C::HCOLS, c = t - r * C::HCOLS;
        dmul(const_cast<double*>(H(r, c)), op.Dh);
      }
      for (int t = threadIdx.x; t < C::VROWS * C::VCOLS; t += C::NTH) {
        const int r = t / C::VCOLS, c = t - r * C::VCOLS;
        dmul(const_cast<double*>(V(c, r)), op.Dv);
      }
      consumer_sync<C::NTH>();
    }
  }
  if constexpr (EPI == EPI_BJ && N1 >= 2) {
    if (a.pec != nullptr) {
      // Prolongation fused into the first post-smoothing sweep (multigrid.py:403 then 405):
      // every staged real facet block becomes x + V ec (p-transfer, facet-local), so the
      // prolonged iterate is never written to memory.  Dirichlet / outside blocks stay 0.
      constexpr int NC = N1 - 1;
      auto padd = [&](double* blk, long long cb) {
        double e[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) e[c] = __ldg(a.pec + cb * NC + c);
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double s = blk[k];
#pragma unroll
          for (int c = 0; c < NC; ++c) s = fma(a.V[k * NC + c], e[c], s);
          blk[k] = s;
        }
      };
      for (int t = threadIdx.x; t < C::HROWS * C::HCOLS; t += C::NTH) {
        const int r = t / C::HCOLS, c = t - r * C::HCOLS;
        const int ig = i0 - 1 + c, jg = j0 - 1 + r;
        if (ig >= 0 && ig < a.nx && jg >= 1 && jg <= a.ny - 1) padd(const_cast<double*>(H(r, c)), hblk(a.nx, ig, jg));
      }
      for (int t = threadIdx.x; t < C::VROWS * C::VCOLS; t += C::NTH) {
        const int c = t / C::VROWS, r = t - c * C::VROWS;   // consecutive threads walk a column
        const int ig = i0 - 1 + c, jg = j0 - 1 + r;
        if (ig >= 1 && ig <= a.nx - 1 && jg >= 0 && jg < a.ny) padd(const_cast<double*>(V(c, r)), vblk(a.nh, a.ny, ig, jg));
      }
      consumer_sync<C::NTH>();
    }
  }
  double ov[F][N1];
  double ohs[STORED ? F : 1][N1];   // stored mode: h outputs wait for the CTA-staged write
  constexpr bool PAIR = STORED && HDG_SYMSTORE && F == 1 && N1 >= HDG_PAIR_MIN_N1;
  double accv_pair[PAIR ? N1 : 1];  // vertical facet's operator value from the merged h/v pass
  bool pair_done = false;
  {
  // ---- horizontal facets: owners (i, j-1) [TOP rows] and (i, j) [BOTTOM rows]
  {
    const double* nb[F][7];
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const int jj = F * w + f + 1;
      nb[f][0] = H(jj - 1, ii); nb[f][1] = H(jj, ii); nb[f][2] = H(jj + 1, ii);
      nb[f][3] = V(ii, jj - 1); nb[f][4] = V(ii + 1, jj - 1); nb[f][5] = V(ii, jj); nb[f][6] = V(ii + 1, jj);
    }
    if constexpr (!STORED) {
      double acc[F][N1];
      if constexpr (C::DMMA) {
        double wa[C::KS];
        dmma_wfrag<N1>(op.Wh, wa, tx);
#pragma unroll
        for (int f = 0; f < F; ++f) apply_dmma_row<N1, false>(Hs, Vs, hpar0, hstep, F * w + f + 1, wa, scr, acc[f], tx);
      } else {
        if constexpr (HDG_SHARED_SYM) apply_shared_sym<N1, F>(nb, op.Wh, acc);
        else apply_shared<N1, F>(nb, op.Wh, acc);
      }
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const int j = j0 + F * w + f;
        const bool rowok = (j >= 1 && j <= a.ny - 1);   // warp-uniform
        double oh[N1];
        const double* bsm = nullptr;
        if constexpr (EPI != EPI_Y) {
          // the row's right-hand side is one contiguous run: load it coalesced into the
          // warp scratch, then each lane reads its facet's n1 values
          if (rowok) {
            const int count = min(TX, a.nx - i0) * N1;
            const double* src = a.b + hblk(a.nx, i0, j) * N1;
#pragma unroll
            for (int q = 0; q < N1; ++q)
              if (tx + 32 * q < count) scr[tx + 32 * q] = __ldg(src + tx + 32 * q);
            __syncwarp();
            bsm = scr + tx * N1;
          }
        }
        if (i < a.nx && rowok)
          facet_epilogue<N1, false, EPI>(a, hblk(a.nx, i, j), nb[f][1], op.Dh, nullptr, acc[f], oh, nrm, bsm);
        if constexpr (EPI != EPI_Y) __syncwarp();
        store_h_row<N1, NO>(a, scr, i0, j, oh, tx);
      }
    } else {
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const int j = j0 + F * w + f;
        if (j >= 1 && j <= a.ny - 1) {  // warp-uniform; lanes i >= nx read zero padding slots
          const long long grp = ((long long)j * a.nxp + i0) >> 5;
          double acc[N1];
          if constexpr (PAIR) {
            // rows 1 .. ny-1 hold both an h and a v facet per slot: one merged pass
            const int jj = F * w + f + 1;
            const double* nv[7] = {V(ii - 1, jj), V(ii, jj), V(ii + 1, jj), H(jj, ii - 1), H(jj + 1, ii - 1),
                                   H(jj, ii), H(jj + 1, ii)};
            const long long sl = (long long)j * a.nxp + i, sd = sl - a.nxp, sw = sl - 1;
            if constexpr (C::PRING)
              apply_stored_pair_ring<N1, C::RSTAGES>(pring, nb[f], nv, wslot<N1>(a.Wh, sl), wslot<N1>(a.Wv, sl),
                                                     wslot<N1>(a.Wh, sd), wslot<N1>(a.Wv, sd), wslot<N1>(a.Wv, sd + 1),
                                                     wslot<N1>(a.Wh, sw), wslot<N1>(a.Wv, sw), acc, accv_pair);
            else
              apply_stored_pair<N1>(nb[f], nv, wslot<N1>(a.Wh, sl), wslot<N1>(a.Wv, sl), wslot<N1>(a.Wh, sd),
                                    wslot<N1>(a.Wv, sd), wslot<N1>(a.Wv, sd + 1), wslot<N1>(a.Wh, sw),
                                    wslot<N1>(a.Wv, sw), acc, accv_pair);
            pair_done = true;
          } else if constexpr (HDG_SYMSTORE) {
            constexpr int B = N1 * N1 * 32;
            const long long sl = (long long)j * a.nxp + i, sd = sl - a.nxp;   // row j-1
            apply_stored_half<N1, false>(nb[f], wslot<N1>(a.Wh, sl), wslot<N1>(a.Wh, sd) + 1 * B,
                                         wslot<N1>(a.Wv, sd) + 3 * B, wslot<N1>(a.Wv, sd + 1) + 2 * B, acc);
          } else {
            apply_stored<N1>(nb[f], a.Wh + (size_t)grp * C::WSZ * 32 + tx, acc);
          }
          if (i < a.nx)
            facet_epilogue<N1, true, EPI>(a, hblk(a.nx, i, j), nb[f][1], nullptr,
                                          a.Dh + (size_t)grp * C::DSZ * 32 + tx, acc, ohs[f], nrm);
        }
      }
    }
  }
  // ---- vertical facets: owners (i-1, j) [RIGHT rows] and (i, j) [LEFT rows]
  {
    const double* nb[F][7];
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const int jj = F * w + f + 1;
      nb[f][0] = V(ii - 1, jj); nb[f][1] = V(ii, jj); nb[f][2] = V(ii + 1, jj);
      nb[f][3] = H(jj, ii - 1); nb[f][4] = H(jj + 1, ii - 1); nb[f][5] = H(jj, ii); nb[f][6] = H(jj + 1, ii);
    }
    if constexpr (!STORED) {
      double acc[F][N1];
      if constexpr (C::DMMA) {
        double wa[C::KS];
        dmma_wfrag<N1>(op.Wv, wa, tx);
#pragma unroll
        for (int f = 0; f < F; ++f) apply_dmma_row<N1, true>(Hs, Vs, hpar0, hstep, F * w + f + 1, wa, scr, acc[f], tx);
      } else {
        if constexpr (HDG_SHARED_SYM) apply_shared_sym<N1, F>(nb, op.Wv, acc);
        else apply_shared<N1, F>(nb, op.Wv, acc);
      }
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const int j = j0 + F * w + f;
        if (i >= 1 && i <= a.nx - 1 && j < a.ny)
          facet_epilogue<N1, false, EPI>(a, vblk(a.nh, a.ny, i, j), nb[f][1], op.Dv, nullptr, acc[f], ov[f], nrm,
                                         C::template stage_b<EPI>() ? buf + C::BUF + ((F * w + f) * TX + tx) * C::SB
                                                                    : nullptr);
      }
    } else {
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const int j = j0 + F * w + f;
        if (j < a.ny) {
          const long long grp = ((long long)j * a.nxp + i0) >> 5;
          double acc[N1];
          if (PAIR && pair_done) {
#pragma unroll
            for (int k = 0; k < N1; ++k) acc[k] = accv_pair[PAIR ? k : 0];
          } else if constexpr (HDG_SYMSTORE) {
            constexpr int B = N1 * N1 * 32;
            const long long sl = (long long)j * a.nxp + i, sw = sl > 0 ? sl - 1 : 0;   // column i-1
            apply_stored_half<N1, true>(nb[f], wslot<N1>(a.Wv, sl), wslot<N1>(a.Wv, sw) + 1 * B,
                                        wslot<N1>(a.Wh, sw) + 3 * B, wslot<N1>(a.Wh, sl) + 2 * B, acc);
          } else {
            apply_stored<N1>(nb[f], a.Wv + (size_t)grp * C::WSZ * 32 + tx, acc);
          }
          if (i >= 1 && i <= a.nx - 1)
            facet_epilogue<N1, true, EPI>(a, vblk(a.nh, a.ny, i, j), nb[f][1], nullptr,
                                          a.Dv + (size_t)grp * C::DSZ * 32 + tx, acc, ov[f], nrm,
                                          C::template stage_b<EPI>() ? buf + C::BUF + ((F * w + f) * TX + tx) * C::SB
                                                                     : nullptr);
        }
      }
    }
  }
  }
  // ---- outputs -> shared (x buffer is consumed) -> contiguous global runs
  consumer_sync<C::NTH>();
  double* Yv = buf;                       // [col tx][row r][NO], column stride YCS (odd)
  double* Yh = buf + TX * C::YCS;         // stored mode: [row r][tx][NO]
#pragma unroll
  for (int f = 0; f < F; ++f) {
    const int r = F * w + f;
#pragma unroll
    for (int k = 0; k < NO; ++k) {
      Yv[tx * C::YCS + r * NO + k] = ov[f][k];
      if constexpr (STORED) Yh[(r * TX + tx) * NO + k] = ohs[f][k];
    }
  }
  consumer_sync<C::NTH>();
  if (a.out == nullptr) return;  // norm-only residual
#ifdef HDG_EXP_NOOUT
  if (a.nx > 0) return;
#endif
  const int lane = tx;
  if constexpr (STORED) {
    // h rows: facets h(i0 .. i0+TX-1, j) -> blocks (j-1)*nx + i, contiguous
    const int hcount = min(TX, a.nx - i0) * NO;
#pragma unroll
    for (int rr = 0; rr < C::TY / C::NW; ++rr) {
      const int r = w + rr * C::NW;
      const int j = j0 + r;
      if (j >= 1 && j <= a.ny - 1) {
        double* dst = a.out + hblk(a.nx, i0, j) * NO + lane;
        const double* src = Yh + r * TX * NO + lane;
#pragma unroll
        for (int q = 0; q < (TX * NO + 31) / 32; ++q)
          if (lane + 32 * q < hcount) dst[32 * q] = src[32 * q];
      }
    }
  }
  // v columns: facets v(i, j0 .. j0+TY-1) -> blocks nh + (i-1)*ny + j, contiguous
  const int vcount = min(C::TY, a.ny - j0) * NO;
#pragma unroll
  for (int cc = 0; cc < TX / C::NW; ++cc) {
    const int c = w + cc * C::NW;
    const int iv = i0 + c;
    if (iv >= 1 && iv <= a.nx - 1) {
      double* dst = a.out + vblk(a.nh, a.ny, iv, j0) * NO + lane;
      const double* src = Yv + c * C::YCS + lane;
#pragma unroll
      for (int q = 0; q < (C::TY * NO + 31) / 32; ++q)
        if (lane + 32 * q < vcount) dst[32 * q] = src[32 * q];
    }
  }
}

// Persistent, double-buffered: CTA c walks tiles c, c + grid, ...; the next tile's stencil
// values stream into the other shared buffer (cp.async group) while this tile computes.
template <int N1, bool STORED, int EPI>
__global__ void __launch_bounds__(Cfg<N1, STORED>::NTH, Cfg<N1, STORED>::MINB)
trace_apply_kernel(const MvArgs a, const __grid_constant__ SharedOp<(STORED ? 1 : N1)> op) {
  using C = Cfg<N1, STORED>;
  extern __shared__ __align__(16) double smem[];
  const int tiles_x = (a.nx + TX - 1) / TX;
  const int ntiles = tiles_x * ((a.ny + C::TY - 1) / C::TY);
  constexpr int NB = C::NBUF;
  constexpr bool SBV = C::template stage_b<EPI>();
  constexpr int BS = C::template bufs<EPI>();
  __shared__ __align__(8) uint64_t bars[NB];
  __shared__ __align__(8) uint64_t rbars[C::PRING ? C::NW * C::RSTAGES : 1];
  double nrm = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NB; ++q) mbar_init(&bars[q], C::NW + C::NTH);  // lane-0 expect_tx + per-thread LDGSTS arrivals
    if constexpr (C::PRING) {
      for (int q = 0; q < C::NW * C::RSTAGES; ++q) mbar_init(&rbars[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  grid_dependency_wait();
  PairRing pring{smem + ((C::template tile_doubles_epi<EPI>() + 3) & ~3) + (threadIdx.x >> 5) * (C::RSTAGES * C::RROW),
                 rbars + (C::PRING ? (threadIdx.x >> 5) * C::RSTAGES : 0), 0u};
  // ring of NB stage buffers: tiles blockIdx.x + it*grid; prefetch distance NB-1
#pragma unroll
  for (int q = 0; q < NB - 1; ++q) {
    const int t = blockIdx.x + q * gridDim.x;
    if (t < ntiles)
      stage_tile<N1, STORED, SBV>(a, smem + q * BS, (t % tiles_x) * TX, (t / tiles_x) * C::TY, &bars[q]);
  }
  int slot = 0;
  unsigned phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int pre = tile + (NB - 1) * gridDim.x;
    if (pre < ntiles) {
      const int ps = (slot + NB - 1) % NB;
      stage_tile<N1, STORED, SBV>(a, smem + ps * BS, (pre % tiles_x) * TX, (pre / tiles_x) * C::TY, &bars[ps]);
    }
    mbar_wait(&bars[slot], phase);
    __syncthreads();
    compute_tile<N1, STORED, EPI>(pring, a, op, smem + slot * BS, smem + NB * BS + (threadIdx.x >> 5) * C::WSCR,
                                  (tile % tiles_x) * TX, (tile / tiles_x) * C::TY, nrm);
    __syncthreads();
    if (++slot == NB) { slot = 0; phase ^= 1u; }
  }
  if constexpr (EPI == EPI_RES) {
    if (a.partials != nullptr) {
      __shared__ double red[C::NW];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < C::NW; ++q) t += red[q];
        a.partials[blockIdx.x] = t;
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

// Slot rows [j0, j1) of the stream (all rows: j0 = 0, j1 = ny).  S holds the element blocks of
// element rows [erow0, ...): a slot row j needs element rows j - 1 (horizontal facet below) and j,
// so a chunk of slot rows [j0, j1) is complete given element rows [max(j0 - 1, 0), j1).
template <int N1>
__global__ void relayout_kernel(const double* __restrict__ S, int nx, int ny, int nxp, bool vert,
                                double* __restrict__ W, bool bcast = false, int j0 = 0, int j1 = -1,
                                int erow0 = 0) {
  using C = Cfg<N1>;
  if (j1 < 0) j1 = ny;
  const long long nslots = (long long)(j1 - j0) * nxp;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= nslots * C::WSZ) return;
  // thread -> (group, entry, lane): consecutive threads write consecutive addresses
  const int lane = tid & 31;
  const long long rest = tid >> 5;
  const int idx = (int)(rest % C::WSZ);
  const long long grp = rest / C::WSZ + (long long)j0 * nxp / 32;   // nxp is a multiple of 32
  const long long slot = grp * 32 + lane;
  const int j = (int)(slot / nxp), i = (int)(slot % nxp);
  const bool valid = vert ? (i >= 1 && i <= nx - 1 && j < ny) : (i < nx && j >= 1 && j <= ny - 1);
  long long e1 = 0, e2 = 0;
  if (valid) {
    e1 = vert ? ((long long)(j - erow0) * nx + (i - 1)) : ((long long)(j - 1 - erow0) * nx + i);
    e2 = (long long)(j - erow0) * nx + i;
    if (bcast) e1 = e2 = 0;   // one block for every element (asymmetric constant operator)
  }
  const int L = 4 * N1;
  int q = idx / (N1 * N1);
  const int k = (idx / N1) % N1, m = idx % N1;
  if (HDG_SYMSTORE) q = (q == 0) ? 1 : (q == 1) ? 2 : (q == 2) ? (vert ? 4 : 5) : 6;   // owned blocks
  double v = 0.0;
  if (valid) {
    int w1, r1, c1, w2, r2, c2;
    merged_entry_src(vert, q, k, m, N1, w1, r1, c1, w2, r2, c2);
    v = S[((w1 ? e2 : e1) * L + r1) * L + c1];
    if (w2 >= 0) v += S[((w2 ? e2 : e1) * L + r2) * L + c2];
  }
  W[(grp * C::WSZ + idx) * 32 + lane] = v;
}

// max |S - S^T| and max |S| over all element blocks (atomicMax on the bit patterns of
// non-negative doubles): the half-stored stream requires a symmetric operator
template <int N1>
__global__ void block_asym_kernel(const double* __restrict__ S, long long E, unsigned long long* out) {
  constexpr int L = 4 * N1;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double asym = 0.0, mag = 0.0;
  if (tid < E * L * L) {
    const long long e = tid / (L * L);
    const int r = (int)((tid / L) % L), c = (int)(tid % L);
    const double a = S[(e * L + r) * L + c], b = S[(e * L + c) * L + r];
    asym = fabs(a - b);
    mag = fabs(a);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
    mag = fmax(mag, __shfl_xor_sync(0xffffffffu, mag, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, (unsigned long long)__double_as_longlong(asym));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(mag));
  }
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
// Meshes may be row WINDOWS of the global fine / coarse meshes (multi-GPU strips): the fine
// window has nyf rows starting at global row jf0, the coarse window nyc rows from jc0; on one
// GPU jf0 = jc0 = 0 and nyf = 2 nyc.  Facets whose transfer needs data outside the windows are
// left untouched (prolongation) or written as 0 (restriction): those are ghost facets, never owned.
struct HArgs {
  int nxc, nyc;           // coarse window (x: whole mesh)
  int nyf;                // fine window rows
  int jf0, jc0;           // global row of window row 0 (fine, coarse)
  long long nhf, nhc;     // interior horizontal block counts of the windows
  double halves[8];
  const double* cross;    // device, (nsets, 4, 2, 8)
  int shared_cross;       // 1 => one set for every coarse element (else one per window element)
  double cross_c[64];     // shared_cross: the one set, read as kernel-parameter constants
};

template <bool SC>
__device__ __forceinline__ const double* hcross(const HArgs& h, int I, int Jl, int cf) {
  if constexpr (SC) return h.cross_c + cf * 16;
  const long long set = (long long)Jl * h.nxc + I;
  return h.cross + (set * 4 + cf) * 16;
}

// SM = true: the vectors live in shared memory (the fused coarse tail below), plain loads;
// otherwise read-only global loads through the texture path.
template <bool SM> __device__ __forceinline__ double vld(const double* p) {
  if constexpr (SM) return *p; else return __ldg(p);
}
template <bool SM> __device__ __forceinline__ double2 vld2(const double2* p) {
  if constexpr (SM) return *p; else return __ldg(p);
}
// coarse side value (2 doubles) of coarse window element (I, Jl), side s; zero when the side is
// a Dirichlet facet or outside the window
template <bool SM>
__device__ __forceinline__ void coarse_side(const HArgs& h, const double* ec, int I, int Jl, int s, double* v) {
  long long blk = -1;
  if (s == 0 && Jl >= 1) blk = (long long)(Jl - 1) * h.nxc + I;
  if (s == 2 && Jl + 1 <= h.nyc - 1) blk = (long long)Jl * h.nxc + I;
  if (s == 3 && I >= 1) blk = h.nhc + (long long)(I - 1) * h.nyc + Jl;
  if (s == 1 && I + 1 <= h.nxc - 1) blk = h.nhc + (long long)I * h.nyc + Jl;
  if (blk >= 0) {
    const double2 e = vld2<SM>(reinterpret_cast<const double2*>(ec) + blk);
    v[0] = e.x; v[1] = e.y;
  } else {
    v[0] = 0.0; v[1] = 0.0;
  }
}

// fine window facet t (n1 = 2, one double2 per facet) += its prolongation from the coarse level
template <bool SM, bool SC>
__device__ __forceinline__ void h_prolong_add_one(const HArgs& h, const double* __restrict__ ec,
                                                  double* __restrict__ xf, long long t) {
  using IT = typename std::conditional<SM, int, long long>::type;   // 32-bit index math for small levels
  const IT nxf = 2 * h.nxc, nyf = h.nyf, nhf = (IT)h.nhf, tt = (IT)t;
  double add[2] = {0.0, 0.0};
  bool half;
  int I, Jl, hf, cf;
  long long cb = 0;
  if (tt < nhf) {  // fine h(i, jl), block (jl-1)*nxf + i
    const int jg = (int)(tt / nxf) + 1 + h.jf0, i = (int)(tt % nxf);
    I = i >> 1;
    half = (jg & 1) == 0;
    if (half) {
      Jl = (jg >> 1) - h.jc0;
      if (Jl < 1 || Jl > h.nyc - 1) return;
      hf = i & 1;
      cb = (long long)(Jl - 1) * h.nxc + I;
    } else {
      Jl = ((jg - 1) >> 1) - h.jc0;
      if (Jl < 0 || Jl >= h.nyc) return;
      cf = (i & 1) ? 3 : 2;
    }
  } else {          // fine v(i, jl), block nhf + (i-1)*nyf + jl
    const IT u = tt - nhf;
    const int i = (int)(u / nyf) + 1, jg = (int)(u % nyf) + h.jf0;
    Jl = (jg >> 1) - h.jc0;
    if (Jl < 0 || Jl >= h.nyc) return;
    half = (i & 1) == 0;
    if (half) { I = i >> 1; hf = jg & 1; cb = h.nhc + (long long)(I - 1) * h.nyc + Jl; }
    else { I = (i - 1) >> 1; cf = (jg & 1) ? 1 : 0; }
  }
  if (half) {
    const double2 e = vld2<SM>(reinterpret_cast<const double2*>(ec) + cb);
    for (int k = 0; k < 2; ++k) add[k] = h.halves[hf * 4 + k * 2] * e.x + h.halves[hf * 4 + k * 2 + 1] * e.y;
  } else {
    const double* tm = hcross<SC>(h, I, Jl, cf);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      double v[2];
      coarse_side<SM>(h, ec, I, Jl, s, v);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if constexpr (SC) add[k] += tm[k * 8 + s * 2] * v[0] + tm[k * 8 + s * 2 + 1] * v[1];
        else add[k] += __ldg(tm + k * 8 + s * 2) * v[0] + __ldg(tm + k * 8 + s * 2 + 1) * v[1];
      }
    }
  }
  double2* xp = reinterpret_cast<double2*>(xf) + t;
  double2 x = *xp;
  x.x += add[0];
  x.y += add[1];
  *xp = x;
}

static __global__ void h_prolong_add_kernel(const __grid_constant__ HArgs h, const double* __restrict__ ec,
                                     double* __restrict__ xf) {
  const long long nvf = (long long)(2 * h.nxc - 1) * h.nyf;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  grid_dependency_wait();
  if (t >= h.nhf + nvf) return;
  if (h.shared_cross) h_prolong_add_one<false, true>(h, ec, xf, t);
  else h_prolong_add_one<false, false>(h, ec, xf, t);
}

// fine window blocks of h(i, jg) / v(i, jg) (global row jg), -1 when outside the window
__device__ __forceinline__ long long fine_h(const HArgs& h, int i, int jg) {
  const int jl = jg - h.jf0;
  return (jl >= 1 && jl <= h.nyf - 1) ? (long long)(jl - 1) * (2 * h.nxc) + i : -1;
}
__device__ __forceinline__ long long fine_v(const HArgs& h, int i, int jg) {
  const int jl = jg - h.jf0;
  return (jl >= 0 && jl < h.nyf) ? h.nhf + (long long)(i - 1) * h.nyf + jl : -1;
}

// contribution of coarse element (I, Jl)'s 4 cross facets to its side-s coarse dofs
template <bool SM, bool SC>
__device__ __forceinline__ bool cross_restrict(const HArgs& h, const double* rf, int I, int Jl, int s, double* acc) {
  const int J = Jl + h.jc0;
  const long long cfb[4] = {fine_v(h, 2 * I + 1, 2 * J),       // right of SW = v(2I+1, 2J)
                            fine_v(h, 2 * I + 1, 2 * J + 1),   // right of NW = v(2I+1, 2J+1)
                            fine_h(h, 2 * I, 2 * J + 1),       // top of SW   = h(2I, 2J+1)
                            fine_h(h, 2 * I + 1, 2 * J + 1)};  // top of SE   = h(2I+1, 2J+1)
  if (cfb[0] < 0 || cfb[1] < 0 || cfb[2] < 0 || cfb[3] < 0 || Jl < 0 || Jl >= h.nyc) return false;
#pragma unroll
  for (int cf = 0; cf < 4; ++cf) {
    const double* tm = hcross<SC>(h, I, Jl, cf);
    const double r0 = vld<SM>(rf + 2 * cfb[cf]), r1 = vld<SM>(rf + 2 * cfb[cf] + 1);
    for (int c = 0; c < 2; ++c) acc[c] += tm[0 * 8 + s * 2 + c] * r0 + tm[1 * 8 + s * 2 + c] * r1;
  }
  return true;
}

template <bool SM, bool SC>
__device__ __forceinline__ void h_restrict_one(const HArgs& h, const double* __restrict__ rf,
                                               double* __restrict__ rc, long long t) {
  using IT = typename std::conditional<SM, int, long long>::type;   // 32-bit index math for small levels
  const IT tt = (IT)t, nhc = (IT)h.nhc;
  double acc[2] = {0.0, 0.0};
  bool ok = true;
  long long kf[2];
  if (tt < nhc) {  // coarse h(I, Jl)
    const int Jl = (int)(tt / h.nxc) + 1, I = (int)(tt % h.nxc);
    const int J = Jl + h.jc0;
    kf[0] = fine_h(h, 2 * I, 2 * J);          // children: fine h(2I, 2J), h(2I+1, 2J)
    kf[1] = fine_h(h, 2 * I + 1, 2 * J);
    ok = kf[0] >= 0 && kf[1] >= 0;
    if (ok) {
      for (int hf = 0; hf < 2; ++hf) {
        const double r0 = vld<SM>(rf + 2 * kf[hf]), r1 = vld<SM>(rf + 2 * kf[hf] + 1);
        for (int c = 0; c < 2; ++c) acc[c] += h.halves[hf * 4 + 0 * 2 + c] * r0 + h.halves[hf * 4 + 1 * 2 + c] * r1;
      }
      ok = cross_restrict<SM, SC>(h, rf, I, Jl - 1, 2, acc)   // element below: this facet is its TOP side
           && cross_restrict<SM, SC>(h, rf, I, Jl, 0, acc);   // element above: BOTTOM side
    }
  } else {          // coarse v(I, Jl)
    const IT u = tt - nhc;
    const int I = (int)(u / h.nyc) + 1, Jl = (int)(u % h.nyc);
    const int J = Jl + h.jc0;
    kf[0] = fine_v(h, 2 * I, 2 * J);          // children: fine v(2I, 2J), v(2I, 2J+1)
    kf[1] = fine_v(h, 2 * I, 2 * J + 1);
    ok = kf[0] >= 0 && kf[1] >= 0;
    if (ok) {
      for (int hf = 0; hf < 2; ++hf) {
        const double r0 = vld<SM>(rf + 2 * kf[hf]), r1 = vld<SM>(rf + 2 * kf[hf] + 1);
        for (int c = 0; c < 2; ++c) acc[c] += h.halves[hf * 4 + 0 * 2 + c] * r0 + h.halves[hf * 4 + 1 * 2 + c] * r1;
      }
      ok = cross_restrict<SM, SC>(h, rf, I - 1, Jl, 1, acc)   // element left: RIGHT side
           && cross_restrict<SM, SC>(h, rf, I, Jl, 3, acc);   // element right: LEFT side
    }
  }
  rc[2 * t] = ok ? acc[0] : 0.0;
  rc[2 * t + 1] = ok ? acc[1] : 0.0;
}

static __global__ void h_restrict_kernel(const __grid_constant__ HArgs h, const double* __restrict__ rf,
                                  double* __restrict__ rc) {
  const long long nvc = (long long)(h.nxc - 1) * h.nyc;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  grid_dependency_wait();
  if (t >= h.nhc + nvc) return;
  if (h.shared_cross) h_restrict_one<false, true>(h, rf, rc, t);
  else h_restrict_one<false, false>(h, rf, rc, t);
}

// ---------------------------------------------------------------------------- small kernels
// dense y = M b, warp per row (coarsest level, multigrid.py:209-212)
static __global__ void dense_gemv_kernel(const double* __restrict__ M, const double* __restrict__ b,
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
static __global__ void dot_partials_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
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

static __global__ void sum_partials_kernel(const double* __restrict__ partials, int n, double* __restrict__ out) {
  // one warp; fixed order => bitwise deterministic
  double s = 0.0;
  for (int t = threadIdx.x; t < n; t += 32) s += partials[t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *out = s;
}

// ------------------------------------------------------------------- Jacobi step from x = 0
// First smoothing sweep of a coarse-level visit starts from x = 0 (multigrid.py:400): the
// operator apply vanishes and the sweep is facet-local, x_f = w D_f^-1 b_f.
template <int N1, bool STORED>
__global__ void bj_zero_kernel(const MvArgs a, const __grid_constant__ SharedOp<(STORED ? 1 : N1)> op, double w,
                               long long nblocks) {
  const long long bk = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (bk >= nblocks) return;
  const bool vert = bk >= a.nh;
  double r[N1], dinv[N1 * N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) r[k] = __ldg(a.b + bk * N1 + k);
  if constexpr (!STORED) {
#pragma unroll
    for (int t = 0; t < N1 * N1; ++t) dinv[t] = vert ? op.Dv[t] : op.Dh[t];
  } else {
    int i, j;
    if (!vert) { j = (int)(bk / a.nx) + 1; i = (int)(bk % a.nx); }
    else { const long long u = bk - a.nh; i = (int)(u / a.ny) + 1; j = (int)(u % a.ny); }
    const long long slot = (long long)j * a.nxp + i;
    const double* D = (vert ? a.Dv : a.Dh) + (size_t)(slot >> 5) * N1 * N1 * 32 + (slot & 31);
#pragma unroll
    for (int t = 0; t < N1 * N1; ++t) dinv[t] = __ldg(D + (size_t)t * 32);
  }
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < N1; ++m) s = fma(dinv[k * N1 + m], r[m], s);
    a.out[bk * N1 + k] = w * s;
  }
}

// ------------------------------------------------------------------------------ FSAI (CSR)
// y = M x  or  x_out = x_in + w (M x)   (multigrid.py:72-74, 83-88); 4 lanes per row
template <bool AXPY>
__global__ void csr_spmv_kernel(int n, const int* __restrict__ rowptr, const int* __restrict__ cols,
                                const double* __restrict__ vals, const double* __restrict__ x, double* __restrict__ y,
                                const double* __restrict__ xin, double w) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 2;
  const int sub = threadIdx.x & 3;
  double s = 0.0;
  if (row < n) {
    const int e = __ldg(rowptr + row + 1);
    for (int k = __ldg(rowptr + row) + sub; k < e; k += 4) s = fma(__ldg(vals + k), __ldg(x + __ldg(cols + k)), s);
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (row < n && sub == 0) {
    if constexpr (AXPY) y[row] = fma(w, s, xin[row]); else y[row] = s;
  }
}

// CG vector updates (trace.py:156-161): x += a d, r -= a ad ;  d = z + beta d
static __global__ void cg_update_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ d,
                                 const double* __restrict__ ad, double alpha, long long n) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    x[t] = fma(alpha, d[t], x[t]);
    r[t] = fma(-alpha, ad[t], r[t]);
  }
}

// two dot products in one pass (same per-thread order as dot_partials_kernel, so each result is
// bitwise the one a separate hdg_dot would give): partials[blk] = a.b, partials[grid + blk] = c.e
static __global__ void dot2_partials_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                     const double* __restrict__ c, const double* __restrict__ e, long long n,
                                     double* __restrict__ partials) {
  double s = 0.0, u = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    s = fma(__ldg(a + t), __ldg(b + t), s);
    u = fma(__ldg(c + t), __ldg(e + t), u);
  }
  __shared__ double red[2][32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    u += __shfl_xor_sync(0xffffffffu, u, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = s; red[1][threadIdx.x >> 5] = u; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t0 += red[0][w]; t1 += red[1][w]; }
    partials[blockIdx.x] = t0;
    partials[gridDim.x + blockIdx.x] = t1;
  }
}

// CG updates with the step lengths read from device scalars (no host round trip):
// sc[0] = r.z, sc[1] = d.Ad, sc[2] = r_new.z_new  (trace.py:156-161)
static __global__ void cg_update_dev_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ d,
                                     const double* __restrict__ ad, const double* __restrict__ sc, long long n) {
  const double alpha = sc[0] / sc[1];
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    x[t] = fma(alpha, d[t], x[t]);
    r[t] = fma(-alpha, ad[t], r[t]);
  }
}

static __global__ void xpby_dev_kernel(const double* __restrict__ z, const double* __restrict__ sc, double* __restrict__ d,
                                long long n) {
  const double beta = sc[2] / sc[0];
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    d[t] = fma(beta, d[t], z[t]);
}

static __global__ void xpby_kernel(const double* __restrict__ z, double beta, double* __restrict__ d, long long n) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    d[t] = fma(beta, d[t], z[t]);
}

// ------------------------------------------------------------------ fused coarse-level tail
// The small p = 1 levels at the bottom of a V/W cycle (multigrid.py:393-406) are latency-bound:
// ~6 dependent launches per level visit, each a few microseconds whatever the level size.  The
// host turns the tail of the cycle (same recursion, sweep weights and buffer roles as the
// launch path) into a flat program of facet-parallel ops that ONE CTA runs with every tail
// vector resident in shared memory and __syncthreads between dependent ops.  Facet applies read
// their 7 stencil blocks from shared memory and the unreduced merged operators from global
// (read-only, L1/L2-resident).  Only the entry right-hand side (and, on a repeated visit, the
// entry iterate) come from global memory, and only the level's result goes back.
enum TailCode { T_BJ = 0, T_BJZ = 1, T_RES = 2, T_RESTRICT = 3, T_PROLONG = 4, T_COARSE = 5, T_COPY = 6, T_ZERO = 7 };

struct TailLevel {          // one level of the tail (n1 = 2)
  int nx, ny, nxp, stored;
  long long nh, nblk;
  const double* W[2];       // merged n1 x 7n1 operators: shared (7*4 doubles, [q][k][m]) or stored streams
  const double* D[2];       // block-Jacobi inverses: shared (4 doubles) or stored streams
  int off[3];               // shared-memory offsets (doubles) of this level's X, T, B vectors
};

struct TailOp {
  short code, lev;          // lev: the level (T_RESTRICT / T_PROLONG: the fine level of the link)
  short x, b, out;          // buffer ids: 3 * level + {0: X, 1: T, 2: B}; -1 unused
  double w;
};

constexpr int TAIL_MAXL = 12;
constexpr int TAIL_MAXOPS = 512;
constexpr int TAIL_THREADS = 512;

struct __align__(16) TailArgs {
  TailLevel lev[TAIL_MAXL];
  HArgs h[TAIL_MAXL];       // h[l]: transfer level l -> l + 1 of the tail
  const double* Ainv;       // coarsest level: dense inverse (n_c x n_c)
  const double* b_in;       // entry right-hand side of the top tail level (global)
  const double* x_in;       // entry iterate of the top tail level (global; nullptr = zero start)
  double* x_out;            // result of the top tail level (global)
  int nc, nops, nlev, pad_;
  TailOp ops[TAIL_MAXOPS];
};

static_assert(sizeof(TailArgs) % sizeof(uint4) == 0, "TailArgs is copied to shared memory as uint4");
constexpr int TAIL_ARGS_DOUBLES = (int)(sizeof(TailArgs) / sizeof(double));

// A x restricted to facet bk of level L (n1 = 2, x in shared memory); out-of-mesh / Dirichlet
// stencil blocks read 0.  32-bit index math: tail levels are small.
__device__ __forceinline__ void tail_facet_apply(const TailLevel& L, const double* x, int bk, double (&y)[2],
                                                 int& slot_out, bool& vert_out) {
  constexpr int N1 = 2;
  const int nx = L.nx, ny = L.ny, nh = (int)L.nh;
  const bool vert = bk >= nh;
  int i, j;
  if (!vert) { j = bk / nx + 1; i = bk - (j - 1) * nx; }
  else { const int u = bk - nh; i = u / ny + 1; j = u - (i - 1) * ny; }
  auto hb = [&](int ii, int jj) -> int { return (ii >= 0 && ii < nx && jj >= 1 && jj <= ny - 1) ? (jj - 1) * nx + ii : -1; };
  auto vb = [&](int ii, int jj) -> int { return (ii >= 1 && ii <= nx - 1 && jj >= 0 && jj < ny) ? nh + (ii - 1) * ny + jj : -1; };
  int q[7];
  if (!vert) {
    q[0] = hb(i, j - 1); q[1] = bk; q[2] = hb(i, j + 1);
    q[3] = vb(i, j - 1); q[4] = vb(i + 1, j - 1); q[5] = vb(i, j); q[6] = vb(i + 1, j);
  } else {
    q[0] = vb(i - 1, j); q[1] = bk; q[2] = vb(i + 1, j);
    q[3] = hb(i - 1, j); q[4] = hb(i - 1, j + 1); q[5] = hb(i, j); q[6] = hb(i, j + 1);
  }
  const int slot = j * L.nxp + i;
  y[0] = 0.0; y[1] = 0.0;
  if (L.stored && HDG_SYMSTORE) {
    // half-stored stream: own blocks + 3 transposed from their owners (apply_stored_half)
    constexpr int B = N1 * N1 * 32;
    const int QO[4] = {1, 2, vert ? 4 : 5, 6};
    const double* own = wslot<N1>(L.W[vert ? 1 : 0], slot);
    const double* tp[3];
    const int QT[3] = {0, 3, vert ? 5 : 4};
    if (!vert) {
      const int sd = slot - L.nxp;
      tp[0] = wslot<N1>(L.W[0], sd) + B; tp[1] = wslot<N1>(L.W[1], sd) + 3 * B; tp[2] = wslot<N1>(L.W[1], sd + 1) + 2 * B;
    } else {
      const int sw = slot - 1;
      tp[0] = wslot<N1>(L.W[1], sw) + B; tp[1] = wslot<N1>(L.W[0], sw) + 3 * B; tp[2] = wslot<N1>(L.W[0], slot) + 2 * B;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int s = QO[t];
      const double2 v = q[s] >= 0 ? reinterpret_cast<const double2*>(x)[q[s]] : make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        y[k] = fma(own[t * B + (k * N1 + 0) * 32], v.x, y[k]);
        y[k] = fma(own[t * B + (k * N1 + 1) * 32], v.y, y[k]);
      }
    }
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int s = QT[t];
      if (q[s] < 0) continue;
      const double2 v = reinterpret_cast<const double2*>(x)[q[s]];
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        y[k] = fma(tp[t][(0 * N1 + k) * 32], v.x, y[k]);
        y[k] = fma(tp[t][(1 * N1 + k) * 32], v.y, y[k]);
      }
    }
  } else {
    const double* W = L.W[vert ? 1 : 0];
    const int ws = L.stored ? 32 : 1;
    if (L.stored) W += (size_t)(slot >> 5) * 7 * N1 * N1 * 32 + (slot & 31);
#pragma unroll
    for (int s = 0; s < 7; ++s) {
      const double2 v = q[s] >= 0 ? reinterpret_cast<const double2*>(x)[q[s]] : make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        y[k] = fma(W[((s * N1 + k) * N1 + 0) * ws], v.x, y[k]);
        y[k] = fma(W[((s * N1 + k) * N1 + 1) * ws], v.y, y[k]);
      }
    }
  }
  slot_out = slot;
  vert_out = vert;
}

__device__ __forceinline__ void tail_dinv(const TailLevel& L, bool vert, int slot, const double (&r)[2],
                                          double (&z)[2]) {
  const double* D = L.D[vert ? 1 : 0];
  int st = 1;
  if (L.stored) { D += (size_t)(slot >> 5) * 4 * 32 + (slot & 31); st = 32; }
  const double d0 = D[0], d1 = D[st], d2 = D[2 * st], d3 = D[3 * st];
  z[0] = fma(d0, r[0], d1 * r[1]);
  z[1] = fma(d2, r[0], d3 * r[1]);
}

__device__ __forceinline__ int tail_slot(const TailLevel& L, int bk, bool& vert) {
  const int nh = (int)L.nh;
  vert = bk >= nh;
  int i, j;
  if (!vert) { j = bk / L.nx + 1; i = bk - (j - 1) * L.nx; }
  else { const int u = bk - nh; i = u / L.ny + 1; j = u - (i - 1) * L.ny; }
  return j * L.nxp + i;
}

static __global__ void __launch_bounds__(TAIL_THREADS, 1) tail_cycle_kernel(const __grid_constant__ TailArgs Ap) {
  extern __shared__ __align__(16) double tsm_raw[];
  const int tid = threadIdx.x;
  // the program and level descriptors are read on every op: copy them from the parameter
  // bank (constant-cache misses on a 15 KB block) into shared memory once
  TailArgs& A = *reinterpret_cast<TailArgs*>(tsm_raw);
  {
    constexpr int NW = (int)(sizeof(TailArgs) / sizeof(uint4));
    const uint4* src = reinterpret_cast<const uint4*>(&Ap);
    uint4* dst = reinterpret_cast<uint4*>(tsm_raw);
    for (int t = tid; t < NW; t += TAIL_THREADS) dst[t] = src[t];
  }
  grid_dependency_wait();   // the program copy above overlaps the previous kernel's tail
  __syncthreads();
  // shared-mode operators (64 doubles per level) next to the program; stored streams stay global
  double* opsm = tsm_raw + TAIL_ARGS_DOUBLES;
  for (int l = 0; l < A.nlev; ++l) {
    if (A.lev[l].stored) continue;
    const double* src = A.lev[l].W[0];   // Wh, Wv, Dh, Dv contiguous (hdg_capi.cu: tail_wd)
    for (int t = tid; t < 64; t += TAIL_THREADS) opsm[64 * l + t] = __ldg(src + t);
  }
  __syncthreads();
  if (tid == 0) {
    for (int l = 0; l < A.nlev; ++l) {
      if (A.lev[l].stored) continue;
      double* o = opsm + 64 * l;
      A.lev[l].W[0] = o; A.lev[l].W[1] = o + 28; A.lev[l].D[0] = o + 56; A.lev[l].D[1] = o + 60;
    }
  }
  __syncthreads();
  double* tsm = opsm + 64 * TAIL_MAXL;
  auto buf = [&](int id) -> double* { return tsm + A.lev[id / 3].off[id % 3]; };
  {  // entry: b (and x) of the top tail level
    const long long n0 = 2 * A.lev[0].nblk;
    double* b0 = buf(2);
    double* x0 = buf(0);
    for (long long t = tid; t < n0; t += TAIL_THREADS) {
      b0[t] = A.b_in[t];
      if (A.x_in) x0[t] = A.x_in[t];
    }
  }
  __syncthreads();
  for (int o = 0; o < A.nops; ++o) {
    const TailOp& op = A.ops[o];
    const TailLevel& L = A.lev[op.lev];
    switch (op.code) {
      case T_BJ:
      case T_RES: {
        const double* x = buf(op.x);
        const double* b = buf(op.b);
        double* out = buf(op.out);
        for (int bk = tid; bk < (int)L.nblk; bk += TAIL_THREADS) {
          double y[2];
          int slot;
          bool vert;
          tail_facet_apply(L, x, bk, y, slot, vert);
          const double r[2] = {b[2 * bk] - y[0], b[2 * bk + 1] - y[1]};
          if (op.code == T_RES) {
            out[2 * bk] = r[0]; out[2 * bk + 1] = r[1];
          } else {
            double z[2];
            tail_dinv(L, vert, slot, r, z);
            out[2 * bk] = fma(op.w, z[0], x[2 * bk]);
            out[2 * bk + 1] = fma(op.w, z[1], x[2 * bk + 1]);
          }
        }
        break;
      }
      case T_BJZ: {
        const double* b = buf(op.b);
        double* out = buf(op.out);
        for (int bk = tid; bk < (int)L.nblk; bk += TAIL_THREADS) {
          bool vert;
          const int slot = tail_slot(L, bk, vert);
          const double r[2] = {b[2 * bk], b[2 * bk + 1]};
          double z[2];
          tail_dinv(L, vert, slot, r, z);
          out[2 * bk] = op.w * z[0];
          out[2 * bk + 1] = op.w * z[1];
        }
        break;
      }
      case T_RESTRICT: {
        const HArgs& h = A.h[op.lev];
        const int nc = (int)(h.nhc + (long long)(h.nxc - 1) * h.nyc);
        if (h.shared_cross)
          for (int t = tid; t < nc; t += TAIL_THREADS) h_restrict_one<true, true>(h, buf(op.x), buf(op.out), t);
        else
          for (int t = tid; t < nc; t += TAIL_THREADS) h_restrict_one<true, false>(h, buf(op.x), buf(op.out), t);
        break;
      }
      case T_PROLONG: {
        const HArgs& h = A.h[op.lev];
        const int nf = (int)(h.nhf + (long long)(2 * h.nxc - 1) * h.nyf);
        if (h.shared_cross)
          for (int t = tid; t < nf; t += TAIL_THREADS) h_prolong_add_one<true, true>(h, buf(op.x), buf(op.out), t);
        else
          for (int t = tid; t < nf; t += TAIL_THREADS) h_prolong_add_one<true, false>(h, buf(op.x), buf(op.out), t);
        break;
      }
      case T_COARSE: {   // warp per row of the dense inverse (multigrid.py:209-212)
        const int lane = tid & 31;
        const double* b = buf(op.b);
        double* out = buf(op.out);
        for (int row = tid >> 5; row < A.nc; row += TAIL_THREADS / 32) {
          double acc = 0.0;
          for (int c = lane; c < A.nc; c += 32) acc = fma(__ldg(A.Ainv + (size_t)row * A.nc + c), b[c], acc);
#pragma unroll
          for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
          if (lane == 0) out[row] = acc;
        }
        break;
      }
      case T_COPY: {
        const double* x = buf(op.x);
        double* out = buf(op.out);
        for (long long t = tid; t < 2 * L.nblk; t += TAIL_THREADS) out[t] = x[t];
        break;
      }
      default: {  // T_ZERO
        double* out = buf(op.out);
        for (long long t = tid; t < 2 * L.nblk; t += TAIL_THREADS) out[t] = 0.0;
        break;
      }
    }
    __syncthreads();
  }
  const long long n0 = 2 * A.lev[0].nblk;
  const double* x0 = buf(0);
  for (long long t = tid; t < n0; t += TAIL_THREADS) A.x_out[t] = x0[t];
}

// ------------------------------------------------------------------- FSAI setup (rows)
// fsai_build's per-row solve (multigrid.py:133-152) for every row at once, one thread per row:
// gather the principal block A[P_i, P_i] of the row's pattern (sorted columns, the diagonal
// last) from A's CSR by binary search, Cholesky-factor it (the block is SPD for an SPD A; a
// non-positive pivot flags the row), solve A_P g = e_last and scale g by 1/sqrt(g_last).
// With A_P = L L^T:  L^-1 e_last = e_last / l_LL, so g = L^-T e_last / l_LL and the scaled row
// is l_LL * g = L^-T e_last.
__device__ __forceinline__ double csr_at(const int* __restrict__ ptr, const int* __restrict__ col,
                                         const double* __restrict__ val, int r, int c) {
  int lo = __ldg(ptr + r), hi = __ldg(ptr + r + 1) - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int cm = __ldg(col + mid);
    if (cm == c) return __ldg(val + mid);
    if (cm < c) lo = mid + 1; else hi = mid - 1;
  }
  return 0.0;
}

template <int MAXL>
__global__ void fsai_rows_kernel(long long n, const int* __restrict__ a_ptr, const int* __restrict__ a_col,
                                 const double* __restrict__ a_val, const int* __restrict__ g_ptr,
                                 const int* __restrict__ g_col, double* __restrict__ g_val,
                                 long long* __restrict__ bad) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int s = __ldg(g_ptr + row), L = __ldg(g_ptr + row + 1) - s;
  if (L < 1 || L > MAXL) { atomicMin(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)row); return; }
  double M[MAXL * (MAXL + 1) / 2];   // packed lower triangle, M(a, b) at a (a + 1) / 2 + b
  int cols[MAXL];
  for (int a = 0; a < L; ++a) cols[a] = __ldg(g_col + s + a);
  for (int a = 0; a < L; ++a)
    for (int b = 0; b <= a; ++b) M[a * (a + 1) / 2 + b] = csr_at(a_ptr, a_col, a_val, cols[a], cols[b]);
  for (int j = 0; j < L; ++j) {       // Cholesky, column by column
    double d = M[j * (j + 1) / 2 + j];
    for (int k = 0; k < j; ++k) d -= M[j * (j + 1) / 2 + k] * M[j * (j + 1) / 2 + k];
    if (!(d > 0.0)) { atomicMin(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)row); return; }
    d = sqrt(d);
    M[j * (j + 1) / 2 + j] = d;
    for (int i = j + 1; i < L; ++i) {
      double v = M[i * (i + 1) / 2 + j];
      for (int k = 0; k < j; ++k) v -= M[i * (i + 1) / 2 + k] * M[j * (j + 1) / 2 + k];
      M[i * (i + 1) / 2 + j] = v / d;
    }
  }
  // back substitution L^T g = e_last (in place of the solution vector, written straight out)
  double g[MAXL];
  for (int a = L - 1; a >= 0; --a) {
    double v = (a == L - 1) ? 1.0 : 0.0;
    for (int i = a + 1; i < L; ++i) v -= M[i * (i + 1) / 2 + a] * g[i];
    g[a] = v / M[a * (a + 1) / 2 + a];
  }
  for (int a = 0; a < L; ++a) g_val[s + a] = g[a];
}

}  // namespace hdg
