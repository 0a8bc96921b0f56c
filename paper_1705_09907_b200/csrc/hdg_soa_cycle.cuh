// hdg_soa_cycle.cuh - the multigrid cycle's kernels on facet records (hdg_soa.cuh layout).
//
// The V-cycle of multigrid.py:393-406 on the constant-coefficient p-ladder of the finest mesh:
// every level vector (iterate, right-hand side, residual, correction) stays in the facet-record
// layout and every smoothing sweep / residual is ONE pass of the element-column streaming apply
// of hdg_soa.cuh with the update fused behind the facet sums:
//   SEPI_BJ     y = x + w D^-1 (b - A x)                   block-Jacobi sweep (slot of
//                                                          lev.smoother.smooth, multigrid.py:398,405)
//   SEPI_BJ0    x1 = w0 D^-1 b ; y = x1 + w D^-1 (b - A x1) the first two sweeps of a visit that starts
//                                                          from x = 0 (multigrid.py:400): the ring
//                                                          streams b, x1 is formed per facet on the fly
//   SEPI_BJ0F   the same double sweep folded (p <= 4): y = D^-1 ((w0 + w) b - w w0 (S D^-1) b), the element
//               product runs on the raw b with the class blocks of S D^-1 (one D^-1 per written facet
//               instead of one per read facet plus one per written facet: 152 instead of 227 FMAs at p = 4)
//   SEPI_RES    y = b - A x                                residual before an h-restriction
//   SEPI_RESPR  y_c = V^T (b - A x)                        residual + p-restriction (multigrid.py:399),
//                                                          written as records of order p - 1
//   PROL        x' = x + V e_c first (multigrid.py:403), for all four facets of each element, e_c
//                                                          streamed through a second record ring
// x (or b for SEPI_BJ0) streams through the per-warp TMA ring exactly as in soa_apply_kernel; b is
// needed only at the facets a lane writes and is read straight from global memory one row ahead.
// One writer per record sector, no atomics, no grid synchronisation.
#pragma once
#include "hdg_soa.cuh"

#ifndef HDG_SOA_BAHEAD_MAX_N1
#define HDG_SOA_BAHEAD_MAX_N1 5    // right-hand side fetched one row ahead up to this n1 (above: spills, p = 8 cycle 7.8 -> 8.1 ms)
#endif

namespace hdg {

template <int N1>
struct SoaCycArgs {
  const double* x;      // ring input records: the iterate (SOA_EPI_BJ0: the right-hand side)
  const double* b;      // right-hand side records
  const double* ec;     // PROL: coarse correction records (order N1 - 2)
  double* y;            // output records
  int nx, ny, W, nss;
  double w, w0;
  double M[SoaCfg<N1>::MSZ];
  double Dh[N1 * N1], Dv[N1 * N1];   // inverse diagonal blocks of horizontal / vertical facets
  double V[N1 * (N1 - 1)];           // p-transfer V[k][c] (multigrid.py:215-219)
};

template <int N1, int EPI, bool PROL>
struct SoaCycCfg {
  using C = SoaCfg<N1>;
  static constexpr int NC = N1 - 1;                       // coarse order + 1 of the p-link
  using CC = SoaCfg<(NC >= 2 ? NC : 2)>;
  static constexpr int NO = EPI == SOA_EPI_RESPR ? NC : N1;   // nodes per output facet
  using CO = SoaCfg<(NO >= 2 ? NO : 2)>;
  static constexpr int ENT2 = PROL ? CC::ENT : 0;         // second ring entry (coarse correction records)
  static constexpr int WSTRIDE = (C::RING * (C::ENT + ENT2) + 2 * C::RING + 3) & ~3;
  static constexpr int SMEM = SoaSmem<N1>::TOTAL * 8 + C::WPB * WSTRIDE * 8;
  static constexpr bool MCONST = N1 <= 5;
  // the fused epilogues need more registers than the plain apply: from n1 = 8 two CTAs per SM
  // without spills beat three with (configs[3] p = 8 cycle: 7.8 vs 8.9 ms)
  static constexpr int MINB = N1 >= 8 ? 2 : SoaCfg<N1>::MINB;
};

template <int N1>
__device__ __forceinline__ void soa_dmul(const double* D, const double* r, double* z) {
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    double s = D[k * N1] * r[0];
#pragma unroll
    for (int m = 1; m < N1; ++m) s = fma(D[k * N1 + m], r[m], s);
    z[k] = s;
  }
}

// out = update of one facet from its operator value ax, iterate xf and right-hand side bf
template <int N1, int EPI>
__device__ __forceinline__ void soa_epi(const SoaCycArgs<N1>& a, const double* D, const double* ax,
                                        const double* xf, const double* bf, bool valid, double* out) {
  double r[N1];
  if constexpr (EPI == SOA_EPI_BJ0F) {
    const double c1 = a.w0 + a.w, c2 = a.w * a.w0;      // ax holds (S D^-1 b) summed over the owners
    double z[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) r[k] = c1 * bf[k] - c2 * ax[k];
    soa_dmul<N1>(D, r, z);
#pragma unroll
    for (int k = 0; k < N1; ++k) out[k] = valid ? z[k] : 0.0;
  } else {
#pragma unroll
    for (int k = 0; k < N1; ++k) r[k] = bf[k] - ax[k];
    if constexpr (EPI == SOA_EPI_RES) {
#pragma unroll
      for (int k = 0; k < N1; ++k) out[k] = valid ? r[k] : 0.0;
    } else if constexpr (EPI == SOA_EPI_RESPR) {
      constexpr int NC = N1 - 1;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double s = a.V[c] * r[0];
#pragma unroll
        for (int k = 1; k < N1; ++k) s = fma(a.V[k * NC + c], r[k], s);
        out[c] = valid ? s : 0.0;
      }
    } else {
      double z[N1];
      soa_dmul<N1>(D, r, z);
#pragma unroll
      for (int k = 0; k < N1; ++k) out[k] = valid ? fma(a.w, z[k], xf[k]) : 0.0;
    }
  }
}

template <int N1, int EPI, bool PROL>
__global__ void __launch_bounds__(SoaCfg<N1>::NTH, SoaCycCfg<N1, EPI, PROL>::MINB)
    soa_cycle_kernel(const __grid_constant__ SoaCycArgs<N1> a) {
  using C = SoaCfg<N1>;
  using K = SoaCycCfg<N1, EPI, PROL>;
  using CO = typename K::CO;
  using CC = typename K::CC;
  constexpr int NT = 4 * N1, RING = C::RING, D = RING - 1, WPB = C::WPB, NO = K::NO, NC = K::NC;
  constexpr int ENT = C::ENT, VOFF = C::VOFF, EOFF = C::EOFF, EB = C::EB;
  constexpr bool MCONST = K::MCONST;
  constexpr bool BJ0 = EPI == SOA_EPI_BJ0;            // ring streams b, x1 = w0 D^-1 b formed per facet
  constexpr bool BJ0F = EPI == SOA_EPI_BJ0F;          // ring streams b, folded form (a.M = blocks of S D^-1)
  constexpr bool BRING = BJ0 || BJ0F;                 // the right-hand side of the written facets is in the ring
  static_assert(!(PROL && BRING), "a prolongation never meets a zero iterate");
  static_assert(!BJ0F || MCONST, "the folded double sweep reads its blocks from the constant bank");
  extern __shared__ __align__(32) double smem_soa[];
  double* Ms = smem_soa;
  if (!MCONST) {
    for (int idx = threadIdx.x; idx < SoaSmem<N1>::TOTAL; idx += blockDim.x) {
      // same packing as soa_load_blocks (upper triangles, padded)
      using M = SoaSmem<N1>;
      constexpr int sz[4] = {C::A0, C::A1, C::A2, C::A3};
      constexpr int so[5] = {M::O0, M::O1, M::O2, M::O3, M::TOTAL};
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
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  double* ring0 = smem_soa + SoaSmem<N1>::TOTAL;
  double* ring = ring0 + q * K::WSTRIDE;
  double* ring2 = ring + RING * ENT;                   // PROL: coarse correction entries
  const int w = blockIdx.x % a.W, ss = blockIdx.x / a.W;
  const int c = 31 * w + lane;
  const int c0 = (int)((long long)ss * a.ny / a.nss), c1 = (int)((long long)(ss + 1) * a.ny / a.nss);
  const int g = (HDG_SOA_BAL && c0 > 0) ? 1 : 0;
  auto lo = [&](int u) { return u <= 0 ? c0 : min(c1, c0 + max(0, (c1 - c0 + g) * u / WPB - g)); };
  const int r0 = lo(q), r1 = lo(q + 1);
  const bool active = r1 > r0;
  int below = -1;
  for (int u = q - 1; u >= 0 && below < 0; --u)
    if (lo(u + 1) > lo(u)) below = u;
  const bool defer = active && below >= 0;
  const int rs = (active && below < 0 && r0 > 0) ? r0 - 1 : r0;
  const int nrows = r1 - rs;
  const double* __restrict__ X = a.x;
  const double* __restrict__ B = a.b;
  double* __restrict__ Y = a.y;
  const long long W = a.W;
  auto rec = [&](int R, long long tile) { return (R * W + tile) * ENT; };          // input records
  auto reco = [&](int R, long long tile) { return (R * W + tile) * CO::ENT; };     // output records
  auto recc = [&](int R, long long tile) { return (R * W + tile) * CC::ENT; };     // correction records

  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + RING * (ENT + K::ENT2));
  if (lane == 0) {
#pragma unroll
    for (int e = 0; e < RING; ++e) mbar_init(bars + e, 1);
  }
  fence_proxy_async();
  __syncwarp();
#if HDG_SOA_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  auto issue = [&](int t) {
    if (t > nrows || lane != 0 || !active) return;
    uint64_t* bar = bars + (t % RING);
    const unsigned bytes = t == 0 ? VOFF * 8u : ENT * 8u;
    const unsigned bytes2 = PROL ? (t == 0 ? CC::VOFF * 8u : CC::ENT * 8u) : 0u;
    mbar_arrive_expect_tx(bar, bytes + bytes2);
    tma_load_1d(ring + (t % RING) * ENT, X + rec(rs + t, w), bytes, bar);
    if constexpr (PROL) tma_load_1d(ring2 + (t % RING) * CC::ENT, a.ec + recc(rs + t, w), bytes2, bar);
  };
#pragma unroll
  for (int t = 0; t < D; ++t) issue(t);

  const bool hcol = c < a.nx;
  const bool vline = lane < 31 && c + 1 <= a.nx - 1;
  const int oL = lane == 0 ? EOFF : VOFF + lane - 1, sL = lane == 0 ? 1 : 31;
  const int oR = lane == 31 ? EOFF + EB : VOFF + lane, sR = lane == 31 ? 1 : 31;
  const int oLc = lane == 0 ? CC::EOFF : CC::VOFF + lane - 1;
  const int oRc = lane == 31 ? CC::EOFF + CC::EB : CC::VOFF + lane;
  // tp: T part of A x of the row below; xC: that row's top iterate = this row's bottom iterate
  double tp[N1], xC[N1], hold[N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) tp[k] = hold[k] = xC[k] = 0.0;

  // iterate of one facet from its ring values: raw (BJ / RES / RESPR), + V e_c (PROL), w0 D^-1 b (BJ0)
  auto facet_h = [&](const double* e, const double* e2, int slot, double* xv) {
    double raw[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) raw[k] = e[k * 32 + slot];
    if constexpr (BJ0) {
      soa_dmul<N1>(a.Dh, raw, xv);
#pragma unroll
      for (int k = 0; k < N1; ++k) xv[k] *= a.w0;
    } else if constexpr (PROL) {
      double ev[NC];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) ev[cc] = e2[cc * 32 + slot];
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double s = raw[k];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) s = fma(a.V[k * NC + cc], ev[cc], s);
        xv[k] = s;
      }
    } else {
#pragma unroll
      for (int k = 0; k < N1; ++k) xv[k] = raw[k];
    }
  };
  auto facet_v = [&](const double* e, const double* e2, int off, int st, int offc, double* xv) {
    double raw[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) raw[k] = e[off + k * st];
    if constexpr (BJ0) {
      soa_dmul<N1>(a.Dv, raw, xv);
#pragma unroll
      for (int k = 0; k < N1; ++k) xv[k] *= a.w0;
    } else if constexpr (PROL) {
      double ev[NC];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) ev[cc] = e2[offc + cc * st];
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double s = raw[k];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) s = fma(a.V[k * NC + cc], ev[cc], s);
        xv[k] = s;
      }
    } else {
#pragma unroll
      for (int k = 0; k < N1; ++k) xv[k] = raw[k];
    }
  };

  // right-hand side of the facets a row writes (H line r, V of element row r), straight from global
  // memory; at the lowest orders a row's arithmetic is too short to cover the load, so the values of
  // the coming row are fetched one row ahead (BAHEAD)
  constexpr bool BAHEAD = !BRING && N1 <= HDG_SOA_BAHEAD_MAX_N1;
  auto loadb = [&](int r, double* bh_out, double* bv_out) {
    const bool ld = r >= r0;
    const double* bh = B + rec(r, w) + lane;
    const double* bv = B + rec(r + 1, w) + VOFF + lane;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      bh_out[k] = ld ? __ldg(bh + k * 32) : 0.0;
      bv_out[k] = (ld && lane < 31) ? __ldg(bv + k * 31) : 0.0;
    }
  };
  double bHn[BAHEAD ? N1 : 1], bVn[BAHEAD ? N1 : 1];
  if constexpr (BAHEAD) {
    if (active) loadb(rs, bHn, bVn);
  }

  if (active) {
#pragma unroll 1
    for (int t = 0; t < nrows; ++t) {
      const int r = rs + t;
      fence_proxy_async();
      issue(t + D);
      // right-hand side of the facets this row writes (H line r, V of element row r), one row
      // ahead of their use; SOA_EPI_BJ0 takes them from the ring (the ring streams b)
      double bH[N1], bV[N1];
      if constexpr (!BRING) {
        if constexpr (BAHEAD) {                          // loaded during the previous row
#pragma unroll
          for (int k = 0; k < N1; ++k) { bH[k] = bHn[k]; bV[k] = bVn[k]; }
          if (t + 1 < nrows) loadb(r + 1, bHn, bVn);
        } else {
          loadb(r, bH, bV);
        }
      }
      if (t == 0) mbar_wait(bars, 0);
      mbar_wait(bars + (t + 1) % RING, ((t + 1) / RING) & 1);
      const double* e0 = ring + (t % RING) * ENT;
      const double* e1 = ring + ((t + 1) % RING) * ENT;
      const double* f0 = ring2 + (t % RING) * CC::ENT;
      const double* f1 = ring2 + ((t + 1) % RING) * CC::ENT;
      double xB[N1], xT[N1], xR[N1], xL[N1];
      if (t == 0) facet_h(e0, f0, lane, xB);
      else {
#pragma unroll
        for (int k = 0; k < N1; ++k) xB[k] = xC[k];
      }
      facet_h(e1, f1, lane, xT);
      facet_v(e1, f1, oL, sL, oLc, xL);
      facet_v(e1, f1, oR, sR, oRc, xR);
      double yB[N1], yR[N1], yT[N1], yL[N1];
      {
        double tv[NT], z[NT];
        soa_forward<N1>(xB, xR, xT, xL, tv);
        if constexpr (BJ0F) soa_blocks_cg<N1>(a.M, tv, z);
        else if (MCONST) soa_blocks_c<N1>(a.M, tv, z);
        else soa_blocks<N1>(Ms, tv, z);
        soa_backward<N1>(z, yB, yR, yT, yL);
      }
      if (r >= r0) {
        if constexpr (BRING) {                          // the raw ring values are the right-hand side
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            bH[k] = e0[k * 32 + lane];
            bV[k] = e1[oR + k * sR];
          }
        }
        if (t == 0 && defer) {
#pragma unroll
          for (int k = 0; k < N1; ++k) hold[k] = yB[k];
        } else {
          const bool hint = hcol && r >= 1;
          double ax[N1], out[NO];
#pragma unroll
          for (int k = 0; k < N1; ++k) ax[k] = tp[k] + yB[k];
          soa_epi<N1, EPI>(a, a.Dh, ax, xB, bH, hint, out);
          double* hrec = Y + reco(r, w);
#pragma unroll
          for (int k = 0; k < NO; ++k) hrec[k * 32 + lane] = out[k];
        }
        double* vrec = Y + reco(r + 1, w);
        double vv[NO];
        {
          double ax[N1];
#pragma unroll
          for (int k = 0; k < N1; ++k) ax[k] = yR[k] + __shfl_down_sync(0xffffffffu, yL[k], 1);
          soa_epi<N1, EPI>(a, a.Dv, ax, xR, bV, vline, vv);
        }
        double* stg = ring + (t % RING) * ENT;
        __syncwarp();                                  // every lane is done with entry t
#pragma unroll
        for (int k = 0; k < NO; ++k)
          if (lane < 31) stg[k * 31 + lane] = vv[k];
        if (lane < CO::VB - NO * 31) stg[NO * 31 + lane] = 0.0;
        __syncwarp();
#pragma unroll
        for (int o = 0; o < CO::VB / 4; o += 32)
          if (o + lane < CO::VB / 4) {
            const double2 v0 = reinterpret_cast<const double2*>(stg)[2 * (o + lane)];
            const double2 v1 = reinterpret_cast<const double2*>(stg)[2 * (o + lane) + 1];
            st_sector(vrec + CO::VOFF + 4 * (o + lane), v0.x, v0.y, v1.x, v1.y);
          }
        if (lane == 30) {
          if (w + 1 < W) soa_store_edge<NO>(vrec + CO::ENT + CO::EOFF, vv);
          else {
#pragma unroll
            for (int k = 0; k < NO; ++k) vv[k] = 0.0;
            soa_store_edge<NO>(vrec + CO::EOFF + CO::EB, vv);
          }
        }
        if (lane == 0) {
          if (w > 0) soa_store_edge<NO>(vrec - CO::ENT + CO::EOFF + CO::EB, vv);
          else {
#pragma unroll
            for (int k = 0; k < NO; ++k) vv[k] = 0.0;
            soa_store_edge<NO>(vrec + CO::EOFF, vv);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        tp[k] = yT[k];
        xC[k] = xT[k];
      }
      __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < N1; ++k) ring[k * 32 + lane] = tp[k];
  }
  __syncthreads();
  if (defer) {
    // line r0: the operator value closes with the lower warp's last top part; iterate and
    // right-hand side of the line are read back from global memory (once per segment)
    const double* src = ring0 + below * K::WSTRIDE;
    const bool hint = hcol && r0 >= 1;
    double ax[N1], xf[N1], bf[N1], out[NO];
#pragma unroll
    for (int k = 0; k < N1; ++k) ax[k] = src[k * 32 + lane] + hold[k];
    const double* xh = X + rec(r0, w) + lane;
    if constexpr (BJ0F) {
#pragma unroll
      for (int k = 0; k < N1; ++k) { bf[k] = xh[k * 32]; xf[k] = 0.0; }
    } else if constexpr (BJ0) {
#pragma unroll
      for (int k = 0; k < N1; ++k) bf[k] = xh[k * 32];
      soa_dmul<N1>(a.Dh, bf, xf);
#pragma unroll
      for (int k = 0; k < N1; ++k) xf[k] *= a.w0;
    } else {
      const double* bh = B + rec(r0, w) + lane;
#pragma unroll
      for (int k = 0; k < N1; ++k) { xf[k] = xh[k * 32]; bf[k] = bh[k * 32]; }
      if constexpr (PROL) {
        const double* eh = a.ec + recc(r0, w) + lane;
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          const double ev = eh[cc * 32];
#pragma unroll
          for (int k = 0; k < N1; ++k) xf[k] = fma(a.V[k * NC + cc], ev, xf[k]);
        }
      }
    }
    soa_epi<N1, EPI>(a, a.Dh, ax, xf, bf, hint, out);
    double* hrec = Y + reco(r0, w);
#pragma unroll
    for (int k = 0; k < NO; ++k) hrec[k * 32 + lane] = out[k];
  }
  if (active && r1 == a.ny) {
    double* hrec = Y + reco(a.ny, w);
#pragma unroll
    for (int k = 0; k < NO; ++k) hrec[k * 32 + lane] = 0.0;
  }
  if (active && r0 == 0) {
    double* vrec = Y + reco(0, w) + CO::VOFF;
    for (int o = lane; o < CO::VB + 2 * CO::EB; o += 32) vrec[o] = 0.0;
  }
}

// ---------------------------------------------------------------- facet-local record kernels
// decode slot s of a record: 0..31 H columns, 32..62 V lines, 63 / 64 the left-in / right-in
// edge lines; returns the offset of node 0 and the node stride
template <int N1>
__device__ __forceinline__ void soa_slot(int s, int& off, int& st) {
  using C = SoaCfg<N1>;
  if (s < 32) { off = s; st = 32; }
  else if (s < 63) { off = C::VOFF + (s - 32); st = 31; }
  else { off = C::EOFF + (s - 63) * C::EB; st = 1; }
}

// x_f += V e_c on records of the same mesh (multigrid.py:215-219, 403); N1 = fine nodes
template <int N1>
__global__ void soa_p_prolong_kernel(const double* __restrict__ ec, double* __restrict__ xf, long long nrec,
                                     const PArgs a) {
  constexpr int NC = N1 - 1;
  using CC = SoaCfg<(NC >= 2 ? NC : 2)>;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrec * 65) return;
  const long long rw = t / 65;
  const int s = (int)(t % 65);
  int of, sf, oc, sc;
  soa_slot<N1>(s, of, sf);
  soa_slot<(NC >= 2 ? NC : 2)>(s, oc, sc);
  const double* e = ec + rw * CC::ENT + oc;
  double* x = xf + rw * SoaCfg<N1>::ENT + of;
  double ev[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) ev[c] = __ldg(e + c * sc);
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    double v = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) v = fma(a.V[k * NC + c], ev[c], v);
    x[k * sf] += v;
  }
}

// h-transfers between p = 1 facet records of the fine mesh and the reference-layout coarse vector
// (multigrid.py:229-298; single GPU: whole meshes, nyf = 2 nyc).  Offsets of node 0 of fine facets:
__device__ __forceinline__ long long rec2_h(int W, int i, int j) {      // h(i, j): line j, column i; stride 32
  const int w = min(i / 31, W - 1);
  return ((long long)j * W + w) * SoaCfg<2>::ENT + (i - 31 * w);
}
__device__ __forceinline__ long long rec2_v(int W, int i, int j) {      // v(i, j): line i, row j; stride 31
  const int w = (i - 1) / 31;
  return ((long long)(j + 1) * W + w) * SoaCfg<2>::ENT + SoaCfg<2>::VOFF + (i - 31 * w - 1);
}

template <bool SC>
__device__ __forceinline__ void rec2_cross_restrict(const HArgs& h, int W, const double* __restrict__ rf, int I,
                                                    int J, int s, double* acc) {
  const long long a0 = rec2_v(W, 2 * I + 1, 2 * J), a1 = rec2_v(W, 2 * I + 1, 2 * J + 1);
  const long long a2 = rec2_h(W, 2 * I, 2 * J + 1), a3 = rec2_h(W, 2 * I + 1, 2 * J + 1);
  const long long ad[4] = {a0, a1, a2, a3};
  const int st[4] = {31, 31, 32, 32};
#pragma unroll
  for (int cf = 0; cf < 4; ++cf) {
    const double* tm = hcross<SC>(h, I, J, cf);
    const double r0 = __ldg(rf + ad[cf]), r1 = __ldg(rf + ad[cf] + st[cf]);
    for (int c = 0; c < 2; ++c) {
      if constexpr (SC) acc[c] += tm[0 * 8 + s * 2 + c] * r0 + tm[1 * 8 + s * 2 + c] * r1;
      else acc[c] += __ldg(tm + 0 * 8 + s * 2 + c) * r0 + __ldg(tm + 1 * 8 + s * 2 + c) * r1;
    }
  }
}

// store helpers for p = 1 records: every copy of a facet (see rec2_add_h / rec2_add_v)
__device__ __forceinline__ void rec2_set_h(double* __restrict__ x, int W, int c, int j, double v0, double v1) {
  const int w = min(c / 31, W - 1);
  double* p = x + ((long long)j * W + w) * SoaCfg<2>::ENT + (c - 31 * w);
  p[0] = v0; p[32] = v1;
  if (c == 31 * w && w > 0) {
    double* q = p - SoaCfg<2>::ENT + 31;
    q[0] = v0; q[32] = v1;
  }
}
__device__ __forceinline__ void rec2_set_v(double* __restrict__ x, int W, int i, int j, double v0, double v1) {
  using C = SoaCfg<2>;
  const int w = (i - 1) / 31;
  double* rec = x + ((long long)(j + 1) * W) * C::ENT;
  double* p = rec + (long long)w * C::ENT + C::VOFF + (i - 31 * w - 1);
  p[0] = v0; p[31] = v1;
  if (i % 31 == 0 && i / 31 < W) {
    double* q = rec + (long long)(i / 31) * C::ENT + C::EOFF;
    q[0] = v0; q[1] = v1;
  }
  if (i >= 32 && (i - 32) % 31 == 0) {
    double* q = rec + (long long)((i - 32) / 31) * C::ENT + C::EOFF + C::EB;
    q[0] = v0; q[1] = v1;
  }
}

// CREC: the coarse vector is a p = 1 record vector too (Wc tiles; every slot that is not a facet stays
// the zero it was allocated with), else the reference layout
template <bool SC, bool CREC = false>
__global__ void soa_h_restrict_kernel(const __grid_constant__ HArgs h, int W, const double* __restrict__ rf,
                                      double* __restrict__ rc, int Wc = 0) {
  const long long nvc = (long long)(h.nxc - 1) * h.nyc;
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  grid_dependency_wait();
  if (t >= h.nhc + nvc) return;
  double acc[2] = {0.0, 0.0};
  if (t < h.nhc) {   // coarse h(I, J): children fine h(2I, 2J), h(2I+1, 2J)
    const int J = (int)(t / h.nxc) + 1, I = (int)(t % h.nxc);
    for (int hf = 0; hf < 2; ++hf) {
      const long long ad = rec2_h(W, 2 * I + hf, 2 * J);
      const double r0 = __ldg(rf + ad), r1 = __ldg(rf + ad + 32);
      for (int c = 0; c < 2; ++c) acc[c] += h.halves[hf * 4 + 0 * 2 + c] * r0 + h.halves[hf * 4 + 1 * 2 + c] * r1;
    }
    rec2_cross_restrict<SC>(h, W, rf, I, J - 1, 2, acc);
    rec2_cross_restrict<SC>(h, W, rf, I, J, 0, acc);
    if constexpr (CREC) { rec2_set_h(rc, Wc, I, J, acc[0], acc[1]); return; }
  } else {           // coarse v(I, J): children fine v(2I, 2J), v(2I, 2J+1)
    // consecutive threads walk I (neighbouring slots of the same fine records: coalesced reads); the
    // coarse vector is vertical-line-major, so the two 8-byte stores are the scattered side
    const long long u = t - h.nhc;
    const int J = (int)(u / (h.nxc - 1)), I = (int)(u % (h.nxc - 1)) + 1;
    t = h.nhc + (long long)(I - 1) * h.nyc + J;
    for (int hf = 0; hf < 2; ++hf) {
      const long long ad = rec2_v(W, 2 * I, 2 * J + hf);
      const double r0 = __ldg(rf + ad), r1 = __ldg(rf + ad + 31);
      for (int c = 0; c < 2; ++c) acc[c] += h.halves[hf * 4 + 0 * 2 + c] * r0 + h.halves[hf * 4 + 1 * 2 + c] * r1;
    }
    rec2_cross_restrict<SC>(h, W, rf, I - 1, J, 1, acc);
    rec2_cross_restrict<SC>(h, W, rf, I, J, 3, acc);
    if constexpr (CREC) { rec2_set_v(rc, Wc, I, J, acc[0], acc[1]); return; }
  }
  rc[2 * t] = acc[0];
  rc[2 * t + 1] = acc[1];
}

// x_f += P_h e_c on p = 1 facet records (multigrid.py:229-298, 403), one thread per coarse element (I, J):
// it loads the element's four coarse sides once and updates the eight fine facets they determine - the
// four cross facets inside the element and the two halves each of its bottom and left coarse facets
// (every fine facet belongs to exactly one coarse element this way).  A fine facet that is stored twice
// (H column on a tile seam; V line that is a neighbouring tile's edge-in line) is updated in every copy.
__device__ __forceinline__ void rec2_add_h(double* __restrict__ xf, int W, int c, int j, const double* add) {
  const int w = min(c / 31, W - 1);
  double* p = xf + ((long long)j * W + w) * SoaCfg<2>::ENT + (c - 31 * w);
  p[0] += add[0]; p[32] += add[1];
  if (c == 31 * w && w > 0) {                    // slot 0 of tile w = slot 31 of tile w - 1
    double* q = p - SoaCfg<2>::ENT + 31;
    q[0] += add[0]; q[32] += add[1];
  }
}
__device__ __forceinline__ void rec2_add_v(double* __restrict__ xf, int W, int i, int j, const double* add) {
  using C = SoaCfg<2>;
  const int w = (i - 1) / 31;
  double* rec = xf + ((long long)(j + 1) * W) * C::ENT;
  double* p = rec + (long long)w * C::ENT + C::VOFF + (i - 31 * w - 1);
  p[0] += add[0]; p[31] += add[1];
  if (i % 31 == 0 && i / 31 < W) {               // left-in line of tile i / 31
    double* q = rec + (long long)(i / 31) * C::ENT + C::EOFF;
    q[0] += add[0]; q[1] += add[1];
  }
  if (i >= 32 && (i - 32) % 31 == 0) {           // right-in line of tile (i - 32) / 31
    double* q = rec + (long long)((i - 32) / 31) * C::ENT + C::EOFF + C::EB;
    q[0] += add[0]; q[1] += add[1];
  }
}

// side s of coarse element (I, J) from a coarse p = 1 record vector (zero on Dirichlet sides)
__device__ __forceinline__ void coarse_side_rec(const HArgs& h, const double* __restrict__ ec, int Wc, int I, int J,
                                                int s, double* v) {
  long long ad = -1;
  int st = 32;
  if (s == 0 && J >= 1) ad = rec2_h(Wc, I, J);
  if (s == 2 && J + 1 <= h.nyc - 1) ad = rec2_h(Wc, I, J + 1);
  if (s == 3 && I >= 1) { ad = rec2_v(Wc, I, J); st = 31; }
  if (s == 1 && I + 1 <= h.nxc - 1) { ad = rec2_v(Wc, I + 1, J); st = 31; }
  v[0] = ad >= 0 ? __ldg(ec + ad) : 0.0;
  v[1] = ad >= 0 ? __ldg(ec + ad + st) : 0.0;
}

template <bool SC, bool CREC = false>
__global__ void soa_h_prolong_kernel(const __grid_constant__ HArgs h, int W, int nxf, int nyf,
                                     const double* __restrict__ ec, double* __restrict__ xf, int Wc = 0) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  grid_dependency_wait();
  if (t >= (long long)h.nxc * h.nyc) return;
  const int J = (int)(t / h.nxc), I = (int)(t - (long long)J * h.nxc);
  double sd[4][2];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if constexpr (CREC) coarse_side_rec(h, ec, Wc, I, J, s, sd[s]);
    else coarse_side<false>(h, ec, I, J, s, sd[s]);
  }
  // cross facets: right of SW = v(2I+1, 2J), right of NW = v(2I+1, 2J+1), top of SW = h(2I, 2J+1),
  // top of SE = h(2I+1, 2J+1)
#pragma unroll
  for (int cf = 0; cf < 4; ++cf) {
    const double* tm = hcross<SC>(h, I, J, cf);
    double add[2] = {0.0, 0.0};
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if constexpr (SC) add[k] += tm[k * 8 + s * 2] * sd[s][0] + tm[k * 8 + s * 2 + 1] * sd[s][1];
        else add[k] += __ldg(tm + k * 8 + s * 2) * sd[s][0] + __ldg(tm + k * 8 + s * 2 + 1) * sd[s][1];
      }
    if (cf < 2) rec2_add_v(xf, W, 2 * I + 1, 2 * J + cf, add);
    else rec2_add_h(xf, W, 2 * I + (cf - 2), 2 * J + 1, add);
  }
  // halves of the bottom coarse facet h(I, J) (J >= 1) and of the left one v(I, J) (I >= 1)
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    double add[2];
    if (J >= 1) {
#pragma unroll
      for (int k = 0; k < 2; ++k) add[k] = h.halves[hf * 4 + k * 2] * sd[0][0] + h.halves[hf * 4 + k * 2 + 1] * sd[0][1];
      rec2_add_h(xf, W, 2 * I + hf, 2 * J, add);
    }
    if (I >= 1) {
#pragma unroll
      for (int k = 0; k < 2; ++k) add[k] = h.halves[hf * 4 + k * 2] * sd[3][0] + h.halves[hf * 4 + k * 2 + 1] * sd[3][1];
      rec2_add_v(xf, W, 2 * I, 2 * J + hf, add);
    }
  }
  (void)nxf; (void)nyf;
}

// a.b (and c.e when c != nullptr) of record vectors over the trace dofs, every dof once: slot 31 of an H
// row repeats the next tile's slot 0 and the edge blocks repeat V lines of the neighbouring tiles; pads
// are zeros.  Per-CTA partials in a fixed order (partials[blk], partials[grid + blk]);
// sum_partials_kernel finishes (deterministic).
template <int N1>
__global__ void __launch_bounds__(256) soa_dot2_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                       const double* __restrict__ c, const double* __restrict__ e,
                                                       long long nrec, int W, double* __restrict__ partials) {
  using C = SoaCfg<N1>;
  double s = 0.0, s2 = 0.0;
  const long long total = nrec * 63;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long rw = t / 63;
    const int sl = (int)(t - rw * 63);
    if (sl == 31 && (int)(rw % W) != W - 1) continue;
    int off, st;
    soa_slot<N1>(sl, off, st);
    const long long o = rw * C::ENT + off;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      s = fma(a[o + k * st], b[o + k * st], s);
      if (c != nullptr) s2 = fma(c[o + k * st], e[o + k * st], s2);
    }
  }
  __shared__ double red[2][8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = s; red[1][threadIdx.x >> 5] = s2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, t2 = 0.0;
    for (int w = 0; w < 8; ++w) { t += red[0][w]; t2 += red[1][w]; }
    partials[blockIdx.x] = t;
    if (c != nullptr) partials[gridDim.x + blockIdx.x] = t2;
  }
}

}  // namespace hdg
