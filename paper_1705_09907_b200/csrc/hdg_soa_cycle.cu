// hdg_soa_cycle.cu - launchers of the record-layout cycle kernels (hdg_soa_cycle.cuh); called by
// the native cycle in hdg_capi.cu.  Reference: multigrid.py:393-406 (_cycle).
#include "hdg_internal.h"
#include "hdg_soa_cycle.cuh"

#include <algorithm>
#include <cstring>

template <int N1, int EPI, bool PROL>
static int cyc_launch(const hdg_level* L, const double* x, const double* b, double* y, double w, double w0,
                      const double* V, const double* ec, cudaStream_t s) {
  using K = SoaCycCfg<N1, EPI, PROL>;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(soa_cycle_kernel<N1, EPI, PROL>, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM));
    attr = true;
  }
  SoaCycArgs<N1> a{};
  a.x = x; a.b = b; a.y = y; a.ec = ec;
  a.nx = L->nx; a.ny = L->ny; a.W = L->soaW; a.nss = L->soaNss;
  // one wave: the level's segment count was sized for the apply kernel's CTAs per SM
  if (K::MINB < SoaCfg<N1>::MINB) a.nss = std::max(1, L->soaNss * K::MINB / SoaCfg<N1>::MINB);
  a.w = w; a.w0 = w0;
  if (EPI == SOA_EPI_BJ0F) {
    if (L->soaM0.size() * sizeof(double) != sizeof(a.M)) return fail(HDG_ESTATE, "record cycle: folded blocks not prepared");
    std::memcpy(a.M, L->soaM0.data(), sizeof(a.M));
  } else {
    std::memcpy(a.M, L->soaM.data(), sizeof(a.M));
  }
  std::memcpy(a.Dh, L->Dh.data(), sizeof(a.Dh));
  std::memcpy(a.Dv, L->Dv.data(), sizeof(a.Dv));
  if (V) std::memcpy(a.V, V, sizeof(a.V));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.W * a.nss));
  cfg.blockDim = dim3(SoaCfg<N1>::NTH);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = HDG_SOA_PDL ? 1 : 0;
  cudaLaunchKernelEx(&cfg, soa_cycle_kernel<N1, EPI, PROL>, a);
  CKL();
  return 0;
}

template <int N1>
static int cyc_sweep_t(const hdg_level* L, int epi, const double* x, const double* b, double* y, double w,
                       double w0, const double* V, const double* ec, cudaStream_t s) {
  if (epi == SOA_EPI_BJ0) return cyc_launch<N1, SOA_EPI_BJ0, false>(L, x, b, y, w, w0, V, ec, s);
  if constexpr (N1 <= 5) {
    if (epi == SOA_EPI_BJ0F) return cyc_launch<N1, SOA_EPI_BJ0F, false>(L, x, b, y, w, w0, V, ec, s);
  }
  if (epi == SOA_EPI_RES) return cyc_launch<N1, SOA_EPI_RES, false>(L, x, b, y, w, w0, V, ec, s);
  if constexpr (N1 >= 3) {
    if (epi == SOA_EPI_RESPR) return cyc_launch<N1, SOA_EPI_RESPR, false>(L, x, b, y, w, w0, V, ec, s);
    if (epi == SOA_EPI_BJ && ec) return cyc_launch<N1, SOA_EPI_BJ, true>(L, x, b, y, w, w0, V, ec, s);
  }
  if (epi == SOA_EPI_BJ && !ec) return cyc_launch<N1, SOA_EPI_BJ, false>(L, x, b, y, w, w0, V, ec, s);
  return fail(HDG_EINVAL, "record cycle: no such sweep at this order");
}

int soa_cyc_sweep(const hdg_level* L, int epi, const double* x, const double* b, double* y, double w, double w0,
                  const double* V, const double* ec, cudaStream_t s) {
  if (L->soa_state != 1 || !L->has_bj) return fail(HDG_ESTATE, "record cycle: level not prepared");
  if (x == y || b == y) return fail(HDG_EINVAL, "record sweeps cannot run in place");
  switch (L->n1) {
    case 2: return cyc_sweep_t<2>(L, epi, x, b, y, w, w0, V, ec, s);
    case 3: return cyc_sweep_t<3>(L, epi, x, b, y, w, w0, V, ec, s);
    case 4: return cyc_sweep_t<4>(L, epi, x, b, y, w, w0, V, ec, s);
    case 5: return cyc_sweep_t<5>(L, epi, x, b, y, w, w0, V, ec, s);
#ifndef HDG_SOA_CYC_LOW_ONLY
    case 6: return cyc_sweep_t<6>(L, epi, x, b, y, w, w0, V, ec, s);
    case 7: return cyc_sweep_t<7>(L, epi, x, b, y, w, w0, V, ec, s);
    case 8: return cyc_sweep_t<8>(L, epi, x, b, y, w, w0, V, ec, s);
    case 9: return cyc_sweep_t<9>(L, epi, x, b, y, w, w0, V, ec, s);
    case 10: return cyc_sweep_t<10>(L, epi, x, b, y, w, w0, V, ec, s);
    case 11: return cyc_sweep_t<11>(L, epi, x, b, y, w, w0, V, ec, s);
    case 12: return cyc_sweep_t<12>(L, epi, x, b, y, w, w0, V, ec, s);
    case 13: return cyc_sweep_t<13>(L, epi, x, b, y, w, w0, V, ec, s);
#endif
    default: return fail(HDG_EINVAL, "record cycle: order not built");
  }
}

int soa_cyc_p_prolong(const hdg_level* Lf, const hdg_level* Lc, const double* ec, double* xf, const double* V,
                      cudaStream_t s) {
  if (Lc->n1 != Lf->n1 - 1 || Lc->nx != Lf->nx || Lc->ny != Lf->ny)
    return fail(HDG_EINVAL, "record p-prolongation: levels do not match");
  const long long nrec = (long long)(Lf->ny + 1) * Lf->soaW;
  PArgs pa{};
  std::memcpy(pa.V, V, sizeof(double) * Lf->n1 * (Lf->n1 - 1));
  const unsigned grid = (unsigned)((nrec * 65 + 255) / 256);
#define PP(N) case N: soa_p_prolong_kernel<N><<<grid, 256, 0, s>>>(ec, xf, nrec, pa); break;
  switch (Lf->n1) {
    PP(3) PP(4) PP(5) PP(6) PP(7) PP(8) PP(9) PP(10) PP(11) PP(12) PP(13)
    default: return fail(HDG_EINVAL, "record p-prolongation: order not built");
  }
#undef PP
  CKL();
  return 0;
}

static int h_check(const hdg_level* Lf, const HArgs& h) {
  if (Lf->n1 != 2 || h.jf0 != 0 || h.jc0 != 0 || h.nyf != 2 * h.nyc || Lf->nx != 2 * h.nxc || Lf->ny != h.nyf)
    return fail(HDG_EINVAL, "record h-transfer: needs whole p = 1 meshes with nyf = 2 nyc");
  return 0;
}

// Lc != nullptr: the coarse vector is a record vector of level Lc (its non-facet slots must be zero)
int soa_cyc_h_restrict(const hdg_level* Lf, const HArgs& h, const double* rf, double* rc, cudaStream_t s,
                       const hdg_level* Lc) {
  int rc0 = h_check(Lf, h);
  if (rc0) return rc0;
  const long long n = h.nhc + (long long)(h.nxc - 1) * h.nyc;
  if (n == 0) return 0;
  const unsigned grid = (unsigned)((n + 127) / 128);
  const int Wc = Lc ? Lc->soaW : 0;
  if (Lc) {
    if (h.shared_cross) launch_pdl(soa_h_restrict_kernel<true, true>, dim3(grid), dim3(128), 0, s, h, Lf->soaW, rf, rc, Wc);
    else launch_pdl(soa_h_restrict_kernel<false, true>, dim3(grid), dim3(128), 0, s, h, Lf->soaW, rf, rc, Wc);
  } else {
    if (h.shared_cross) launch_pdl(soa_h_restrict_kernel<true, false>, dim3(grid), dim3(128), 0, s, h, Lf->soaW, rf, rc, Wc);
    else launch_pdl(soa_h_restrict_kernel<false, false>, dim3(grid), dim3(128), 0, s, h, Lf->soaW, rf, rc, Wc);
  }
  CKL();
  return 0;
}

int soa_cyc_h_prolong(const hdg_level* Lf, const HArgs& h, const double* ec, double* xf, cudaStream_t s,
                      const hdg_level* Lc) {
  int rc0 = h_check(Lf, h);
  if (rc0) return rc0;
  const long long n = (long long)h.nxc * h.nyc;           // one thread per coarse element
  if (n == 0) return 0;
  const unsigned grid = (unsigned)((n + 127) / 128);
  const int Wc = Lc ? Lc->soaW : 0;
  if (Lc) {
    if (h.shared_cross) launch_pdl(soa_h_prolong_kernel<true, true>, dim3(grid), dim3(128), 0, s, h, Lf->soaW, Lf->nx, Lf->ny, ec, xf, Wc);
    else launch_pdl(soa_h_prolong_kernel<false, true>, dim3(grid), dim3(128), 0, s, h, Lf->soaW, Lf->nx, Lf->ny, ec, xf, Wc);
  } else {
    if (h.shared_cross) launch_pdl(soa_h_prolong_kernel<true, false>, dim3(grid), dim3(128), 0, s, h, Lf->soaW, Lf->nx, Lf->ny, ec, xf, Wc);
    else launch_pdl(soa_h_prolong_kernel<false, false>, dim3(grid), dim3(128), 0, s, h, Lf->soaW, Lf->nx, Lf->ny, ec, xf, Wc);
  }
  CKL();
  return 0;
}

// out[0] = a.b, and out2[0] = c.e when c is given, over the trace dofs of record vectors (device scalars);
// `partials` holds at least 2 * nblocks doubles
int soa_cyc_dot2(const hdg_level* L, const double* a, const double* b, double* out, const double* c, const double* e,
                 double* out2, double* partials, int nblocks, cudaStream_t s) {
  if (L->soa_state != 1) return fail(HDG_ESTATE, "record dot: level not prepared");
  const long long nrec = (long long)(L->ny + 1) * L->soaW;
#define DOT(N) case N: soa_dot2_kernel<N><<<nblocks, 256, 0, s>>>(a, b, c, e, nrec, L->soaW, partials); break;
  switch (L->n1) {
    DOT(2) DOT(3) DOT(4) DOT(5) DOT(6) DOT(7) DOT(8) DOT(9) DOT(10) DOT(11) DOT(12) DOT(13)
    default: return fail(HDG_EINVAL, "record dot: order not built");
  }
#undef DOT
  CKL();
  sum_partials_kernel<<<1, 32, 0, s>>>(partials, nblocks, out);
  CKL();
  if (c) {
    sum_partials_kernel<<<1, 32, 0, s>>>(partials + nblocks, nblocks, out2);
    CKL();
  }
  return 0;
}

int soa_cyc_norm2(const hdg_level* L, const double* r, double* out, double* partials, int nblocks, cudaStream_t s) {
  return soa_cyc_dot2(L, r, r, out, nullptr, nullptr, nullptr, partials, nblocks, s);
}
