// hdg_capi.cu - C ABI (include/hdgb200.h) and native runtime: operator objects, transfers,
// the device-resident multigrid cycle and its CUDA-graph cache.
// Reference interfaces replaced: see include/hdgb200.h (each entry cites trace.py / multigrid.py).
#include "hdg_internal.h"
#include "hdg_soa.cuh"
#include "hdg_fsai.cuh"

#include <algorithm>
#include <climits>
#include <atomic>
#define _USE_MATH_DEFINES
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

bool hdg_pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("HDG_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// ------------------------------------------------------------------------------ helpers

static void host_invert(std::vector<double>& a, int n) {  // SPD Gauss-Jordan, no pivoting
  for (int c = 0; c < n; ++c) {
    const double piv = 1.0 / a[c * n + c];
    for (int m = 0; m < n; ++m) a[c * n + m] *= piv;
    a[c * n + c] = piv;
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = a[r * n + c];
      a[r * n + c] = 0.0;
      for (int m = 0; m < n; ++m) a[r * n + m] -= f * a[c * n + m];
      a[r * n + c] = -f * piv;
    }
  }
}


template <int N1, bool STORED, int EPI>
static auto kernel_ptr() {
  return trace_apply_kernel<N1, STORED, EPI>;
}

template <int N1, bool STORED, int EPI>
static int set_attr() {
  const size_t smem = Cfg<N1, STORED>::template smem_doubles_epi<EPI>() * sizeof(double);
  CK(cudaFuncSetAttribute(kernel_ptr<N1, STORED, EPI>(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return 0;
}

template <int N1, bool STORED>
static int prepare_t() {
  int rc = 0;
  if ((rc = set_attr<N1, STORED, EPI_Y>())) return rc;
  if ((rc = set_attr<N1, STORED, EPI_RES>())) return rc;
  if ((rc = set_attr<N1, STORED, EPI_BJ>())) return rc;
  if ((rc = set_attr<N1, STORED, EPI_RESPR>())) return rc;
  return 0;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

static int vec_blocks();
static int dot_into(const double* a, const double* b, int64_t n, double* out, double* partials, cudaStream_t s);

// persistent grid: every SM gets as many CTAs as fit (<= MAX_CTAS_PER_SM), never more than tiles
template <int N1, bool STORED, int EPI>
static int grid_for(const hdg_level* L) {
  using C = Cfg<N1, STORED>;
  static int occ = -1;
  if (occ < 0) {
    const size_t smem = C::template smem_doubles_epi<EPI>() * sizeof(double);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel_ptr<N1, STORED, EPI>(), C::NTH, smem) !=
            cudaSuccess || occ < 1)
      occ = 1;
    if (occ > MAX_CTAS_PER_SM) occ = MAX_CTAS_PER_SM;
  }
  const long long tiles = (long long)((L->nx + TX - 1) / TX) * ((L->ny + C::TY - 1) / C::TY);
  const long long g = (long long)sm_count() * occ;
  return (int)(tiles < g ? tiles : g);
}

template <int N1, bool STORED, int EPI>
static int apply_t(const hdg_level* L, MvArgs& a, cudaStream_t s) {
  using C = Cfg<N1, STORED>;
  const size_t smem = C::template smem_doubles_epi<EPI>() * sizeof(double);
  const int grid = grid_for<N1, STORED, EPI>(L);
  SharedOp<(STORED ? 1 : N1)> op;
  if constexpr (!STORED) {
    if constexpr (HDG_SHARED_SYM) {   // kernel reads the reduced stencils from op.Wh / op.Wv
      std::memset(op.Wh, 0, sizeof(op.Wh));
      std::memset(op.Wv, 0, sizeof(op.Wv));
      std::memcpy(op.Wh, L->Gh.data(), sizeof(double) * Sym<N1>::SIZE);
      std::memcpy(op.Wv, L->Gv.data(), sizeof(double) * Sym<N1>::SIZE);
    } else {
      std::memcpy(op.Wh, L->Wh.data(), sizeof(op.Wh));
      std::memcpy(op.Wv, L->Wv.data(), sizeof(op.Wv));
    }
    if (L->has_bj) {
      std::memcpy(op.Dh, L->Dh.data(), sizeof(op.Dh));
      std::memcpy(op.Dv, L->Dv.data(), sizeof(op.Dv));
    } else {
      std::memset(op.Dh, 0, sizeof(op.Dh));
      std::memset(op.Dv, 0, sizeof(op.Dv));
    }
  } else {
    std::memset(&op, 0, sizeof(op));
  }
  launch_pdl(kernel_ptr<N1, STORED, EPI>(), dim3(grid), dim3(C::NTH), smem, s, a, op);
  CKL();
  return 0;
}

#define HDG_N1_SWITCH(n1, CALL)                                       \
  switch (n1) {                                                       \
    case 2: CALL(2); case 3: CALL(3); case 4: CALL(4); case 5: CALL(5); \
    case 6: CALL(6); case 7: CALL(7); case 8: CALL(8); case 9: CALL(9); \
    case 10: CALL(10); case 11: CALL(11); case 12: CALL(12); case 13: CALL(13); \
    default: return fail(HDG_EINVAL, "order p must be in [1, 12]");   \
  }

static int apply(const hdg_level* L, int epi, MvArgs& a, cudaStream_t s, double omega_override = 0.0) {
  a.nx = L->nx; a.ny = L->ny; a.nxp = L->nxp; a.nh = (int)L->nh;
  a.Wh = L->dWh; a.Wv = L->dWv; a.Dh = L->dDh; a.Dv = L->dDv;
  a.omega = omega_override != 0.0 ? omega_override : L->omega;
  if (L->ndof == 0) return 0;
#define APPLY_CASE(N)                                                                 \
  {                                                                                   \
    if (L->stored) {                                                                  \
      if (epi == EPI_Y) return apply_t<N, true, EPI_Y>(L, a, s);                      \
      if (epi == EPI_RES) return apply_t<N, true, EPI_RES>(L, a, s);                  \
      if (epi == EPI_BJ) return apply_t<N, true, EPI_BJ>(L, a, s);                    \
      return apply_t<N, true, EPI_RESPR>(L, a, s);                                    \
    }                                                                                 \
    if (epi == EPI_Y) return apply_t<N, false, EPI_Y>(L, a, s);                       \
    if (epi == EPI_RES) return apply_t<N, false, EPI_RES>(L, a, s);                   \
    if (epi == EPI_BJ) return apply_t<N, false, EPI_BJ>(L, a, s);                     \
    return apply_t<N, false, EPI_RESPR>(L, a, s);                                     \
  }
  HDG_N1_SWITCH(L->n1, APPLY_CASE)
#undef APPLY_CASE
}

static int prepare(int n1, bool stored) {
#define PREP_CASE(N) return stored ? prepare_t<N, true>() : prepare_t<N, false>();
  HDG_N1_SWITCH(n1, PREP_CASE)
#undef PREP_CASE
}

static int init_level(hdg_level* L, int nx, int ny, int p) {
  if (nx < 1 || ny < 1) return fail(HDG_EINVAL, "mesh element counts must be positive");
  if (p < 1 || p > MAXN1 - 1) return fail(HDG_EINVAL, "order p must be in [1, 12]");
  L->nx = nx; L->ny = ny; L->p = p; L->n1 = p + 1;
  L->nxp = ((nx + 1 + 31) / 32) * 32;   // >= nx + 1: the half-stored stream reads slot (j, i + 1)
  L->nh = (long long)nx * (ny - 1);
  L->n_blocks = L->nh + (long long)(nx - 1) * ny;
  L->ndof = L->n_blocks * L->n1;
  if (L->ndof >= (1LL << 31) - 64) return fail(HDG_EINVAL, "one level must hold < 2^31 trace dofs per GPU");
  L->npart = sm_count() * MAX_CTAS_PER_SM;
  CK(cudaMalloc(&L->partials, sizeof(double) * (L->npart + 1)));
  return 0;
}

// Mirror reduction of a merged facet stencil W (7 n1 x n1 blocks, stencil order of
// merged_entry_src) into Sym<N1> form (hdg_kernels.cuh, apply_shared_sym).  Returns false when
// W is not invariant under the two facet mirrors to 1e-11 of max|W|; otherwise G receives the
// group-averaged (in exact arithmetic: identical) operator's even / odd blocks.
static bool mirror_reduce(const std::vector<double>& W, int n1, std::vector<double>& G) {
  const int h = (n1 + 1) / 2, l = n1 / 2, ke = 2 * h + n1, ko = 2 * l + n1;
  auto w = [&](int q, int k, int m) { return W[(q * n1 + k) * n1 + m]; };
  auto rv = [&](int k) { return n1 - 1 - k; };
  std::vector<double> B0(n1 * n1), B1(n1 * n1), B3(n1 * n1), B4(n1 * n1);
  double scale = 0.0, defect = 0.0;
  for (double v : W) scale = std::fmax(scale, std::fabs(v));
  auto dev = [&](double a, double b) { defect = std::fmax(defect, std::fabs(a - b)); };
  for (int k = 0; k < n1; ++k)
    for (int m = 0; m < n1; ++m) {   // normal mirror: W q0 = q2, q3 = q5 R, q4 = q6 R
      dev(w(0, k, m), w(2, k, m));
      dev(w(3, k, m), w(5, k, rv(m)));
      dev(w(4, k, m), w(6, k, rv(m)));
      B0[k * n1 + m] = 0.5 * (w(0, k, m) + w(2, k, m));
      B1[k * n1 + m] = w(1, k, m);
      B3[k * n1 + m] = 0.5 * (w(3, k, m) + w(5, k, rv(m)));
      B4[k * n1 + m] = 0.5 * (w(4, k, m) + w(6, k, rv(m)));
    }
  std::vector<double> C0(n1 * n1), C1(n1 * n1), C3(n1 * n1);
  for (int k = 0; k < n1; ++k)
    for (int m = 0; m < n1; ++m) {   // tangential mirror: R B0 R = B0, R B1 R = B1, R B4 = B3
      dev(B0[k * n1 + m], B0[rv(k) * n1 + rv(m)]);
      dev(B1[k * n1 + m], B1[rv(k) * n1 + rv(m)]);
      dev(B3[k * n1 + m], B4[rv(k) * n1 + m]);
      C0[k * n1 + m] = 0.5 * (B0[k * n1 + m] + B0[rv(k) * n1 + rv(m)]);
      C1[k * n1 + m] = 0.5 * (B1[k * n1 + m] + B1[rv(k) * n1 + rv(m)]);
      C3[k * n1 + m] = 0.5 * (B3[k * n1 + m] + B4[rv(k) * n1 + m]);
    }
  if (!(defect <= 1e-11 * scale)) return false;
  G.assign(h * ke + l * ko, 0.0);
  double* Ge = G.data();
  double* Go = G.data() + h * ke;
  for (int k = 0; k < h; ++k) {
    for (int m = 0; m < l; ++m) {
      Ge[k * ke + m] = 0.5 * (C0[k * n1 + m] + C0[k * n1 + rv(m)]);
      Ge[k * ke + h + m] = 0.5 * (C1[k * n1 + m] + C1[k * n1 + rv(m)]);
    }
    if (n1 & 1) {
      Ge[k * ke + h - 1] = C0[k * n1 + h - 1];
      Ge[k * ke + 2 * h - 1] = C1[k * n1 + h - 1];
    }
    for (int m = 0; m < n1; ++m) Ge[k * ke + 2 * h + m] = 0.5 * (C3[k * n1 + m] + C3[rv(k) * n1 + m]);
  }
  for (int k = 0; k < l; ++k) {
    for (int m = 0; m < l; ++m) {
      Go[k * ko + m] = 0.5 * (C0[k * n1 + m] - C0[k * n1 + rv(m)]);
      Go[k * ko + l + m] = 0.5 * (C1[k * n1 + m] - C1[k * n1 + rv(m)]);
    }
    for (int m = 0; m < n1; ++m) Go[k * ko + 2 * l + m] = 0.5 * (C3[k * n1 + m] - C3[rv(k) * n1 + m]);
  }
  return true;
}

static void delete_level_keep_error(hdg_level* L) {
  cudaFree(L->partials);
  delete L;
}

// ------------------------------------------------------------------------------- C ABI

extern "C" {

const char* hdg_last_error(void) { return g_err.c_str(); }
int hdg_version(void) { return 1; }
int64_t hdg_launch_count(void) { return g_launches.load(); }

static int create_stored(int nx, int ny, int p, const double* blocks, bool bcast, hdg_level** out);

int hdg_level_create_shared(int nx, int ny, int p, const double* block, hdg_level** out) {
  if (!out || !block) return fail(HDG_EINVAL, "null argument");
  hdg_level* L = new hdg_level();
  int rc = init_level(L, nx, ny, p);
  if (rc) { delete L; return rc; }
  const int n1 = L->n1, Lw = 4 * n1;
  L->blk.assign(block, block + (size_t)Lw * Lw);
  L->Wh.assign(7 * n1 * n1, 0.0);
  L->Wv.assign(7 * n1 * n1, 0.0);
  for (int vert = 0; vert < 2; ++vert) {
    std::vector<double>& W = vert ? L->Wv : L->Wh;
    for (int q = 0; q < 7; ++q)
      for (int k = 0; k < n1; ++k)
        for (int m = 0; m < n1; ++m) {
          int w1, r1, c1, w2, r2, c2;
          merged_entry_src(vert != 0, q, k, m, n1, w1, r1, c1, w2, r2, c2);
          double v = block[r1 * Lw + c1];
          if (w2 >= 0) v += block[r2 * Lw + c2];
          W[(q * n1 + k) * n1 + m] = v;
        }
  }
  if (HDG_SHARED_SYM) {
    const bool ok = mirror_reduce(L->Wh, n1, L->Gh) && mirror_reduce(L->Wv, n1, L->Gv);
    if (!ok) {
      // not mirror-symmetric (e.g. side-dependent tau): stream the one block as stored facets
      delete_level_keep_error(L);
      if (nx < 1 || ny < 1 || p < 1 || p > MAXN1 - 1) return fail(HDG_EINVAL, "bad level shape");
      const size_t bb = sizeof(double) * 16 * (size_t)n1 * n1;
      double* dblk = nullptr;
      CK(cudaMalloc(&dblk, bb));
      CK(cudaMemcpy(dblk, block, bb, cudaMemcpyHostToDevice));
      rc = create_stored(nx, ny, p, dblk, true, out);
      cudaFree(dblk);
      return rc;
    }
  }
  if ((rc = prepare(n1, false))) { hdg_level_destroy(L); return rc; }
  *out = L;
  return 0;
}

int hdg_level_create_stored(int nx, int ny, int p, const double* blocks, hdg_level** out) {
  return create_stored(nx, ny, p, blocks, false, out);
}

static int create_stored(int nx, int ny, int p, const double* blocks, bool bcast, hdg_level** out) {
  if (!out) return fail(HDG_EINVAL, "null argument");
  hdg_level* L = new hdg_level();
  L->stored = true;
  int rc = init_level(L, nx, ny, p);
  if (rc) { delete L; return rc; }
  const int n1 = L->n1;
  const long long nslots = (long long)ny * L->nxp;
  const size_t wbytes = sizeof(double) * (size_t)nslots * (HDG_SYMSTORE ? 4 : 7) * n1 * n1;
  L->op_bytes = 0;
  if (L->ndof > 0) {
    if (!blocks) { hdg_level_destroy(L); return fail(HDG_EINVAL, "null blocks"); }
    if (cudaMalloc(&L->dWh, wbytes) != cudaSuccess || cudaMalloc(&L->dWv, wbytes) != cudaSuccess) {
      hdg_level_destroy(L);
      return fail(HDG_ENOMEM, "cannot allocate stored operator streams");
    }
    if (HDG_SYMSTORE && !bcast) {
      // each coupling block is stored once and read transposed by its partner: the element
      // blocks must be symmetric (the condensed operator is, local.py:223-237)
      unsigned long long* dchk = nullptr;
      CK(cudaMalloc(&dchk, 2 * sizeof(unsigned long long)));
      CK(cudaMemset(dchk, 0, 2 * sizeof(unsigned long long)));
      const long long E = (long long)nx * ny, tot = E * 16 * n1 * n1;
#define ASYM_CASE(N) { block_asym_kernel<N><<<(unsigned)((tot + 255) / 256), 256>>>(blocks, E, dchk); CKL(); break; }
      HDG_N1_SWITCH(n1, ASYM_CASE)
#undef ASYM_CASE
      unsigned long long hchk[2];
      CK(cudaMemcpy(hchk, dchk, sizeof(hchk), cudaMemcpyDeviceToHost));
      cudaFree(dchk);
      double asym, mag;
      std::memcpy(&asym, &hchk[0], sizeof(double));
      std::memcpy(&mag, &hchk[1], sizeof(double));
      if (!(asym <= 1e-10 * mag)) {
        hdg_level_destroy(L);
        return fail(HDG_EINVAL, "stored element blocks are not symmetric (max |S - S^T| = " + std::to_string(asym) +
                                    ", max |S| = " + std::to_string(mag) + ")");
      }
    }
    const long long nthr = nslots * (HDG_SYMSTORE ? 4 : 7) * n1 * n1;
    const int bs = 256;
    const long long nbk = (nthr + bs - 1) / bs;
#define RELAYOUT_CASE(N)                                                                         \
  {                                                                                              \
    relayout_kernel<N><<<(unsigned)nbk, bs>>>(blocks, nx, ny, L->nxp, false, L->dWh, bcast);   \
    CKL();                                                                                       \
    relayout_kernel<N><<<(unsigned)nbk, bs>>>(blocks, nx, ny, L->nxp, true, L->dWv, bcast);    \
    CKL();                                                                                       \
    break;                                                                                       \
  }
    HDG_N1_SWITCH(n1, RELAYOUT_CASE)
#undef RELAYOUT_CASE
    CK(cudaDeviceSynchronize());
    // algorithmic operator bytes: the facets' merged matrices (boundary padding excluded)
    L->op_bytes = (long long)L->n_blocks * (HDG_SYMSTORE ? 4 : 7) * n1 * n1 * 8;
  }
  if ((rc = prepare(n1, true))) { hdg_level_destroy(L); return rc; }
  *out = L;
  return 0;
}

// --------------------------------------------------------- stored levels filled by row chunks
// A level whose element blocks never exist at once (configs[4]: 214.7 GB of blocks for a 107 GB
// half-stored stream): the stream is allocated empty and filled chunk by chunk.

int hdg_level_create_stored_empty(int nx, int ny, int p, hdg_level** out) {
  if (!out) return fail(HDG_EINVAL, "null argument");
  hdg_level* L = new hdg_level();
  L->stored = true;
  int rc = init_level(L, nx, ny, p);
  if (rc) { delete L; return rc; }
  const int n1 = L->n1;
  const long long nslots = (long long)ny * L->nxp;
  const size_t wbytes = sizeof(double) * (size_t)nslots * (HDG_SYMSTORE ? 4 : 7) * n1 * n1;
  L->op_bytes = 0;
  if (L->ndof > 0) {
    if (cudaMalloc(&L->dWh, wbytes) != cudaSuccess || cudaMalloc(&L->dWv, wbytes) != cudaSuccess) {
      hdg_level_destroy(L);
      return fail(HDG_ENOMEM, "cannot allocate stored operator streams");
    }
    CK(cudaMemset(L->dWh, 0, wbytes));
    CK(cudaMemset(L->dWv, 0, wbytes));
    L->op_bytes = (long long)L->n_blocks * (HDG_SYMSTORE ? 4 : 7) * n1 * n1 * 8;
  }
  if ((rc = prepare(n1, true))) { hdg_level_destroy(L); return rc; }
  *out = L;
  return 0;
}

int hdg_level_fill_stored_rows(hdg_level* L, int row0, int nrows, const double* blocks, void* stream) {
  if (!L || !L->stored) return fail(HDG_EINVAL, "need a stored level");
  if (row0 < 0 || nrows < 1 || row0 + nrows > L->ny) return fail(HDG_EINVAL, "row chunk outside the mesh");
  if (L->ndof == 0) return 0;
  if (!blocks) return fail(HDG_EINVAL, "null blocks");
  const int n1 = L->n1, nx = L->nx;
  const int erow0 = row0 > 0 ? row0 - 1 : 0;
  const long long E = (long long)(row0 + nrows - erow0) * nx;
  cudaStream_t s = S(stream);
  if (HDG_SYMSTORE) {
    unsigned long long* dchk = nullptr;
    CK(cudaMallocAsync((void**)&dchk, 2 * sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(dchk, 0, 2 * sizeof(unsigned long long), s));
    const long long tot = E * 16 * n1 * n1;
#define ASYMC_CASE(N) { block_asym_kernel<N><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(blocks, E, dchk); CKL(); break; }
    HDG_N1_SWITCH(n1, ASYMC_CASE)
#undef ASYMC_CASE
    unsigned long long hchk[2];
    CK(cudaMemcpyAsync(hchk, dchk, sizeof(hchk), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFreeAsync(dchk, s);
    double asym, mag;
    std::memcpy(&asym, &hchk[0], sizeof(double));
    std::memcpy(&mag, &hchk[1], sizeof(double));
    if (!(asym <= 1e-10 * mag)) return fail(HDG_EINVAL, "stored element blocks are not symmetric");
  }
  const long long nthr = (long long)nrows * L->nxp * (HDG_SYMSTORE ? 4 : 7) * n1 * n1;
  const int bs = 256;
  const long long nbk = (nthr + bs - 1) / bs;
#define RELAYC_CASE(N)                                                                                        \
  {                                                                                                           \
    relayout_kernel<N><<<(unsigned)nbk, bs, 0, s>>>(blocks, nx, L->ny, L->nxp, false, L->dWh, false, row0,   \
                                                    row0 + nrows, erow0);                                     \
    CKL();                                                                                                    \
    relayout_kernel<N><<<(unsigned)nbk, bs, 0, s>>>(blocks, nx, L->ny, L->nxp, true, L->dWv, false, row0,    \
                                                    row0 + nrows, erow0);                                     \
    CKL();                                                                                                    \
    break;                                                                                                    \
  }
  HDG_N1_SWITCH(n1, RELAYC_CASE)
#undef RELAYC_CASE
  return 0;
}

int hdg_level_destroy(hdg_level* L) {
  if (!L) return 0;
  cudaFree(L->dWh); cudaFree(L->dWv); cudaFree(L->dDh); cudaFree(L->dDv); cudaFree(L->partials);
  cudaFree(L->tail_wd);
  cudaFree(L->g_ptr); cudaFree(L->g_col); cudaFree(L->g_val);
  cudaFree(L->gt_ptr); cudaFree(L->gt_col); cudaFree(L->gt_val);
  cudaFree(L->fGh); cudaFree(L->fGv);
  delete L;
  return 0;
}

int64_t hdg_level_ndof(const hdg_level* L) { return L ? L->ndof : -1; }
int64_t hdg_level_operator_bytes(const hdg_level* L) { return L ? L->op_bytes : -1; }

}  // extern "C"

// a new smoother invalidates the fused-tail copy of D and every cycle graph captured with the old one
static void smoother_changed(hdg_level* L) {
  ++L->smoother_gen;
  if (L->tail_wd) { cudaFree(L->tail_wd); L->tail_wd = nullptr; }
}

extern "C" {

int hdg_level_set_blockjacobi(hdg_level* L, double omega) {
  if (!L) return fail(HDG_EINVAL, "null level");
  L->omega = omega;
  const int n1 = L->n1;
  if (!L->stored) {
    L->Dh.assign(L->Wh.begin() + n1 * n1, L->Wh.begin() + 2 * n1 * n1);  // stencil block q = 1
    L->Dv.assign(L->Wv.begin() + n1 * n1, L->Wv.begin() + 2 * n1 * n1);
    host_invert(L->Dh, n1);
    host_invert(L->Dv, n1);
  } else if (L->ndof > 0 && !L->has_bj) {
    const long long nslots = (long long)L->ny * L->nxp;
    const size_t dbytes = sizeof(double) * (size_t)nslots * n1 * n1;
    CK(cudaMalloc(&L->dDh, dbytes));
    CK(cudaMalloc(&L->dDv, dbytes));
    // D = q=1 stencil block of the merged stream; copy it out, then invert in place
    const int bs = 256;
#define DIAG_CASE(N)                                                                      \
  {                                                                                       \
    constexpr int WSZ = Cfg<N>::WSZ, DSZ = Cfg<N>::DSZ;                                  \
    for (int vert = 0; vert < 2; ++vert) {                                                \
      const double* W = vert ? L->dWv : L->dWh;                                           \
      double* D = vert ? L->dDv : L->dDh;                                                 \
      CK(cudaMemcpy2D(D, sizeof(double) * 32 * DSZ, W + (size_t)(HDG_SYMSTORE ? 0 : DSZ) * 32, \
                      sizeof(double) * 32 * WSZ, sizeof(double) * 32 * DSZ, nslots / 32,  \
                      cudaMemcpyDeviceToDevice));                                         \
      invert_kernel<N><<<(unsigned)((nslots + bs - 1) / bs), bs>>>(D, nslots);            \
      CKL();                                                                              \
    }                                                                                     \
    break;                                                                                \
  }
    HDG_N1_SWITCH(n1, DIAG_CASE)
#undef DIAG_CASE
    CK(cudaDeviceSynchronize());
  }
  L->has_bj = true;
  L->use_fsai = false;
  L->bj_cheb = false;
  smoother_changed(L);
  return 0;
}

int hdg_matvec(const hdg_level* L, const double* x, double* y, void* stream) {
  if (!L) return fail(HDG_EINVAL, "null level");
  MvArgs a{};
  a.x = x; a.out = y;
  return apply(L, EPI_Y, a, S(stream));
}

static int res_grid(const hdg_level* L) {
#define RESG_CASE(N) return L->stored ? grid_for<N, true, EPI_RES>(L) : grid_for<N, false, EPI_RES>(L);
  HDG_N1_SWITCH(L->n1, RESG_CASE)
#undef RESG_CASE
}

static int finish_norm(const hdg_level* L, double* norm2_out, cudaStream_t s) {
  const int g = res_grid(L);
  if (g < 0 || g > L->npart) return fail(HDG_ESTATE, "norm partial buffer too small");
  sum_partials_kernel<<<1, 32, 0, s>>>(L->partials, g, norm2_out);
  CKL();
  return 0;
}

int hdg_residual(const hdg_level* L, const double* b, const double* x, double* r, double* norm2_out,
                 void* stream) {
  if (!L) return fail(HDG_EINVAL, "null level");
  if (L->ndof == 0) {
    if (norm2_out) CK(cudaMemsetAsync(norm2_out, 0, sizeof(double), S(stream)));
    return 0;
  }
  MvArgs a{};
  a.x = x; a.b = b; a.out = r; a.partials = norm2_out ? L->partials : nullptr;
  int rc = apply(L, EPI_RES, a, S(stream));
  if (rc || !norm2_out) return rc;
  return finish_norm(L, norm2_out, S(stream));
}

static int bj_sweep_w(const hdg_level* L, const double* b, const double* x_in, double* x_out, double w,
                      cudaStream_t s) {
  if (!L) return fail(HDG_EINVAL, "null level");
  if (!L->has_bj) return fail(HDG_ESTATE, "block-Jacobi state not set (hdg_level_set_blockjacobi)");
  if (x_in == x_out && L->ndof > 0) return fail(HDG_EINVAL, "Jacobi sweep needs x_out != x_in");
  MvArgs a{};
  a.x = x_in; a.b = b; a.out = x_out;
  return apply(L, EPI_BJ, a, s, w);
}

int hdg_bj_sweep(const hdg_level* L, const double* b, const double* x_in, double* x_out, void* stream) {
  return bj_sweep_w(L, b, x_in, x_out, 0.0, S(stream));
}

}  // extern "C"
template <int N1, bool STORED>
static int bj_zero_t(const hdg_level* L, MvArgs& a, double w, cudaStream_t s) {
  SharedOp<(STORED ? 1 : N1)> op;
  if constexpr (!STORED) {
    std::memset(op.Wh, 0, sizeof(op.Wh));
    std::memset(op.Wv, 0, sizeof(op.Wv));
    std::memcpy(op.Dh, L->Dh.data(), sizeof(op.Dh));
    std::memcpy(op.Dv, L->Dv.data(), sizeof(op.Dv));
  } else {
    std::memset(&op, 0, sizeof(op));
  }
  const int bs = 128;
  bj_zero_kernel<N1, STORED><<<(unsigned)((L->n_blocks + bs - 1) / bs), bs, 0, s>>>(a, op, w, L->n_blocks);
  CKL();
  return 0;
}

// x_out = w D^-1 b  (the Jacobi step from x = 0, no operator apply)
static int bj_sweep_zero(const hdg_level* L, const double* b, double* x_out, double w, cudaStream_t s) {
  if (!L->has_bj) return fail(HDG_ESTATE, "block-Jacobi state not set");
  if (L->ndof == 0) return 0;
  MvArgs a{};
  a.nx = L->nx; a.ny = L->ny; a.nxp = L->nxp; a.nh = (int)L->nh;
  a.b = b; a.out = x_out; a.Dh = L->dDh; a.Dv = L->dDv;
#define BJZ_CASE(N) return L->stored ? bj_zero_t<N, true>(L, a, w, s) : bj_zero_t<N, false>(L, a, w, s);
  HDG_N1_SWITCH(L->n1, BJZ_CASE)
#undef BJZ_CASE
}
extern "C" {

// weight of Jacobi step k (1-based) of `steps`: omega, or 1/theta_k (Chebyshev nodes)
static double bj_weight(const hdg_level* L, int k, int steps) {
  if (!L->bj_cheb) return L->omega;
  const double mid = 0.5 * (L->bj_hi + L->bj_lo), half = 0.5 * (L->bj_hi - L->bj_lo);
  return 1.0 / (mid + half * std::cos(M_PI * (2.0 * k - 1.0) / (2.0 * steps)));
}

int hdg_level_set_bj_chebyshev(hdg_level* L, double lo, double hi) {
  if (!L) return fail(HDG_EINVAL, "null level");
  if (!L->has_bj) return fail(HDG_ESTATE, "set block-Jacobi first");
  if (!(hi > lo && lo > 0.0)) return fail(HDG_EINVAL, "need 0 < lo < hi");
  L->bj_cheb = true; L->bj_lo = lo; L->bj_hi = hi;
  smoother_changed(L);
  return 0;
}

int hdg_bj_sweeps(const hdg_level* L, const double* b, double* x, double* work, int steps, void* stream) {
  // `steps` (Chebyshev-)weighted Jacobi sweeps in place (ping-pong through work)
  double* cur = x;
  double* oth = work;
  int rc;
  for (int k = 1; k <= steps; ++k) {
    if ((rc = bj_sweep_w(L, b, cur, oth, bj_weight(L, k, steps), S(stream)))) return rc;
    std::swap(cur, oth);
  }
  if (cur != x && L->ndof > 0)
    CK(cudaMemcpyAsync(x, cur, sizeof(double) * L->ndof, cudaMemcpyDeviceToDevice, S(stream)));
  return 0;
}

// -------------------------------------------------------------------------------- FSAI

}  // extern "C"
template <typename T>
static int upload(T** dst, const T* src, size_t n) {
  cudaFree(*dst);
  *dst = nullptr;
  CK(cudaMalloc(dst, sizeof(T) * (n ? n : 1)));
  if (n) CK(cudaMemcpy(*dst, src, sizeof(T) * n, cudaMemcpyHostToDevice));
  return 0;
}
extern "C" {

int hdg_fsai_rows(int64_t n, const int32_t* a_ptr, const int32_t* a_col, const double* a_val, const int32_t* g_ptr,
                  const int32_t* g_col, double* g_val, int32_t max_len, int64_t* bad_row, void* stream) {
  if (n < 0 || !bad_row) return fail(HDG_EINVAL, "bad arguments");
  if (n == 0) { *bad_row = -1; return 0; }
  long long* dbad = nullptr;
  CK(cudaMalloc(&dbad, sizeof(long long)));
  const long long init = LLONG_MAX;
  CK(cudaMemcpyAsync(dbad, &init, sizeof(long long), cudaMemcpyHostToDevice, S(stream)));
  const int bs = 128;
  const unsigned grid = (unsigned)((n + bs - 1) / bs);
  int rc = 0;
  if (max_len <= 24) fsai_rows_kernel<24><<<grid, bs, 0, S(stream)>>>(n, a_ptr, a_col, a_val, g_ptr, g_col, g_val, dbad);
  else if (max_len <= 40) fsai_rows_kernel<40><<<grid, bs, 0, S(stream)>>>(n, a_ptr, a_col, a_val, g_ptr, g_col, g_val, dbad);
  else if (max_len <= 64) fsai_rows_kernel<64><<<grid, bs, 0, S(stream)>>>(n, a_ptr, a_col, a_val, g_ptr, g_col, g_val, dbad);
  else if (max_len <= 96) fsai_rows_kernel<96><<<grid, bs, 0, S(stream)>>>(n, a_ptr, a_col, a_val, g_ptr, g_col, g_val, dbad);
  else rc = fail(HDG_EINVAL, "FSAI pattern rows longer than 96 entries");
  if (!rc) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = fail(HDG_ECUDA, std::string("fsai rows: ") + cudaGetErrorString(e));
  }
  long long hb = LLONG_MAX;
  if (!rc) {
    cudaError_t e = cudaMemcpyAsync(&hb, dbad, sizeof(long long), cudaMemcpyDeviceToHost, S(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
    if (e != cudaSuccess) rc = fail(HDG_ECUDA, std::string("fsai rows: ") + cudaGetErrorString(e));
  }
  cudaFree(dbad);
  *bad_row = (hb == LLONG_MAX) ? -1 : hb;
  return rc;
}

int hdg_level_set_fsai(hdg_level* L, int64_t n, const int32_t* g_ptr, const int32_t* g_col, const double* g_val,
                       int64_t nnz, const int32_t* gt_ptr, const int32_t* gt_col, const double* gt_val,
                       double lam_max, double cheb_fraction, double omega) {
  if (!L) return fail(HDG_EINVAL, "null level");
  if (n != L->ndof) return fail(HDG_EINVAL, "FSAI factor size != level ndof");
  // invalidate first: a failed upload must leave a level the cycle refuses, never stale graphs
  // replaying freed factor arrays
  L->has_fsai = false;
  L->use_fsai = false;
  smoother_changed(L);
  int rc;
  if ((rc = upload(&L->g_ptr, g_ptr, n + 1)) || (rc = upload(&L->g_col, g_col, nnz)) ||
      (rc = upload(&L->g_val, g_val, nnz)) || (rc = upload(&L->gt_ptr, gt_ptr, n + 1)) ||
      (rc = upload(&L->gt_col, gt_col, nnz)) || (rc = upload(&L->gt_val, gt_val, nnz)))
    return rc;
  L->lam_max = lam_max; L->cheb_frac = cheb_fraction; L->fsai_omega = omega;
  L->fsai_struct = false;
  L->has_fsai = true;
  L->use_fsai = true;
  smoother_changed(L);
  return 0;
}

}  // extern "C"
template <int N1>
static int fsai_struct_apply_t(const hdg_level* L, bool transposed, const double* x, double* y, const double* xin,
                               double w, cudaStream_t s) {
  FsaiApplyArgs a{};
  a.Gh = L->fGh; a.Gv = L->fGv; a.x = x; a.y = y; a.xin = xin; a.w = w;
  a.nx = L->nx; a.ny = L->ny; a.nh = L->nh; a.nvf = (long long)(L->nx - 1) * L->ny;
  const long long nf = a.nh + a.nvf;
  const int bs = 128;
  const unsigned grid = (unsigned)((nf + bs - 1) / bs);
  if (!transposed) fsai_g_kernel<N1><<<grid, bs, 0, s>>>(a);
  else if (xin) fsai_gt_kernel<N1, true><<<grid, bs, 0, s>>>(a);
  else fsai_gt_kernel<N1, false><<<grid, bs, 0, s>>>(a);
  CKL();
  return 0;
}

#define HDG_FSAI_SWITCH(n1, CALL)                                             \
  switch (n1) {                                                               \
    case 2: CALL(2); case 3: CALL(3); case 4: CALL(4); case 5: CALL(5);       \
    case 6: CALL(6); case 7: CALL(7); case 8: CALL(8); case 9: CALL(9);       \
    default: return fail(HDG_EINVAL, "structured FSAI: p <= 8");              \
  }

static int spmv(const hdg_level* L, bool transposed, const double* x, double* y, const double* xin, double w,
                cudaStream_t s) {
  const int n = (int)L->ndof;
  if (n == 0) return 0;
  if (L->fsai_struct) {
#define FSA_CASE(N) return fsai_struct_apply_t<N>(L, transposed, x, y, xin, w, s);
    HDG_FSAI_SWITCH(L->n1, FSA_CASE)
#undef FSA_CASE
  }
  const int bs = 256;
  const unsigned grid = (unsigned)(((long long)n * 4 + bs - 1) / bs);
  const int* rp = transposed ? L->gt_ptr : L->g_ptr;
  const int* ci = transposed ? L->gt_col : L->g_col;
  const double* v = transposed ? L->gt_val : L->g_val;
  if (xin) csr_spmv_kernel<true><<<grid, bs, 0, s>>>(n, rp, ci, v, x, y, xin, w);
  else csr_spmv_kernel<false><<<grid, bs, 0, s>>>(n, rp, ci, v, x, y, nullptr, 0.0);
  CKL();
  return 0;
}

extern "C" {

// Chebyshev-weighted steps (multigrid.py:76-81)
static double fsai_weight(const hdg_level* L, int k, int steps) {
  const double lo = L->cheb_frac * L->lam_max, hi = L->lam_max;
  const double mid = 0.5 * (hi + lo), half = 0.5 * (hi - lo);
  const double theta = mid + half * std::cos(M_PI * (2.0 * k - 1.0) / (2.0 * steps));
  return L->fsai_omega / theta;
}

int hdg_fsai_apply(const hdg_level* L, const double* r, double* z, void* stream) {
  if (!L || !L->has_fsai) return fail(HDG_ESTATE, "FSAI state not set");
  if (L->ndof == 0) return 0;
  double* t = nullptr;
  CK(cudaMallocAsync(&t, sizeof(double) * L->ndof, S(stream)));
  int rc = spmv(L, false, r, t, nullptr, 0.0, S(stream));
  if (!rc) rc = spmv(L, true, t, z, nullptr, 0.0, S(stream));
  cudaFreeAsync(t, S(stream));
  return rc;
}

// x_zero: x is all zeros on entry (a cycle visit from x = 0, multigrid.py:400): the first step's residual
// is b itself, so its operator apply - a full pass over the level's block stream - is skipped
// (b - A 0 = b exactly: the iterates are bitwise the same)
static int fsai_sweeps(const hdg_level* L, const double* b, double* x, double* r, double* t, int steps,
                       cudaStream_t s, bool x_zero = false) {
  for (int k = 1; k <= steps; ++k) {
    int rc;
    const double* rk = r;
    if (k == 1 && x_zero) rk = b;
    else if ((rc = hdg_residual(L, b, x, r, nullptr, s))) return rc;         // r = b - A x
    if ((rc = spmv(L, false, rk, t, nullptr, 0.0, s))) return rc;            // t = G r
    if ((rc = spmv(L, true, t, x, x, fsai_weight(L, k, steps), s))) return rc;  // x += w G't
  }
  return 0;
}

int hdg_fsai_sweeps(const hdg_level* L, const double* b, double* x, double* work_r, double* work_t, int steps,
                    void* stream) {
  if (!L || !L->has_fsai) return fail(HDG_ESTATE, "FSAI state not set");
  if (L->ndof == 0 || steps < 1) return 0;
  return fsai_sweeps(L, b, x, work_r, work_t, steps, S(stream));
}

}  // extern "C"

// --------------------------------------------------------------- facet-structured FSAI setup

template <int N1>
static int fsai_struct_setup_t(hdg_level* L, const double* S, const long long* cls, const double* v0, int iters,
                               double* lams_host, long long* bad_host, cudaStream_t s) {
  const long long nvf = (long long)(L->nx - 1) * L->ny;
  const size_t ghb = sizeof(double) * (size_t)L->nh * N1 * 2 * N1;
  const size_t gvb = sizeof(double) * (size_t)nvf * N1 * 6 * N1;
  cudaFree(L->fGh); cudaFree(L->fGv);
  L->fGh = L->fGv = nullptr;
  if (cudaMalloc(&L->fGh, ghb ? ghb : 8) != cudaSuccess || cudaMalloc(&L->fGv, gvb ? gvb : 8) != cudaSuccess)
    return fail(HDG_ENOMEM, "cannot allocate the FSAI factor");
  double* Dg = nullptr;
  long long* bad = nullptr;
  CK(cudaMallocAsync((void**)&Dg, sizeof(double) * (size_t)L->n_blocks * N1 * N1, s));
  CK(cudaMallocAsync((void**)&bad, sizeof(long long), s));
  const long long init = LLONG_MAX;
  CK(cudaMemcpyAsync(bad, &init, sizeof(long long), cudaMemcpyHostToDevice, s));
  const long long nd = L->n_blocks * N1 * N1;
  fsai_diag_kernel<N1><<<(unsigned)((nd + 255) / 256), 256, 0, s>>>(S, cls, L->nx, L->ny, L->nh, L->n_blocks, Dg);
  CKL();
  static int occ = -1;
  if (occ < 0) {
    CK(cudaFuncSetAttribute(fsai_setup_kernel<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, FsaiCfg<N1>::SMEM));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fsai_setup_kernel<N1>, 32 * FsaiCfg<N1>::WARPS,
                                                      FsaiCfg<N1>::SMEM) != cudaSuccess || occ < 1)
      occ = 1;
  }
  FsaiSetupArgs a{};
  a.S = S; a.cls = cls; a.Dg = Dg; a.Gh = L->fGh; a.Gv = L->fGv; a.bad = bad;
  a.nx = L->nx; a.ny = L->ny; a.nh = L->nh; a.nvf = nvf;
  const long long nf = L->nh + nvf;
  const long long want = (nf + FsaiCfg<N1>::WARPS - 1) / FsaiCfg<N1>::WARPS;
  const long long grid = std::min(want, (long long)sm_count() * occ);
  fsai_setup_kernel<N1><<<(unsigned)std::max(grid, 1LL), 32 * FsaiCfg<N1>::WARPS, FsaiCfg<N1>::SMEM, s>>>(a);
  CKL();
  cudaFreeAsync(Dg, s);
  CK(cudaMemcpyAsync(bad_host, bad, sizeof(long long), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(bad, s);
  CK(cudaStreamSynchronize(s));
  if (*bad_host != LLONG_MAX) return 0;
  // lambda_max(G'G A): power iteration from the caller's start vector (multigrid.py:162-173)
  L->fsai_struct = true;   // spmv() below dispatches to the structured kernels
  const size_t vb = sizeof(double) * (size_t)L->ndof;
  double *v = nullptr, *q = nullptr, *t = nullptr, *w = nullptr, *nrm = nullptr, *lam = nullptr, *part = nullptr;
  CK(cudaMallocAsync((void**)&v, vb, s)); CK(cudaMallocAsync((void**)&q, vb, s));
  CK(cudaMallocAsync((void**)&t, vb, s)); CK(cudaMallocAsync((void**)&w, vb, s));
  CK(cudaMallocAsync((void**)&nrm, sizeof(double), s));
  CK(cudaMallocAsync((void**)&lam, sizeof(double) * std::max(iters, 1), s));
  CK(cudaMallocAsync((void**)&part, sizeof(double) * vec_blocks(), s));
  CK(cudaMemcpyAsync(v, v0, vb, cudaMemcpyDeviceToDevice, s));
  int rc = 0;
  for (int it = 0; it < iters && !rc; ++it) {
    MvArgs ma{};
    ma.x = v; ma.out = q;
    rc = apply(L, EPI_Y, ma, s);                                      // A v
    if (!rc) rc = spmv(L, false, q, t, nullptr, 0.0, s);              // G A v
    if (!rc) rc = spmv(L, true, t, w, nullptr, 0.0, s);               // G' G A v
    if (!rc) rc = dot_into(w, w, L->ndof, nrm, part, s);
    if (!rc) { fsai_scale_kernel<<<vec_blocks(), 256, 0, s>>>(w, nrm, v, lam + it, L->ndof); CKL(); }
  }
  if (!rc && iters > 0) {
    if (cudaMemcpyAsync(lams_host, lam, sizeof(double) * iters, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      rc = fail(HDG_ECUDA, "lambda_max readback");
  }
  cudaFreeAsync(v, s); cudaFreeAsync(q, s); cudaFreeAsync(t, s); cudaFreeAsync(w, s);
  cudaFreeAsync(nrm, s); cudaFreeAsync(lam, s); cudaFreeAsync(part, s);
  return rc;
}

extern "C" {

int hdg_level_set_fsai_struct(hdg_level* L, const double* S_cls, const int64_t* elem_class, const double* v0,
                              int lam_iters, double cheb_fraction, double omega, double* lam_max_out,
                              int64_t* bad_row, void* stream) {
  if (!L || !lam_max_out || !bad_row) return fail(HDG_EINVAL, "null argument");
  *bad_row = -1;
  // invalidate first (a failure leaves a level the cycle refuses)
  L->has_fsai = L->use_fsai = L->fsai_struct = false;
  smoother_changed(L);
  if (L->ndof == 0) {
    *lam_max_out = 1.0;
    L->lam_max = 1.0; L->cheb_frac = cheb_fraction; L->fsai_omega = omega;
    L->fsai_struct = L->has_fsai = L->use_fsai = true;
    return 0;
  }
  if (!S_cls || !elem_class || !v0 || lam_iters < 1) return fail(HDG_EINVAL, "null argument");
  std::vector<double> lams(lam_iters, 0.0);
  long long bad = LLONG_MAX;
  cudaStream_t s = S(stream);
  int rc;
#define FSS_CASE(N) { rc = fsai_struct_setup_t<N>(L, S_cls, reinterpret_cast<const long long*>(elem_class), v0, \
                                                  lam_iters, lams.data(), &bad, s); break; }
  switch (L->n1) {
    case 2: FSS_CASE(2) case 3: FSS_CASE(3) case 4: FSS_CASE(4) case 5: FSS_CASE(5)
    case 6: FSS_CASE(6) case 7: FSS_CASE(7) case 8: FSS_CASE(8) case 9: FSS_CASE(9)
    default: return fail(HDG_EINVAL, "structured FSAI: p <= 8");
  }
#undef FSS_CASE
  if (rc) { L->fsai_struct = false; return rc; }
  if (bad != LLONG_MAX) {
    L->fsai_struct = false;
    *bad_row = bad;
    return fail(HDG_ESTATE, "non-SPD principal submatrix in FSAI row " + std::to_string(bad));
  }
  double lam = 1.0;
  for (int it = 0; it < lam_iters; ++it) {            // multigrid.py:167-172
    lam = lams[it];
    if (lam == 0.0) { lam = 1.0; break; }
  }
  *lam_max_out = lam;
  L->lam_max = lam; L->cheb_frac = cheb_fraction; L->fsai_omega = omega;
  L->fsai_struct = L->has_fsai = L->use_fsai = true;
  smoother_changed(L);
  return 0;
}

int hdg_level_fsai_struct_get(const hdg_level* L, double* gh_host, double* gv_host) {
  if (!L || !L->fsai_struct) return fail(HDG_ESTATE, "no structured FSAI on this level");
  const long long nvf = (long long)(L->nx - 1) * L->ny;
  const int n1 = L->n1;
  if (L->nh && gh_host) CK(cudaMemcpy(gh_host, L->fGh, sizeof(double) * L->nh * n1 * 2 * n1, cudaMemcpyDeviceToHost));
  if (nvf && gv_host) CK(cudaMemcpy(gv_host, L->fGv, sizeof(double) * nvf * n1 * 6 * n1, cudaMemcpyDeviceToHost));
  return 0;
}

// ---------------------------------------------------------------------------- transfers

int hdg_transfer_create_p(const hdg_level* fine, const hdg_level* coarse, const double* V, hdg_transfer** out) {
  if (!fine || !coarse || !V || !out) return fail(HDG_EINVAL, "null argument");
  if (fine->nx != coarse->nx || fine->ny != coarse->ny || fine->n1 != coarse->n1 + 1)
    return fail(HDG_EINVAL, "p-transfer needs the same mesh and p_coarse = p_fine - 1");
  hdg_transfer* t = new hdg_transfer();
  t->fine = fine; t->coarse = coarse;
  std::memcpy(t->pa.V, V, sizeof(double) * fine->n1 * coarse->n1);
  *out = t;
  return 0;
}

int hdg_transfer_create_h_window(const hdg_level* fine, const hdg_level* coarse, const double* halves,
                                 const double* cross, int64_t nsets, int fine_row0, int coarse_row0,
                                 hdg_transfer** out) {
  if (!fine || !coarse || !halves || !cross || !out) return fail(HDG_EINVAL, "null argument");
  if (fine->n1 != 2 || coarse->n1 != 2) return fail(HDG_EINVAL, "h-transfer runs at p = 1");
  if (fine->nx != 2 * coarse->nx) return fail(HDG_EINVAL, "h-transfer needs nx_fine = 2 nx_coarse");
  if (fine_row0 < 0 || coarse_row0 < 0) return fail(HDG_EINVAL, "negative window offset");
  const long long Ec = (long long)coarse->nx * coarse->ny;
  if (nsets != 1 && nsets != Ec) return fail(HDG_EINVAL, "cross maps: 1 shared set or one per coarse element");
  hdg_transfer* t = new hdg_transfer();
  t->is_h = true; t->fine = fine; t->coarse = coarse;
  t->ha.nxc = coarse->nx; t->ha.nyc = coarse->ny; t->ha.nyf = fine->ny;
  t->ha.jf0 = fine_row0; t->ha.jc0 = coarse_row0;
  t->ha.nhf = fine->nh; t->ha.nhc = coarse->nh;
  std::memcpy(t->ha.halves, halves, sizeof(double) * 8);
  const size_t bytes = sizeof(double) * 64 * (size_t)nsets;
  if (cudaMalloc(&t->dcross, bytes) != cudaSuccess) { delete t; return fail(HDG_ENOMEM, "cross maps"); }
  CK(cudaMemcpy(t->dcross, cross, bytes, cudaMemcpyHostToDevice));
  t->ha.cross = t->dcross;
  t->ha.shared_cross = (nsets == 1) ? 1 : 0;
  if (nsets == 1) std::memcpy(t->ha.cross_c, cross, sizeof(t->ha.cross_c));
  *out = t;
  return 0;
}

int hdg_transfer_create_h(const hdg_level* fine, const hdg_level* coarse, const double* halves, const double* cross,
                          int64_t nsets, hdg_transfer** out) {
  if (fine && coarse && fine->ny != 2 * coarse->ny)
    return fail(HDG_EINVAL, "h-transfer needs the fine mesh = 2x the coarse mesh");
  return hdg_transfer_create_h_window(fine, coarse, halves, cross, nsets, 0, 0, out);
}

int hdg_transfer_destroy(hdg_transfer* t) {
  if (!t) return 0;
  cudaFree(t->dcross);
  delete t;
  return 0;
}

int hdg_prolong_add(const hdg_transfer* t, const double* ec, double* xf, void* stream) {
  if (!t) return fail(HDG_EINVAL, "null transfer");
  const long long nf = t->fine->n_blocks;
  if (nf == 0) return 0;
  const int bs = 256;
  const unsigned grid = (unsigned)((nf + bs - 1) / bs);
  if (t->is_h) {
    launch_pdl(h_prolong_add_kernel, dim3(grid), dim3(bs), 0, S(stream), t->ha, ec, xf);
    CKL();
    return 0;
  }
#define PPROL_CASE(N) { p_prolong_add_kernel<N><<<grid, bs, 0, S(stream)>>>(ec, xf, nf, t->pa); CKL(); return 0; }
  HDG_N1_SWITCH(t->fine->n1, PPROL_CASE)
#undef PPROL_CASE
}

int hdg_restrict(const hdg_transfer* t, const double* rf, double* rc, void* stream) {
  if (!t) return fail(HDG_EINVAL, "null transfer");
  const int bs = 256;
  if (t->is_h) {
    const long long nc = t->coarse->n_blocks;
    if (nc == 0) return 0;
    launch_pdl(h_restrict_kernel, dim3((unsigned)((nc + bs - 1) / bs)), dim3(bs), 0, S(stream), t->ha, rf, rc);
    CKL();
    return 0;
  }
  const long long nf = t->fine->n_blocks;
  if (nf == 0) return 0;
  const unsigned grid = (unsigned)((nf + bs - 1) / bs);
#define PRES_CASE(N) { p_restrict_kernel<N><<<grid, bs, 0, S(stream)>>>(rf, rc, nf, t->pa); CKL(); return 0; }
  HDG_N1_SWITCH(t->fine->n1, PRES_CASE)
#undef PRES_CASE
}

// ---------------------------------------------------------------------------- reductions

}  // extern "C"

// streaming grid of the vector kernels: 4 CTAs of 256 threads per SM of this device
static int vec_blocks() { return 4 * sm_count(); }

// partials live in a stream-ordered allocation per call: concurrent streams / threads never share
// a buffer, and the allocation is captured as a graph node when the call is captured
static int dot_into(const double* a, const double* b, int64_t n, double* out, double* partials, cudaStream_t s) {
  const int nb = vec_blocks();
  dot_partials_kernel<<<nb, 256, 0, s>>>(a, b, n, partials);
  CKL();
  sum_partials_kernel<<<1, 32, 0, s>>>(partials, nb, out);
  CKL();
  return 0;
}

extern "C" {

int hdg_dot(const double* a, const double* b, int64_t n, double* out, void* stream) {
  if (!out || (n > 0 && (!a || !b))) return fail(HDG_EINVAL, "null argument");
  double* partials = nullptr;
  CK(cudaMallocAsync((void**)&partials, sizeof(double) * vec_blocks(), S(stream)));
  const int rc = dot_into(a, b, n, out, partials, S(stream));
  cudaFreeAsync(partials, S(stream));
  return rc;
}

int hdg_cg_update(double* x, double* r, const double* d, const double* ad, double alpha, int64_t n, void* stream) {
  if (n <= 0) return 0;
  cg_update_kernel<<<vec_blocks(), 256, 0, S(stream)>>>(x, r, d, ad, alpha, n);
  CKL();
  return 0;
}

int hdg_xpby(const double* z, double beta, double* d, int64_t n, void* stream) {
  if (n <= 0) return 0;
  xpby_kernel<<<vec_blocks(), 256, 0, S(stream)>>>(z, beta, d, n);
  CKL();
  return 0;
}

// ----------------------------------------------------------------------------- multigrid

int hdg_mg_create(hdg_level* const* levels, hdg_transfer* const* transfers, int n, hdg_mg** out) {
  if (!levels || !out || n < 1) return fail(HDG_EINVAL, "need at least one level");
  hdg_mg* mg = new hdg_mg();
  mg->n = n;
  for (int k = 0; k < n; ++k) {
    if (!levels[k]) { delete mg; return fail(HDG_EINVAL, "null level"); }
    mg->L.push_back(levels[k]);
    if (k + 1 < n) {
      hdg_transfer* t = transfers ? transfers[k] : nullptr;
      if (!t || t->fine != levels[k] || t->coarse != levels[k + 1]) {
        delete mg;
        return fail(HDG_EINVAL, "transfer k must map level k+1 into level k");
      }
      mg->T.push_back(t);
      if (!levels[k]->has_bj && !levels[k]->has_fsai) {
        delete mg;
        return fail(HDG_ESTATE, "every non-coarsest level needs a smoother");
      }
    }
  }
  mg->X.assign(n, nullptr); mg->Tm.assign(n, nullptr); mg->B.assign(n, nullptr); mg->R.assign(n, nullptr);
  for (int k = 0; k < n; ++k) {
    const size_t bytes = sizeof(double) * (size_t)(mg->L[k]->ndof + 1);
    if (k > 0) {
      CK(cudaMalloc(&mg->X[k], bytes));
      CK(cudaMalloc(&mg->B[k], bytes));
    }
    CK(cudaMalloc(&mg->Tm[k], bytes));
    if (k + 1 < n) CK(cudaMalloc(&mg->R[k], bytes));
  }
  CK(cudaStreamCreateWithFlags(&mg->cs, cudaStreamNonBlocking));
  *out = mg;
  return 0;
}

int hdg_mg_destroy(hdg_mg* mg) {
  if (!mg) return 0;
  for (auto& kv : mg->graphs) cudaGraphExecDestroy(kv.second.exec);
  for (int k = 0; k < mg->n; ++k) {
    if (k > 0) cudaFree(mg->X[k]);
    cudaFree(mg->Tm[k]); cudaFree(mg->B[k]); cudaFree(mg->R[k]);
  }
  cudaFree(mg->Ainv);
  for (double* q : mg->Xr) cudaFree(q);
  for (double* q : mg->Tr) cudaFree(q);
  for (double* q : mg->Br) cudaFree(q);
  cudaFree(mg->Rr);
  if (mg->cs) cudaStreamDestroy(mg->cs);
  delete mg;
  return 0;
}

int hdg_mg_set_records(hdg_mg* mg, int mode) {
  if (!mg || mode < 0 || mode > 4)
    return fail(HDG_EINVAL, "record mode must be 0 (off), 1 (auto), 2 (on), 3 (on, unfused), 4 (on, every h-level)");
  mg->rec_mode = mode >= 3 ? 2 : mode;
  mg->rec_h_all = mode == 4;
  mg->rec_fuse_prolong = mode != 3;
  mg->rec_fold_first = mode != 3;
  for (auto& kv : mg->graphs) cudaGraphExecDestroy(kv.second.exec);
  mg->graphs.clear();
  return 0;
}

int hdg_mg_record_levels(const hdg_mg* mg) { return mg ? mg->rec_m : -1; }

int hdg_mg_set_fused_tail(hdg_mg* mg, int enable) {
  if (!mg) return fail(HDG_EINVAL, "null mg");
  mg->tail_enabled = enable != 0;
  mg->fuse_first = enable != 0;
  for (auto& kv : mg->graphs) cudaGraphExecDestroy(kv.second.exec);
  mg->graphs.clear();
  return 0;
}

int hdg_mg_set_coarse_inverse(hdg_mg* mg, const double* inv, int64_t n) {
  if (!mg || !inv) return fail(HDG_EINVAL, "null argument");
  if (n != mg->L[mg->n - 1]->ndof) return fail(HDG_EINVAL, "coarse inverse size != coarsest ndof");
  cudaFree(mg->Ainv);
  mg->Ainv = nullptr;
  mg->nc = n;
  if (n > 0) {
    CK(cudaMalloc(&mg->Ainv, sizeof(double) * n * n));
    CK(cudaMemcpy(mg->Ainv, inv, sizeof(double) * n * n, cudaMemcpyHostToDevice));
  }
  for (auto& kv : mg->graphs) cudaGraphExecDestroy(kv.second.exec);
  mg->graphs.clear();
  return 0;
}

static int coarse_apply(hdg_mg* mg, const double* b, double* x, cudaStream_t s) {
  if (mg->nc == 0) return 0;
  if (!mg->Ainv) return fail(HDG_ESTATE, "coarse inverse not set");
  const int rows_per_block = 8;
  dense_gemv_kernel<<<(unsigned)((mg->nc + rows_per_block - 1) / rows_per_block), 32 * rows_per_block, 0, s>>>(
      mg->Ainv, b, x, (int)mg->nc);
  CKL();
  return 0;
}

int hdg_coarse_solve(hdg_mg* mg, const double* b, double* x, void* stream) {
  if (!mg) return fail(HDG_EINVAL, "null mg");
  return coarse_apply(mg, b, x, S(stream));
}

// ------------------------------------------------------------------ fused coarse-level tail
// Levels k0..n-1 run as one single-CTA kernel with all their vectors in shared memory
// (hdg_kernels.cuh: tail_cycle_kernel) when they are all p = 1, linked by h-transfers and
// smoothed by block-Jacobi, and their X, T, B vectors fit the shared-memory budget.
// vectors; + the program copy + shared operators <= 218 KB
static const long long TAIL_SMEM_DOUBLES = 27200 - TAIL_ARGS_DOUBLES - 64 * TAIL_MAXL;

static const long long TAIL_MAX_TOP_DOF = 2048;

static long long tail_footprint(const hdg_mg* mg, int k0) {
  long long d = 0;
  for (int k = k0; k < mg->n; ++k) d += 3 * (mg->L[k]->ndof + (mg->L[k]->ndof & 1));
  return d;
}

static int tail_find(const hdg_mg* mg) {
  if (!mg->tail_enabled) return -1;
  int k0 = -1;
  for (int k = mg->n - 1; k >= 0; --k) {
    const hdg_level* L = mg->L[k];
    if (L->n1 != 2) break;
    if (k < mg->n - 1 && (!mg->T[k]->is_h || L->use_fsai || !L->has_bj)) break;
    if (mg->n - k > TAIL_MAXL || tail_footprint(mg, k) > TAIL_SMEM_DOUBLES) break;
    // one CTA beats ~6 launches per level visit only while the level is small (measured on B200:
    // a 960-dof level costs 14 us inside the tail vs 26 us as launches, a 3968-dof level 43 vs 27)
    if (L->ndof > TAIL_MAX_TOP_DOF) break;
    k0 = k;
  }
  return (k0 >= 0 && k0 < mg->n - 1) ? k0 : -1;   // a tail needs at least one smoothed level
}

// device copies of the shared-mode operators of the tail levels (outside any stream capture)
static int tail_prepare(hdg_mg* mg) {
  mg->tail_k0 = tail_find(mg);
  if (mg->tail_k0 < 0) return 0;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(tail_cycle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)((TAIL_SMEM_DOUBLES + TAIL_ARGS_DOUBLES + 64 * TAIL_MAXL) * sizeof(double))));
    attr = true;
  }
  for (int k = mg->tail_k0; k < mg->n; ++k) {
    hdg_level* L = mg->L[k];
    if (L->stored || L->tail_wd) continue;
    std::vector<double> h(64, 0.0);
    std::copy(L->Wh.begin(), L->Wh.end(), h.begin());
    std::copy(L->Wv.begin(), L->Wv.end(), h.begin() + 28);
    if (L->has_bj) {
      std::copy(L->Dh.begin(), L->Dh.end(), h.begin() + 56);
      std::copy(L->Dv.begin(), L->Dv.end(), h.begin() + 60);
    }
    CK(cudaMalloc(&L->tail_wd, sizeof(double) * 64));
    CK(cudaMemcpy(L->tail_wd, h.data(), sizeof(double) * 64, cudaMemcpyHostToDevice));
  }
  return 0;
}

// the same recursion, sweep weights and buffer roles as cycle_rec (multigrid.py:393-406), on
// buffer ids 3 * (k - k0) + {0: X, 1: T, 2: B}; the residual reuses the free T buffer
struct TailGen {
  hdg_mg* mg;
  TailArgs* A;
  int k0, nu1, nu2, visits;
  bool overflow = false;
  void emit(int code, int k, int x, int b, int out, double w = 0.0) {
    if (A->nops >= TAIL_MAXOPS) { overflow = true; return; }
    TailOp& o = A->ops[A->nops++];
    o.code = (short)code; o.lev = (short)(k - k0); o.x = (short)x; o.b = (short)b; o.out = (short)out; o.w = w;
  }
  int id(int k, int role) const { return 3 * (k - k0) + role; }
  void gen(int k, bool zero_init) {
    hdg_level* L = mg->L[k];
    const int xk = id(k, 0), bk = id(k, 2);
    if (k == mg->n - 1) { if (mg->nc > 0) emit(T_COARSE, k, -1, bk, xk); return; }
    if (L->ndof == 0) return;
    int cur = xk, oth = id(k, 1), first = 0;
    if (zero_init) {
      if (nu1 >= 1) {
        emit(T_BJZ, k, -1, bk, oth, bj_weight(L, 1, nu1));
        std::swap(cur, oth);
        first = 1;
      } else {
        emit(T_ZERO, k, -1, -1, xk);
      }
    }
    for (int it = first; it < nu1; ++it) {
      emit(T_BJ, k, cur, bk, oth, bj_weight(L, it + 1, nu1));
      std::swap(cur, oth);
    }
    emit(T_RES, k, cur, bk, oth);
    emit(T_RESTRICT, k, oth, -1, id(k + 1, 2));
    for (int v = 0; v < visits; ++v) gen(k + 1, v == 0);
    emit(T_PROLONG, k, id(k + 1, 0), -1, cur);
    for (int it = 0; it < nu2; ++it) {
      emit(T_BJ, k, cur, bk, oth, bj_weight(L, it + 1, nu2));
      std::swap(cur, oth);
    }
    if (cur != xk) emit(T_COPY, k, cur, -1, xk);
  }
};

// returns 1 when the tail was issued, 0 when it does not apply (program too long), < 0 on error
static int tail_issue(hdg_mg* mg, const double* b, bool zero_init, int nu1, int nu2, int visits, cudaStream_t s) {
  const int k0 = mg->tail_k0;
  if (mg->nc > 0 && !mg->Ainv) return fail(HDG_ESTATE, "coarse inverse not set");
  TailArgs* A = new TailArgs();
  std::memset(A, 0, sizeof(TailArgs));
  long long off = 0;
  for (int k = k0; k < mg->n; ++k) {
    const hdg_level* L = mg->L[k];
    TailLevel& t = A->lev[k - k0];
    t.nx = L->nx; t.ny = L->ny; t.nxp = L->nxp; t.stored = L->stored ? 1 : 0;
    t.nh = L->nh; t.nblk = L->n_blocks;
    if (L->stored) {
      t.W[0] = L->dWh; t.W[1] = L->dWv; t.D[0] = L->dDh; t.D[1] = L->dDv;
    } else {
      t.W[0] = L->tail_wd; t.W[1] = L->tail_wd + 28; t.D[0] = L->tail_wd + 56; t.D[1] = L->tail_wd + 60;
    }
    const long long len = L->ndof + (L->ndof & 1);   // keep every vector 16-byte aligned
    for (int r = 0; r < 3; ++r) { t.off[r] = (int)off; off += len; }
    if (k + 1 < mg->n) A->h[k - k0] = mg->T[k]->ha;
  }
  A->Ainv = mg->Ainv;
  A->nc = (int)mg->nc;
  A->nlev = mg->n - k0;
  A->b_in = b;
  A->x_in = zero_init ? nullptr : mg->X[k0];
  A->x_out = mg->X[k0];
  TailGen g{mg, A, k0, nu1, nu2, visits};
  g.gen(k0, zero_init);
  if (g.overflow) { delete A; return 0; }
  launch_pdl(tail_cycle_kernel, dim3(1), dim3(TAIL_THREADS), (size_t)(off + TAIL_ARGS_DOUBLES + 64 * TAIL_MAXL) * sizeof(double), s, *A);
  delete A;
  CKL();
  return 1;
}

// multigrid.py:393-406, device resident: on entry the level-k iterate is X[k] (or zero),
// on exit the result is in X[k].
static int cycle_rec(hdg_mg* mg, int k, const double* b, bool zero_init, int nu1, int nu2, int visits,
                     cudaStream_t s) {
  hdg_level* L = mg->L[k];
  double* xk = mg->X[k];
  if (k == mg->tail_k0) {
    const int t = tail_issue(mg, b, zero_init, nu1, nu2, visits, s);
    if (t != 0) return t < 0 ? t : 0;
  }
  if (k == mg->n - 1) return coarse_apply(mg, b, xk, s);
  const size_t bytes = sizeof(double) * (size_t)L->ndof;
  double* cur = xk;
  double* oth = mg->Tm[k];
  int rc;
  const bool fsai = L->use_fsai;   // the smoother attached last (FSAI or block-Jacobi)
  int first = 0;
  if (zero_init && L->ndof > 0) {
    if (!fsai && nu1 >= 2 && !L->stored && mg->fuse_first) {
      // x = 0: x_1 = w1 D^-1 b is formed on the staged tile of b inside the second sweep's
      // kernel (one pass instead of bj_zero + sweep)
      MvArgs a{};
      a.x = b; a.b = b; a.out = oth; a.w_first = bj_weight(L, 1, nu1);
      if ((rc = apply(L, EPI_BJ, a, s, bj_weight(L, 2, nu1)))) return rc;
      std::swap(cur, oth);
      first = 2;
    } else if (!fsai && nu1 >= 1) {
      // x = 0: the first Jacobi step needs no operator apply (x_1 = w D^-1 b)
      if ((rc = bj_sweep_zero(L, b, oth, bj_weight(L, 1, nu1), s))) return rc;
      std::swap(cur, oth);
      first = 1;
    } else {
      CK(cudaMemsetAsync(xk, 0, bytes, s));
    }
  }
  if (fsai) {
    if ((rc = fsai_sweeps(L, b, cur, mg->R[k], oth, nu1, s, zero_init && L->ndof > 0))) return rc;
  } else {
    for (int it = first; it < nu1; ++it) {
      if ((rc = bj_sweep_w(L, b, cur, oth, bj_weight(L, it + 1, nu1), s))) return rc;
      std::swap(cur, oth);
    }
  }
  hdg_transfer* T = mg->T[k];
  if (!T->is_h) {
    MvArgs a{};
    a.x = cur; a.b = b; a.out = mg->B[k + 1];
    std::memcpy(a.V, T->pa.V, sizeof(a.V));
    if ((rc = apply(L, EPI_RESPR, a, s))) return rc;
  } else {
    if ((rc = hdg_residual(L, b, cur, mg->R[k], nullptr, s))) return rc;
    if ((rc = hdg_restrict(T, mg->R[k], mg->B[k + 1], s))) return rc;
  }
  for (int v = 0; v < visits; ++v)
    if ((rc = cycle_rec(mg, k + 1, mg->B[k + 1], v == 0, nu1, nu2, visits, s))) return rc;
  int post0 = 0;
  if (!T->is_h && !fsai && nu2 >= 1 && mg->fuse_first) {
    // p-prolongation fused into the first post-smoothing sweep: x + V e_c is formed on the
    // staged tile and never stored
    MvArgs a{};
    a.x = cur; a.b = b; a.out = oth; a.pec = mg->X[k + 1];
    std::memcpy(a.V, T->pa.V, sizeof(a.V));
    if ((rc = apply(L, EPI_BJ, a, s, bj_weight(L, 1, nu2)))) return rc;
    std::swap(cur, oth);
    post0 = 1;
  } else if ((rc = hdg_prolong_add(T, mg->X[k + 1], cur, s))) {
    return rc;
  }
  if (fsai) {
    if ((rc = fsai_sweeps(L, b, cur, mg->R[k], oth, nu2, s))) return rc;
  } else {
    for (int it = post0; it < nu2; ++it) {
      if ((rc = bj_sweep_w(L, b, cur, oth, bj_weight(L, it + 1, nu2), s))) return rc;
      std::swap(cur, oth);
    }
  }
  if (cur != xk && L->ndof > 0) CK(cudaMemcpyAsync(xk, cur, bytes, cudaMemcpyDeviceToDevice, s));
  return 0;
}

// ------------------------------------------------------------------ record-layout cycle
// Levels 0 .. m-1 qualify when they are the constant-coefficient (shared, mirror-symmetric) p-ladder of
// the finest mesh, smoothed by block-Jacobi, and level m-1 (p = 1) is linked to level m by a whole-mesh
// h-transfer; the recursion below level m-1 is cycle_rec on the reference layout.
static long long rec_min_dof() {
  static long long v = -1;
  if (v < 0) {
    const char* e = std::getenv("HDG_REC_MIN_DOF");
    v = e ? std::atoll(e) : (1LL << 13);
  }
  return v;
}

static long long rec_h_min_dof() {
  static long long v = -1;
  if (v < 0) {
    const char* e = std::getenv("HDG_REC_H_MIN_DOF");
    v = e ? std::atoll(e) : 50000;   // measured on the configs[1] hierarchy: 0.746 ms without, 0.728 / 0.725 / 0.722 ms
                                     // with the levels down to 512^2 / 256^2 / 128^2 on records
  }
  return v;
}

static int rec_find(hdg_mg* mg) {
  if (mg->rec_mode == 0 || mg->n < 2) return 0;
  hdg_level* L0 = mg->L[0];
  // automatic mode: hierarchies with a p-ladder from ~8k fine dofs (measured faster from 32^2, p = 4 up to
  // 1024^2, p = 4; a p = 1 hierarchy has a single record level and only pays the layout changes)
  if (mg->rec_mode == 1 && (L0->ndof < rec_min_dof() || L0->n1 < 3)) return 0;
  int m = 0;
  for (int k = 0; k + 1 < mg->n; ++k) {
    hdg_level* L = mg->L[k];
    if (L->stored || L->blk.empty() || L->n1 > SOA_CYCLE_MAXN1 || !L->has_bj || L->use_fsai || L->nx != L0->nx ||
        L->ny != L0->ny || L->ndof == 0)
      return 0;
    if (soa_prepare(L)) return 0;
    soa_prepare_bj0(L);
    if (mg->T[k]->is_h) {
      const HArgs& h = mg->T[k]->ha;
      if (L->n1 != 2 || h.jf0 != 0 || h.jc0 != 0 || h.nyf != 2 * h.nyc || L->nx != 2 * h.nxc || L->ny != h.nyf)
        return 0;
      m = k + 1;
      break;
    }
  }
  // h-coarsened p = 1 levels that are still large keep their vectors as records too (record-to-record
  // h-transfers); the first level below them is the reference-layout one
  while (m >= 1 && m + 1 < mg->n) {
    hdg_level* L = mg->L[m];
    const HArgs& h = mg->T[m]->ha;
    if (L->stored || L->blk.empty() || L->n1 != 2 || !L->has_bj || L->use_fsai ||
        (!mg->rec_h_all && L->ndof < rec_h_min_dof()) ||
        !mg->T[m]->is_h || h.jf0 != 0 || h.jc0 != 0 || h.nyf != 2 * h.nyc || L->nx != 2 * h.nxc || L->ny != h.nyf)
      break;
    if (soa_prepare(L)) break;
    soa_prepare_bj0(L);
    ++m;
  }
  return m;
}

// allocate the record vectors (outside any stream capture)
static int rec_prepare(hdg_mg* mg) {
  const int m = rec_find(mg);
  if (m == mg->rec_m && (m == 0 || !mg->Xr.empty())) return 0;
  for (double* q : mg->Xr) cudaFree(q);
  for (double* q : mg->Tr) cudaFree(q);
  for (double* q : mg->Br) cudaFree(q);
  cudaFree(mg->Rr);
  mg->Xr.clear(); mg->Tr.clear(); mg->Br.clear(); mg->Rr = nullptr;
  mg->rec_m = m;
  for (int k = 0; k < m; ++k) {
    const size_t bytes = sizeof(double) * (size_t)soa_len(mg->L[k]);
    double *a = nullptr, *b = nullptr, *c = nullptr;
    CK(cudaMalloc(&a, bytes)); mg->Xr.push_back(a);
    CK(cudaMalloc(&b, bytes)); mg->Tr.push_back(b);
    CK(cudaMalloc(&c, bytes)); mg->Br.push_back(c);
    CK(cudaMemset(c, 0, bytes));   // a record-to-record restriction writes facet slots only
  }
  for (int k = 0; k < m && !mg->Rr; ++k)   // residual records of the h-linked levels: the first is the largest
    if (mg->T[k]->is_h) CK(cudaMalloc(&mg->Rr, sizeof(double) * (size_t)soa_len(mg->L[k])));
  return 0;
}

static int cycle_rec(hdg_mg* mg, int k, const double* b, bool zero_init, int nu1, int nu2, int visits,
                     cudaStream_t s);

// multigrid.py:393-406 on facet records: level-k right-hand side b and iterate x_in (null: zero) are
// records; the result is left in one of the level's two buffers, returned through x_out
static int cycle_rec_soa(hdg_mg* mg, int k, const double* b, const double* x_in, double** x_out, int nu1, int nu2,
                         int visits, cudaStream_t s, double* final_out = nullptr) {
  hdg_level* L = mg->L[k];
  double* const A = mg->Xr[k];
  double* const Bf = mg->Tr[k];
  auto other = [&](const double* q) { return q == A ? Bf : A; };
  const double* cur = x_in;
  int rc, first = 0;
  if (!x_in) {
    if (nu1 >= 1) {
      // x = 0: x1 = w1 D^-1 b is formed per facet on the streamed b records and the second sweep
      // runs in the same pass (nu1 = 1: the second step has weight 0)
      const double w1 = bj_weight(L, 1, nu1), w2 = nu1 >= 2 ? bj_weight(L, 2, nu1) : 0.0;
      const int epi0 = (!L->soaM0.empty() && mg->rec_fold_first) ? SOA_EPI_BJ0F : SOA_EPI_BJ0;
      if ((rc = soa_cyc_sweep(L, epi0, b, b, A, w2, w1, nullptr, nullptr, s))) return rc;
      first = nu1 >= 2 ? 2 : 1;
    } else {
      CK(cudaMemsetAsync(A, 0, sizeof(double) * (size_t)soa_len(L), s));
    }
    cur = A;
  }
  for (int it = first; it < nu1; ++it) {
    double* out = other(cur);
    if ((rc = soa_cyc_sweep(L, SOA_EPI_BJ, cur, b, out, bj_weight(L, it + 1, nu1), 0.0, nullptr, nullptr, s))) return rc;
    cur = out;
  }
  hdg_transfer* T = mg->T[k];
  int post0 = 0;
  if (!T->is_h) {
    if ((rc = soa_cyc_sweep(L, SOA_EPI_RESPR, cur, b, mg->Br[k + 1], 0.0, 0.0, T->pa.V, nullptr, s))) return rc;
    double* xc = nullptr;
    for (int v = 0; v < visits; ++v)
      if ((rc = cycle_rec_soa(mg, k + 1, mg->Br[k + 1], xc, &xc, nu1, nu2, visits, s))) return rc;
    if (nu2 >= 1 && mg->rec_fuse_prolong) {
      double* out = (final_out && nu2 == 1 && final_out != cur && final_out != b) ? final_out : other(cur);
      if ((rc = soa_cyc_sweep(L, SOA_EPI_BJ, cur, b, out, bj_weight(L, 1, nu2), 0.0, T->pa.V, xc, s))) return rc;
      cur = out;
      post0 = 1;
    } else if ((rc = soa_cyc_p_prolong(L, mg->L[k + 1], xc, const_cast<double*>(cur), T->pa.V, s))) {
      return rc;
    }
  } else if (k + 1 < mg->rec_m) {
    // h-link between two record levels
    hdg_level* Lc = mg->L[k + 1];
    if ((rc = soa_cyc_sweep(L, SOA_EPI_RES, cur, b, mg->Rr, 0.0, 0.0, nullptr, nullptr, s))) return rc;
    if ((rc = soa_cyc_h_restrict(L, T->ha, mg->Rr, mg->Br[k + 1], s, Lc))) return rc;
    double* xc = nullptr;
    for (int v = 0; v < visits; ++v)
      if ((rc = cycle_rec_soa(mg, k + 1, mg->Br[k + 1], xc, &xc, nu1, nu2, visits, s))) return rc;
    if ((rc = soa_cyc_h_prolong(L, T->ha, xc, const_cast<double*>(cur), s, Lc))) return rc;
  } else {
    if ((rc = soa_cyc_sweep(L, SOA_EPI_RES, cur, b, mg->Rr, 0.0, 0.0, nullptr, nullptr, s))) return rc;
    if ((rc = soa_cyc_h_restrict(L, T->ha, mg->Rr, mg->B[k + 1], s))) return rc;
    for (int v = 0; v < visits; ++v)
      if ((rc = cycle_rec(mg, k + 1, mg->B[k + 1], v == 0, nu1, nu2, visits, s))) return rc;
    if ((rc = soa_cyc_h_prolong(L, T->ha, mg->X[k + 1], const_cast<double*>(cur), s))) return rc;
  }
  for (int it = post0; it < nu2; ++it) {
    // the caller's result buffer receives the last sweep directly
    double* out = (final_out && it == nu2 - 1 && final_out != cur && final_out != b) ? final_out : other(cur);
    if ((rc = soa_cyc_sweep(L, SOA_EPI_BJ, cur, b, out, bj_weight(L, it + 1, nu2), 0.0, nullptr, nullptr, s))) return rc;
    cur = out;
  }
  if (final_out && cur != final_out) {
    CK(cudaMemcpyAsync(final_out, cur, sizeof(double) * (size_t)soa_len(L), cudaMemcpyDeviceToDevice, s));
    cur = final_out;
  }
  *x_out = const_cast<double*>(cur);
  return 0;
}

static int cycle_issue(hdg_mg* mg, const double* b, const double* x0, double* x, int nu1, int nu2, int visits,
                       cudaStream_t s) {
  if (mg->rec_m > 0) {
    hdg_level* L0 = mg->L[0];
    int rc;
    if ((rc = hdg_soa_pack(L0, b, mg->Br[0], s))) return rc;
    const double* xin = nullptr;
    if (x0) {
      if ((rc = hdg_soa_pack(L0, x0, mg->Xr[0], s))) return rc;
      xin = mg->Xr[0];
    }
    double* res = nullptr;
    if ((rc = cycle_rec_soa(mg, 0, mg->Br[0], xin, &res, nu1, nu2, visits, s))) return rc;
    return hdg_soa_unpack(L0, res, x, s);
  }
  const size_t bytes = sizeof(double) * (size_t)mg->L[0]->ndof;
  mg->X[0] = x;
  bool zero = (x0 == nullptr);
  if (!zero && x0 != x && bytes) CK(cudaMemcpyAsync(x, x0, bytes, cudaMemcpyDeviceToDevice, s));
  return cycle_rec(mg, 0, b, zero, nu1, nu2, visits, s);
}

// smoothers re-attached since the last capture: every cached cycle graph is stale
static void refresh_graphs(hdg_mg* mg) {
  std::vector<unsigned> gens(mg->n);
  for (int k = 0; k < mg->n; ++k) gens[k] = mg->L[k]->smoother_gen;
  if (gens != mg->gens) {
    for (auto& kv : mg->graphs) cudaGraphExecDestroy(kv.second.exec);
    mg->graphs.clear();
    mg->gens = gens;
  }
}

// records = true: b, x0, x are facet records of level 0 (no pack / unpack at the boundary)
static int cycle_issue_any(hdg_mg* mg, bool records, const double* b, const double* x0, double* x, int nu1, int nu2,
                           int visits, cudaStream_t s) {
  if (!records) return cycle_issue(mg, b, x0, x, nu1, nu2, visits, s);
  if (x0 && nu1 == 0) {   // no pre-sweep: the correction would be added to the caller's x0 in place
    CK(cudaMemcpyAsync(mg->Xr[0], x0, sizeof(double) * (size_t)soa_len(mg->L[0]), cudaMemcpyDeviceToDevice, s));
    x0 = mg->Xr[0];
  }
  double* res = nullptr;
  return cycle_rec_soa(mg, 0, b, x0, &res, nu1, nu2, visits, s, x);
}

static int run_cycle(hdg_mg* mg, bool records, const double* b, const double* x0, double* x, int nu1, int nu2,
                     int visits, int use_graph, void* stream) {
  if (!mg || !b || !x) return fail(HDG_EINVAL, "null argument");
  refresh_graphs(mg);
  if (nu1 < 0 || nu2 < 0 || visits < 1) return fail(HDG_EINVAL, "bad cycle parameters");
  if (mg->L[0]->ndof == 0) return 0;
  cudaStream_t s = S(stream);
  int rc0 = tail_prepare(mg);
  if (rc0) return rc0;
  const int m0 = mg->rec_m;
  if ((rc0 = rec_prepare(mg))) return rc0;
  if (m0 != mg->rec_m) {                       // the record levels changed: cached graphs are stale
    for (auto& kv : mg->graphs) cudaGraphExecDestroy(kv.second.exec);
    mg->graphs.clear();
  }
  if (records) {
    if (mg->rec_m == 0) return fail(HDG_ESTATE, "this hierarchy has no record levels (hdg_mg_set_records)");
    if (b == x) return fail(HDG_EINVAL, "record cycle: x must not alias b");
  }
  if (!use_graph) return cycle_issue_any(mg, records, b, x0, x, nu1, nu2, visits, s);
  auto key = std::make_tuple((const void*)b, (const void*)x0, (void*)x, nu1, nu2, records ? -visits : visits);
  auto it = mg->graphs.find(key);
  if (it == mg->graphs.end()) {
    const long long c0 = g_launches.load();
    CK(cudaStreamBeginCapture(mg->cs, cudaStreamCaptureModeThreadLocal));
    int rc = cycle_issue_any(mg, records, b, x0, x, nu1, nu2, visits, mg->cs);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(mg->cs, &g);
    if (rc) { if (g) cudaGraphDestroy(g); return rc; }
    if (e != cudaSuccess) return fail(HDG_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
    GraphEntry ge{};
    e = cudaGraphInstantiate(&ge.exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(HDG_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    ge.nkern = g_launches.load() - c0;
    g_launches.fetch_sub(ge.nkern);
    ++mg->graph_captures;
    while (mg->graphs.size() >= MAX_CYCLE_GRAPHS) {          // LRU eviction
      auto old = mg->graphs.begin();
      for (auto g2 = mg->graphs.begin(); g2 != mg->graphs.end(); ++g2)
        if (g2->second.last_use < old->second.last_use) old = g2;
      cudaGraphExecDestroy(old->second.exec);
      mg->graphs.erase(old);
    }
    it = mg->graphs.emplace(key, ge).first;
  }
  it->second.last_use = ++mg->use_clock;
  CK(cudaGraphLaunch(it->second.exec, s));
  g_launches.fetch_add(it->second.nkern);
  return 0;
}

int hdg_mg_cycle(hdg_mg* mg, const double* b, const double* x0, double* x, int nu1, int nu2, int visits,
                 int use_graph, void* stream) {
  return run_cycle(mg, false, b, x0, x, nu1, nu2, visits, use_graph, stream);
}

int hdg_mg_cycle_records(hdg_mg* mg, const double* b_rec, const double* x0_rec, double* x_rec, int nu1, int nu2,
                         int visits, int use_graph, void* stream) {
  return run_cycle(mg, true, b_rec, x0_rec, x_rec, nu1, nu2, visits, use_graph, stream);
}

int64_t hdg_mg_graph_captures(const hdg_mg* mg) { return mg ? mg->graph_captures : -1; }

// ------------------------------------------------------------------ native solve loops
// solve_mg (multigrid.py:421-439) and solve_cg (trace.py:142-163) with every vector on the
// device: one scalar crosses to the host per cycle / iteration (the stop test), as in the
// reference's own loop structure.

static int fetch(const double* dsrc, double* h, int count, cudaStream_t s) {
  CK(cudaMemcpyAsync(h, dsrc, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

static int run_cycle(hdg_mg* mg, bool records, const double* b, const double* x0, double* x, int nu1, int nu2,
                     int visits, int use_graph, void* stream);

int hdg_solve_mg(hdg_mg* mg, const double* b, double* x, int nu1, int nu2, int visits, double tol,
                 int max_cycles, double* res_hist, int* ncycles, void* stream) {
  if (!mg || !b || !x || !res_hist || !ncycles) return fail(HDG_EINVAL, "null argument");
  if (max_cycles < 0) return fail(HDG_EINVAL, "max_cycles must be >= 0");
  cudaStream_t s = S(stream);
  hdg_level* L0 = mg->L[0];
  const long long n = L0->ndof;
  *ncycles = 0;
  if (n == 0) { res_hist[0] = 0.0; return 0; }
  refresh_graphs(mg);
  int rc = tail_prepare(mg);
  if (!rc) rc = rec_prepare(mg);
  if (rc) return rc;
  // with record levels the whole loop keeps b, x and the residual as facet records: one pack of b and
  // x0, one unpack of x, no layout change per cycle
  const bool rec = mg->rec_m > 0;
  const int nb = vec_blocks();
  double *scal = nullptr, *partials = nullptr, *bR = nullptr, *xR = nullptr, *rR = nullptr;
  CK(cudaMallocAsync((void**)&scal, sizeof(double) * 2, s));
  CK(cudaMallocAsync((void**)&partials, sizeof(double) * nb, s));
  if (rec) {
    const size_t rb = sizeof(double) * (size_t)soa_len(L0);
    CK(cudaMallocAsync((void**)&bR, rb, s));
    CK(cudaMallocAsync((void**)&xR, rb, s));
    CK(cudaMallocAsync((void**)&rR, rb, s));
    rc = hdg_soa_pack(L0, b, bR, s);
    if (!rc) rc = hdg_soa_pack(L0, x, xR, s);
  }
  auto resnorm = [&]() -> int {                                   // scal[1] = ||b - A x||^2
    if (!rec) return hdg_residual(L0, b, x, nullptr, scal + 1, s);
    int r2 = soa_cyc_sweep(L0, SOA_EPI_RES, xR, bR, rR, 0.0, 0.0, nullptr, nullptr, s);
    return r2 ? r2 : soa_cyc_norm2(L0, rR, scal + 1, partials, nb, s);
  };
  if (!rc) rc = dot_into(b, b, n, scal, partials, s);
  double h[2];
  if (!rc) rc = resnorm();
  if (!rc) rc = fetch(scal, h, 2, s);
  const double bnorm = (rc || h[0] == 0.0) ? 1.0 : std::sqrt(h[0]);
  if (!rc) res_hist[0] = std::sqrt(h[1]);
  int k = 0;
  while (!rc && k < max_cycles) {
    if (res_hist[k] <= tol * bnorm) break;                     // multigrid.py:433
    rc = rec ? run_cycle(mg, true, bR, xR, xR, nu1, nu2, visits, 1, stream)
             : hdg_mg_cycle(mg, b, x, x, nu1, nu2, visits, 1, stream);
    if (!rc) rc = resnorm();
    if (!rc) rc = fetch(scal + 1, h + 1, 1, s);
    if (rc) break;
    res_hist[++k] = std::sqrt(h[1]);
    if (k >= 5) {                                               // monitor.diverged(): 5 rho >= 1
      bool div = true;
      for (int i = k - 5; i < k; ++i) {
        const double rho = res_hist[i] > 0.0 ? res_hist[i + 1] / res_hist[i] : 0.0;
        if (!(rho >= 1.0)) { div = false; break; }
      }
      if (div) break;
    }
  }
  if (rec && !rc) rc = hdg_soa_unpack(L0, xR, x, s);
  if (rec) { cudaFreeAsync(rR, s); cudaFreeAsync(xR, s); cudaFreeAsync(bR, s); }
  cudaFreeAsync(partials, s);
  cudaFreeAsync(scal, s);
  *ncycles = k;
  return rc;
}

int hdg_pcg(const hdg_level* L, hdg_mg* mg, const double* b, double* x, int use_x0, double tol, int maxiter,
            int nu1, int nu2, double* res_hist, int* iters, void* stream) {
  if (!L || !b || !x || !iters) return fail(HDG_EINVAL, "null argument");
  if (mg && mg->L[0]->ndof != L->ndof) return fail(HDG_EINVAL, "preconditioner size != operator size");
  if (maxiter < 0) return fail(HDG_EINVAL, "maxiter must be >= 0");
  cudaStream_t s = S(stream);
  const long long n = L->ndof;
  *iters = 0;
  if (n == 0) { if (res_hist) res_hist[0] = 0.0; return 0; }
  const int nb = vec_blocks();
  int rc = 0;
  if (mg) { refresh_graphs(mg); if ((rc = tail_prepare(mg))) return rc; if ((rc = rec_prepare(mg))) return rc; }
  // preconditioner with record levels on the operator's own level: every CG vector is a facet record for
  // the whole solve (operator apply = the record kernel, dots masked to the trace dofs, updates
  // slot-wise: pads and duplicate slots stay consistent); b and x0 are packed once, x unpacked once
  hdg_level* L0 = mg ? mg->L[0] : nullptr;
  const bool rec = mg && mg->rec_m > 0 && L0 == L;
  const long long N = rec ? soa_len(L0) : n;                     // vector length of the loop
  const size_t vb = sizeof(double) * (size_t)N;
  double *r = nullptr, *z = nullptr, *d = nullptr, *ad = nullptr, *scal = nullptr, *part = nullptr;
  double *xw = x, *bw = nullptr;                                 // working iterate / packed right-hand side
  CK(cudaMallocAsync((void**)&r, vb, s));
  CK(cudaMallocAsync((void**)&d, vb, s));
  CK(cudaMallocAsync((void**)&ad, vb, s));
  if (mg) CK(cudaMallocAsync((void**)&z, vb, s)); else z = r;
  if (rec) { CK(cudaMallocAsync((void**)&xw, vb, s)); CK(cudaMallocAsync((void**)&bw, vb, s)); }
  CK(cudaMallocAsync((void**)&scal, sizeof(double) * 8, s));
  CK(cudaMallocAsync((void**)&part, sizeof(double) * 2 * nb, s));
  cudaStream_t cs = nullptr;
  cudaGraphExec_t body = nullptr;
  auto precond = [&](cudaStream_t st) -> int {                   // z = M r (one V-cycle from zero)
    if (!mg) return 0;
    return rec ? cycle_issue_any(mg, true, r, nullptr, z, nu1, nu2, 1, st) : cycle_issue(mg, r, nullptr, z, nu1, nu2, 1, st);
  };
  auto dot = [&](const double* u, const double* v, double* out, cudaStream_t st) -> int {
    return rec ? soa_cyc_dot2(L0, u, v, out, nullptr, nullptr, nullptr, part, nb, st) : dot_into(u, v, n, out, part, st);
  };
  do {
    // r = b - A x0 (trace.py:147), z = M r, d = z, rz = r.z
    if (rec && (rc = hdg_soa_pack(L0, b, bw, s))) break;
    if (use_x0) {
      if (rec) {
        if ((rc = hdg_soa_pack(L0, x, xw, s))) break;
        if ((rc = soa_cyc_sweep(L0, SOA_EPI_RES, xw, bw, r, 0.0, 0.0, nullptr, nullptr, s))) break;
      } else if ((rc = hdg_residual(L, b, x, r, nullptr, s))) break;
    } else {
      if (cudaMemsetAsync(xw, 0, vb, s) != cudaSuccess ||
          cudaMemcpyAsync(r, rec ? bw : b, vb, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
        rc = fail(HDG_ECUDA, "pcg init copies"); break;
      }
    }
    if ((rc = precond(s))) break;
    if (cudaMemcpyAsync(d, z, vb, cudaMemcpyDeviceToDevice, s) != cudaSuccess) { rc = fail(HDG_ECUDA, "pcg copy"); break; }
    if ((rc = dot(r, z, scal + 0, s))) break;
    if ((rc = dot_into(b, b, n, scal + 4, part, s))) break;
    if ((rc = dot(r, r, scal + 3, s))) break;
    // one iteration body (trace.py:153-162) captured once, replayed per iteration
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) { rc = fail(HDG_ECUDA, "stream"); break; }
    const long long c0 = g_launches.load();
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { rc = fail(HDG_ECUDA, "capture"); break; }
    {
      if (rec) {
        rc = hdg_matvec_soa(L0, d, ad, cs);                                   // ad = A d
      } else {
        MvArgs a{};
        a.x = d; a.out = ad;
        rc = apply(L, EPI_Y, a, cs);
      }
      if (!rc) rc = dot(d, ad, scal + 1, cs);                                 // d.Ad
      if (!rc) { cg_update_dev_kernel<<<nb, 256, 0, cs>>>(xw, r, d, ad, scal, N); CKL(); }
      if (!rc) rc = precond(cs);                                              // z = M r
      if (rec) {
        if (!rc) rc = soa_cyc_dot2(L0, r, z, scal + 2, r, r, scal + 3, part, nb, cs);        // r.z, r.r
      } else {
        if (!rc) { dot2_partials_kernel<<<nb, 256, 0, cs>>>(r, z, r, r, n, part); CKL(); }
        if (!rc) { sum_partials_kernel<<<1, 32, 0, cs>>>(part, nb, scal + 2); CKL(); }       // r.z
        if (!rc) { sum_partials_kernel<<<1, 32, 0, cs>>>(part + nb, nb, scal + 3); CKL(); }  // r.r
      }
      if (!rc) { xpby_dev_kernel<<<nb, 256, 0, cs>>>(z, scal, d, N); CKL(); }              // d = z + beta d
      if (!rc && cudaMemcpyAsync(scal, scal + 2, sizeof(double), cudaMemcpyDeviceToDevice, cs) != cudaSuccess)
        rc = fail(HDG_ECUDA, "pcg scalar copy");
    }
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(cs, &g);
    const long long nk = g_launches.load() - c0;
    g_launches.fetch_sub(nk);
    if (rc) { if (g) cudaGraphDestroy(g); break; }
    if (ec != cudaSuccess) { rc = fail(HDG_ECUDA, std::string("pcg capture: ") + cudaGetErrorString(ec)); break; }
    const cudaError_t ei = cudaGraphInstantiate(&body, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) { rc = fail(HDG_ECUDA, std::string("pcg instantiate: ") + cudaGetErrorString(ei)); break; }
    double h[2];
    if ((rc = fetch(scal + 3, h, 2, s))) break;                   // r.r, b.b
    const double bnorm = h[1] > 0.0 ? std::sqrt(h[1]) : 1.0;
    double rr = h[0];
    int it = 0;
    for (; it < maxiter; ++it) {
      const double rn = std::sqrt(rr);
      if (res_hist) res_hist[it] = rn;
      if (rn <= tol * bnorm) break;                                // trace.py:152
      if (cudaGraphLaunch(body, s) != cudaSuccess) { rc = fail(HDG_ECUDA, "pcg graph launch"); break; }
      g_launches.fetch_add(nk);
      if ((rc = fetch(scal + 3, &rr, 1, s))) break;
    }
    if (!rc && it == maxiter && res_hist) res_hist[maxiter] = std::sqrt(rr);
    *iters = it;
    if (!rc && rec) rc = hdg_soa_unpack(L0, xw, x, s);
  } while (false);
  if (body) cudaGraphExecDestroy(body);
  if (cs) cudaStreamDestroy(cs);
  cudaFreeAsync(part, s); cudaFreeAsync(scal, s);
  if (rec) { cudaFreeAsync(bw, s); cudaFreeAsync(xw, s); }
  cudaFreeAsync(ad, s); cudaFreeAsync(d, s); cudaFreeAsync(r, s);
  if (mg) cudaFreeAsync(z, s);
  return rc;
}

}  // extern "C"

// ----------------------------------------------------------- facet-plane (SoA) layout

// Symmetry-adapted blocks of the element block (hdg_soa.cuh).  T = forward butterflies (rows
// orthogonal, T T^T = D), y = T^T M T x with M = D^-1 T S T^T D^-1; M is block diagonal when S
// commutes with both element mirrors, and symmetric when S is (the kernel stores the upper
// triangles).  Off-block entries or asymmetry above 1e-11 max|M| -> not available.
template <int N1>
static bool soa_reduce(const std::vector<double>& S, std::vector<double>& out, bool symmetric = true) {
  using C = SoaCfg<N1>;
  constexpr int NT = 4 * N1;
  std::vector<double> T(NT * NT), TT(NT * NT);
  for (int j = 0; j < NT; ++j) {                      // columns of T
    double x[NT] = {}, t[NT];
    x[j] = 1.0;
    soa_forward<N1>(x, x + N1, x + 2 * N1, x + 3 * N1, t);
    for (int i = 0; i < NT; ++i) T[i * NT + j] = t[i];
  }
  for (int i = 0; i < NT; ++i) {                      // columns of the backward map must be rows of T
    double t[NT] = {}, y[NT];
    t[i] = 1.0;
    soa_backward<N1>(t, y, y + N1, y + 2 * N1, y + 3 * N1);
    for (int j = 0; j < NT; ++j)
      if (y[j] != T[i * NT + j]) return false;
  }
  std::vector<double> D(NT, 0.0);
  for (int i = 0; i < NT; ++i) {
    for (int j = 0; j < NT; ++j) D[i] += T[i * NT + j] * T[i * NT + j];
    for (int m = 0; m < NT; ++m)
      if (m != i) {
        double dot = 0.0;
        for (int j = 0; j < NT; ++j) dot += T[i * NT + j] * T[m * NT + j];
        if (dot != 0.0) return false;
      }
  }
  std::vector<double> A(NT * NT, 0.0), M(NT * NT, 0.0);   // A = S T^T, M = T A / (D_i D_j)
  for (int r = 0; r < NT; ++r)
    for (int m = 0; m < NT; ++m) {
      double acc = 0.0;
      for (int j = 0; j < NT; ++j) acc += S[r * NT + j] * T[m * NT + j];
      A[r * NT + m] = acc;
    }
  double mx = 0.0;
  for (int i = 0; i < NT; ++i)
    for (int m = 0; m < NT; ++m) {
      double acc = 0.0;
      for (int r = 0; r < NT; ++r) acc += T[i * NT + r] * A[r * NT + m];
      M[i * NT + m] = acc / (D[i] * D[m]);
      mx = std::fmax(mx, std::fabs(M[i * NT + m]));
    }
  const int off[5] = {0, C::A0, C::A0 + C::A1, C::A0 + C::A1 + C::A2, NT};
  auto cls = [&](int i) { int c = 0; while (i >= off[c + 1]) ++c; return c; };
  double defect = 0.0;
  for (int i = 0; i < NT; ++i)
    for (int m = 0; m < NT; ++m)
      defect = std::fmax(defect, cls(i) != cls(m) ? std::fabs(M[i * NT + m])
                                                  : (symmetric ? std::fabs(M[i * NT + m] - M[m * NT + i]) : 0.0));
  if (!(defect <= 1e-11 * mx)) return false;
  out.clear();
  for (int c = 0; c < 4; ++c)
    for (int i = off[c]; i < off[c + 1]; ++i)
      for (int m = off[c]; m < off[c + 1]; ++m)
        out.push_back(symmetric ? 0.5 * (M[i * NT + m] + M[m * NT + i]) : M[i * NT + m]);
  return (int)out.size() == C::MSZ;
}

// class blocks of S' = S blockdiag(Dh^-1, Dv^-1, Dh^-1, Dv^-1) (sides bottom, right, top, left): the
// zero-start double sweep x2 = D^-1((w0 + w) b - w w0 S' b) applies them to the raw right-hand side
int soa_prepare_bj0(hdg_level* L) {
  if (L->soaM0_gen == L->smoother_gen && !L->soaM0.empty()) return 0;
  L->soaM0.clear();
  if (L->n1 > 5 || !L->has_bj || L->blk.empty() || L->Dh.empty() || L->Dv.empty()) return 0;
  const int n1 = L->n1, NT = 4 * n1;
  std::vector<double> Sp((size_t)NT * NT, 0.0);
  for (int r = 0; r < NT; ++r)
    for (int sd = 0; sd < 4; ++sd) {
      const std::vector<double>& Dm = (sd & 1) ? L->Dv : L->Dh;
      for (int c = 0; c < n1; ++c) {
        double acc = 0.0;
        for (int k = 0; k < n1; ++k) acc += L->blk[(size_t)r * NT + sd * n1 + k] * Dm[k * n1 + c];
        Sp[(size_t)r * NT + sd * n1 + c] = acc;
      }
    }
  bool ok = false;
  switch (n1) {
    case 2: ok = soa_reduce<2>(Sp, L->soaM0, false); break;
    case 3: ok = soa_reduce<3>(Sp, L->soaM0, false); break;
    case 4: ok = soa_reduce<4>(Sp, L->soaM0, false); break;
    case 5: ok = soa_reduce<5>(Sp, L->soaM0, false); break;
    default: break;
  }
  if (!ok) L->soaM0.clear();   // D^-1 does not commute with the element mirrors: keep the unfolded sweep
  L->soaM0_gen = L->smoother_gen;
  return 0;
}

template <int N1>
static int soa_occupancy() {
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(soa_apply_kernel<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, soa_smem_bytes<N1>());
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, soa_apply_kernel<N1>, SoaCfg<N1>::NTH,
                                                      soa_smem_bytes<N1>()) != cudaSuccess || occ < 1)
      occ = 1;
    // the segment height follows from the resident warps: more CTAs per SM than the launch bound
    // asks for only shortens the segments (16 warps/SM, J = 15: 38.9 us vs 12 warps/SM, J = 20:
    // 36.7 us at 1024^2, p = 4)
    occ = std::min(occ, SoaCfg<N1>::MINB);
  }
  return occ;
}

int soa_prepare(hdg_level* L) {
  if (L->soa_state == 1) return 0;
  if (L->soa_state == -1 || L->stored || L->blk.empty() || L->n1 > SOA_MAXN1)
    return fail(HDG_EINVAL, "facet-plane layout needs a shared-block (constant coefficient, mirror-symmetric) "
                            "level with p <= 12");
  bool ok = false;
  int occ = 1;
#define SOA_PREP(N) { ok = soa_reduce<N>(L->blk, L->soaM); occ = soa_occupancy<N>(); break; }
  switch (L->n1) {
    case 2: SOA_PREP(2) case 3: SOA_PREP(3) case 4: SOA_PREP(4) case 5: SOA_PREP(5)
    case 6: SOA_PREP(6) case 7: SOA_PREP(7) case 8: SOA_PREP(8) case 9: SOA_PREP(9)
    case 10: SOA_PREP(10) case 11: SOA_PREP(11) case 12: SOA_PREP(12) case 13: SOA_PREP(13)
    default: break;
  }
#undef SOA_PREP
  if (!ok) {
    L->soa_state = -1;
    return fail(HDG_EINVAL, "element block is not invariant under the element mirrors: no facet-plane apply");
  }
  L->soaW = std::max(1, (L->nx - 1 + 30) / 31);       // tile w = columns 31w .. 31w+31 (overlap 1)
  // one wave of CTAs: nss super-segments (CTAs) per tile, each split into 4 stacked warp segments
  const long long resident = (long long)sm_count() * occ;
  long long nss = std::max(1LL, resident / L->soaW);
  nss = std::min(nss, (long long)std::max(1, L->ny / (SoaCfg<2>::WPB * 2)));   // >= 2 rows per warp
  if (const char* e = std::getenv("HDG_SOA_NSS")) nss = std::max(1, std::atoi(e));
  L->soaNss = (int)nss;
  L->soa_state = 1;
  return 0;
}

long long soa_len(const hdg_level* L) {
  return (long long)(L->ny + 1) * L->soaW * (L->n1 * 32 + ((L->n1 * 31 + 3) & ~3) + 2 * ((L->n1 + 3) & ~3));   // SoaCfg<N1>::ENT
}

template <int N1>
static int soa_apply_t(const hdg_level* L, const double* xs, double* ys, cudaStream_t s) {
  SoaArgs<N1> a{};
  a.x = xs; a.y = ys;
  a.nx = L->nx; a.ny = L->ny; a.W = L->soaW; a.nss = L->soaNss;
  std::memcpy(a.M, L->soaM.data(), sizeof(a.M));
  static_assert(SoaCfg<N1>::ENT % 4 == 0, "records are whole 32-byte sectors");
  // programmatic stream serialization: this launch's prologue (barrier init, index setup) may
  // overlap the tail of the kernel before it in the stream; the kernel executes
  // griddepcontrol.wait (full completion + flush of that kernel) before touching x or y
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.W * a.nss));
  cfg.blockDim = dim3(SoaCfg<N1>::NTH);
  cfg.dynamicSmemBytes = soa_smem_bytes<N1>();
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = HDG_SOA_PDL ? 1 : 0;
  cudaLaunchKernelEx(&cfg, soa_apply_kernel<N1>, a);
  CKL();
  return 0;
}

extern "C" {

int hdg_soa_length(hdg_level* L, int64_t* n) {
  if (!L || !n) return fail(HDG_EINVAL, "null argument");
  int rc = soa_prepare(L);
  if (rc) return rc;
  *n = soa_len(L);
  return 0;
}

int hdg_soa_pack(hdg_level* L, const double* x, double* xs, void* stream) {
  if (!L || (!x && L->ndof) || !xs) return fail(HDG_EINVAL, "null argument");
  int rc = soa_prepare(L);
  if (rc) return rc;
  const unsigned grid = (unsigned)(L->soaW * ((L->ny + 1 + soa_pb(L->n1) - 1) / soa_pb(L->n1)));
#define SOA_PACK(N) { soa_pack_blocked_kernel<N><<<grid, 256, 0, S(stream)>>>(x, xs, L->nx, L->ny, L->soaW, L->nh); CKL(); return 0; }
  switch (L->n1) {
    case 2: SOA_PACK(2) case 3: SOA_PACK(3) case 4: SOA_PACK(4) case 5: SOA_PACK(5)
    case 6: SOA_PACK(6) case 7: SOA_PACK(7) case 8: SOA_PACK(8) case 9: SOA_PACK(9)
    case 10: SOA_PACK(10) case 11: SOA_PACK(11) case 12: SOA_PACK(12) case 13: SOA_PACK(13)
    default: return fail(HDG_EINVAL, "facet-plane layout: p <= 12");
  }
#undef SOA_PACK
}

int hdg_soa_unpack(hdg_level* L, const double* xs, double* x, void* stream) {
  if (!L || !xs || (!x && L->ndof)) return fail(HDG_EINVAL, "null argument");
  int rc = soa_prepare(L);
  if (rc) return rc;
  if (L->ndof == 0) return 0;
  const unsigned grid = (unsigned)(L->soaW * ((L->ny + 1 + soa_pb(L->n1) - 1) / soa_pb(L->n1)));
#define SOA_UNPACK(N) { soa_unpack_blocked_kernel<N><<<grid, 256, 0, S(stream)>>>(xs, x, L->nx, L->ny, L->soaW, L->nh); CKL(); return 0; }
  switch (L->n1) {
    case 2: SOA_UNPACK(2) case 3: SOA_UNPACK(3) case 4: SOA_UNPACK(4) case 5: SOA_UNPACK(5)
    case 6: SOA_UNPACK(6) case 7: SOA_UNPACK(7) case 8: SOA_UNPACK(8) case 9: SOA_UNPACK(9)
    case 10: SOA_UNPACK(10) case 11: SOA_UNPACK(11) case 12: SOA_UNPACK(12) case 13: SOA_UNPACK(13)
    default: return fail(HDG_EINVAL, "facet-plane layout: p <= 12");
  }
#undef SOA_UNPACK
}

int hdg_matvec_soa(hdg_level* L, const double* xs, double* ys, void* stream) {
  if (!L || !xs || !ys) return fail(HDG_EINVAL, "null argument");
  if (xs == ys) return fail(HDG_EINVAL, "facet-plane apply cannot run in place");
  int rc = soa_prepare(L);
  if (rc) return rc;
#define SOA_APPLY(N) return soa_apply_t<N>(L, xs, ys, S(stream));
  switch (L->n1) {
    case 2: SOA_APPLY(2) case 3: SOA_APPLY(3) case 4: SOA_APPLY(4) case 5: SOA_APPLY(5)
    case 6: SOA_APPLY(6) case 7: SOA_APPLY(7) case 8: SOA_APPLY(8) case 9: SOA_APPLY(9)
    case 10: SOA_APPLY(10) case 11: SOA_APPLY(11) case 12: SOA_APPLY(12) case 13: SOA_APPLY(13)
    default: return fail(HDG_EINVAL, "facet-plane layout: p <= 12");
  }
#undef SOA_APPLY
}

}  // extern "C"
