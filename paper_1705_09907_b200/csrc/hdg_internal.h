// hdg_internal.h - state shared by the translation units of libhdgb200.so (not part of the C ABI).
#pragma once
#include "hdgb200.h"
#include "hdg_kernels.cuh"
#include "hdg_soa.cuh"

#include <atomic>
#include <map>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

using namespace hdg;

static const int SOA_MAXN1 = 13;        // facet-record apply (hdg_soa.cuh)
static const int SOA_CYCLE_MAXN1 = 13;   // record-layout cycle kernels (hdg_soa_cycle.cuh)

extern std::atomic<long long> g_launches;
int fail(int code, const std::string& msg);   // sets hdg_last_error, returns code

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) return fail(HDG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKL()                                                                             \
  do {                                                                                    \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                   \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess) return fail(HDG_ECUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Launch with programmatic stream serialization: the grid may be scheduled while the kernel before
// it in the stream drains, and runs its prologue up to its `griddepcontrol.wait` (every kernel
// launched this way executes one before its first global access).  The cycle's small levels are
// chains of 5 us kernels, where the launch gap is a large part of the time.  HDG_PDL=0 turns it off.
bool hdg_pdl_enabled();
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = hdg_pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

struct hdg_level {
  int nx = 0, ny = 0, p = 0, n1 = 0, nxp = 0;
  long long nh = 0, n_blocks = 0, ndof = 0;
  bool stored = false;
  std::vector<double> Wh, Wv, Dh, Dv;                // shared mode (host copies -> kernel params)
  std::vector<double> Gh, Gv;                        // shared mode: mirror-reduced stencils (Sym<N1>)
  double *dWh = nullptr, *dWv = nullptr;             // stored mode streams
  double *dDh = nullptr, *dDv = nullptr;
  bool has_bj = false;
  double omega = 0.8;
  // Chebyshev-weighted block-Jacobi steps on [cheb_lo, cheb_hi] of D^-1 A (robust smoother
  // for high-contrast K; same weighting rule as the reference FSAI sweeps, multigrid.py:76-81)
  bool bj_cheb = false;
  double bj_lo = 0.0, bj_hi = 1.0;
  double* partials = nullptr;                        // per-CTA norm partials
  int npart = 0;
  long long op_bytes = 0;
  // FSAI smoother (multigrid.py:47-88): G and G' in CSR on the device
  bool has_fsai = false;
  bool use_fsai = false;   // active smoother of the cycle: the one attached last
  int *g_ptr = nullptr, *g_col = nullptr, *gt_ptr = nullptr, *gt_col = nullptr;
  double *g_val = nullptr, *gt_val = nullptr;
  double lam_max = 1.0, cheb_frac = 0.15, fsai_omega = 1.0;
  // facet-structured FSAI (hdg_fsai.cuh): G rows per facet, no column indices, G' by gathers
  bool fsai_struct = false;
  double *fGh = nullptr, *fGv = nullptr;
  unsigned smoother_gen = 0;     // bumped by every smoother setter: cycle graphs captured before are stale
  double* tail_wd = nullptr;   // fused coarse tail, shared mode: device copy of Wh, Wv, Dh, Dv (n1 = 2)
  // facet-plane (SoA) device layout, shared mode (hdg_soa.cuh): element block + adapted blocks
  std::vector<double> blk;     // the 4n1 x 4n1 element block (shared mode)
  int soa_state = 0;           // 0: not prepared, 1: ready, -1: not available for this level
  std::vector<double> soaM;
  std::vector<double> soaM0;   // class blocks of S D^-1 (general, full rows): the folded zero-start double sweep
  unsigned soaM0_gen = ~0u;    // smoother_gen they were formed at
  int soaW = 0, soaNss = 0;
};

struct hdg_transfer {
  bool is_h = false;
  const hdg_level* fine = nullptr;
  const hdg_level* coarse = nullptr;
  PArgs pa{};
  HArgs ha{};
  double* dcross = nullptr;
};

struct GraphEntry {
  cudaGraphExec_t exec;
  long long nkern;
  unsigned long long last_use;
};
// cycle graphs are keyed by buffer pointers: callers whose addresses vary would otherwise grow the
// cache without bound, so the least recently replayed graph is dropped beyond this many
static const size_t MAX_CYCLE_GRAPHS = 8;

struct hdg_mg {
  std::vector<hdg_level*> L;
  std::vector<hdg_transfer*> T;
  int n = 0;
  std::vector<double*> X, Tm, B, R;
  double* Ainv = nullptr;
  long long nc = 0;
  cudaStream_t cs = nullptr;
  std::map<std::tuple<const void*, const void*, void*, int, int, int>, GraphEntry> graphs;
  int tail_k0 = -1;              // first level of the fused coarse tail (-1: none)
  bool tail_enabled = true;
  bool fuse_first = true;        // first two Jacobi steps from x = 0 in one kernel (shared levels)
  std::vector<unsigned> gens;    // levels' smoother_gen when the cached graphs were captured
  unsigned long long use_clock = 0;
  long long graph_captures = 0;  // graphs instantiated so far (tests: re-capture after a smoother change)
  // record-layout cycle (hdg_soa_cycle.cuh): levels 0 .. rec_m-1 (the constant-coefficient p-ladder of
  // the finest mesh) keep their vectors as facet records
  int rec_mode = 1;              // 0: off, 1: automatic (large levels), 2: whenever the levels qualify
  int rec_m = 0;
  bool rec_fuse_prolong = true;  // p-prolongation inside the first post-smoothing sweep
  bool rec_fold_first = true;    // zero-start double sweep in its folded form (p <= 4)
  bool rec_h_all = false;        // every qualifying h-coarsened level on records, whatever its size (tests)
  std::vector<double*> Xr, Tr, Br;
  double* Rr = nullptr;
};

// facet records (hdg_capi.cu)
int sm_count();
int soa_prepare(hdg_level* L);
long long soa_len(const hdg_level* L);
int soa_prepare_bj0(hdg_level* L);   // soaM0 from the element block and the block-Jacobi inverses (n1 <= 5)

// record-layout cycle pieces (hdg_soa_cycle.cu)
int soa_cyc_sweep(const hdg_level* L, int epi, const double* x, const double* b, double* y, double w, double w0,
                  const double* V, const double* ec, cudaStream_t s);
int soa_cyc_p_prolong(const hdg_level* Lf, const hdg_level* Lc, const double* ec, double* xf, const double* V,
                      cudaStream_t s);
int soa_cyc_h_restrict(const hdg_level* Lf, const HArgs& h, const double* rf, double* rc, cudaStream_t s,
                       const hdg_level* Lc = nullptr);
int soa_cyc_h_prolong(const hdg_level* Lf, const HArgs& h, const double* ec, double* xf, cudaStream_t s,
                      const hdg_level* Lc = nullptr);
int soa_cyc_norm2(const hdg_level* L, const double* r, double* out, double* partials, int nblocks, cudaStream_t s);
int soa_cyc_dot2(const hdg_level* L, const double* a, const double* b, double* out, const double* c, const double* e,
                 double* out2, double* partials, int nblocks, cudaStream_t s);
