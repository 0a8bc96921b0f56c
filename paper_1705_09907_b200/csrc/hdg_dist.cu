// hdg_dist.cu - multi-GPU element-row strips behind the C ABI (SURVEY section 8(b) hdg_dist_init,
// 8(e)): halo exchange of a strip's ghost facet rows and the owned-dof reduction over a caller's
// NCCL communicator, all enqueued on the caller's stream (no host wait).  The reference has no
// distributed code; the data path is trace.py:87-94 applied to a window of the mesh, and what
// crosses a strip boundary is the facet rows the window's stencils read (distributed.py:
// StripLayout is the host-side statement of the same row lists).
//
// NCCL is resolved at run time (dlopen of the libnccl the process already uses), so the library
// loads - and the CPU-only tests run - on machines without NCCL.
#include "hdg_internal.h"

#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);   // the copy already in the process
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
  api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
  api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
  api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.ok = api.GroupStart && api.GroupEnd && api.Send && api.Recv && api.AllReduce && api.GetErrorString;
  return api;
}

// up to three facet rows of a window, concatenated in this order in the message
struct HaloRows {
  int n;
  int is_h[3];
  int jl[3];        // window row (h: line jl, 1 <= jl <= nyl-1; v: element row jl)
  int off[4];       // offsets of the rows in the message (doubles)
};

// message <-> window vector; to_msg = 1 packs, 0 unpacks
__global__ void halo_copy_kernel(double* __restrict__ x, double* __restrict__ msg, int nx, int nyl, int n1,
                                 long long nh, const HaloRows r, int to_msg) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= r.off[r.n]) return;
  int q = 0;
  while (q + 1 < r.n && t >= r.off[q + 1]) ++q;
  const int u = t - r.off[q], i = u / n1, k = u - i * n1;
  const long long dof = r.is_h[q] ? ((long long)(r.jl[q] - 1) * nx + i) * n1 + k
                                  : (nh + (long long)i * nyl + r.jl[q]) * n1 + k;
  if (to_msg) msg[t] = x[dof];
  else x[dof] = msg[t];
}

}  // namespace

struct hdg_dist {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  double* buf[4] = {nullptr, nullptr, nullptr, nullptr};   // send down, recv down, send up, recv up
  size_t cap = 0;                                          // doubles per buffer
};

static int ensure(hdg_dist* d, size_t n) {
  if (n <= d->cap) return 0;
  for (double*& b : d->buf) { cudaFree(b); b = nullptr; }
  for (double*& b : d->buf) CK(cudaMalloc(&b, sizeof(double) * n));
  d->cap = n;
  return 0;
}

// rows of the window in message order; h rows on the global Dirichlet lines 0 / ny are not dofs
static HaloRows rows_of(const int* j_global, const int* is_h, int n, int lo, int nx, int n1, int ny_global) {
  HaloRows r{};
  int off = 0;
  for (int q = 0; q < n; ++q) {
    if (is_h[q] && (j_global[q] < 1 || j_global[q] > ny_global - 1)) continue;
    r.is_h[r.n] = is_h[q];
    r.jl[r.n] = j_global[q] - lo;
    r.off[r.n] = off;
    off += (is_h[q] ? nx : nx - 1) * n1;
    ++r.n;
  }
  r.off[r.n] = off;
  return r;
}

extern "C" {

int hdg_dist_init(void* nccl_comm, int rank, int nranks, hdg_dist** out) {
  if (!nccl_comm || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(HDG_EINVAL, "dist_init: bad argument");
  if (!nccl().ok) return fail(HDG_ESTATE, "dist_init: libnccl.so.2 not found in this process");
  hdg_dist* d = new hdg_dist();
  d->comm = (ncclComm_t)nccl_comm;
  d->rank = rank;
  d->nranks = nranks;
  *out = d;
  return 0;
}

int hdg_dist_destroy(hdg_dist* d) {
  if (!d) return 0;
  for (double* b : d->buf) cudaFree(b);
  delete d;
  return 0;
}

int hdg_dist_halo(hdg_dist* d, const hdg_level* win, int lo, int r0, int r1, int ny_global, int kind, double* x,
                  void* stream) {
  if (!d || !win || !x) return fail(HDG_EINVAL, "dist_halo: null argument");
  const bool loopback = (kind & 0x100) != 0;   // self-test: this rank is its own lower and upper neighbour
  kind &= 0xff;
  if (kind != 0 && kind != 1) return fail(HDG_EINVAL, "dist_halo: kind must be 0 (operator) or 1 (residual)");
  const int nx = win->nx, nyl = win->ny, n1 = win->n1;
  if (lo > r0 || r1 > lo + nyl || r0 >= r1) return fail(HDG_EINVAL, "dist_halo: owned rows outside the window");
  const bool down = loopback || d->rank > 0, up = loopback || d->rank < d->nranks - 1;
  const int pd = loopback ? d->rank : d->rank - 1, pu = loopback ? d->rank : d->rank + 1;
  const int H = 1, V = 0;
  HaloRows sd{}, rd{}, su{}, ru{};
  if (kind == 0) {
    // operator halo: the neighbour below needs my h(r0); I need its h(r0-1), v(r0-1); symmetric above
    if (down) {
      const int js[1] = {r0}, ks[1] = {H};
      sd = rows_of(js, ks, 1, lo, nx, n1, ny_global);
      const int jr[2] = {r0 - 1, r0 - 1}, kr[2] = {H, V};
      rd = rows_of(jr, kr, 2, lo, nx, n1, ny_global);
    }
    if (up) {
      const int js[2] = {r1 - 1, r1 - 1}, ks[2] = {H, V};
      su = rows_of(js, ks, 2, lo, nx, n1, ny_global);
      const int jr[1] = {r1}, kr[1] = {H};
      ru = rows_of(jr, kr, 1, lo, nx, n1, ny_global);
    }
  } else {
    // residual halo before an h-restriction: the strip above needs v(r1-2), v(r1-1), h(r1-1)
    if (up) {
      const int js[3] = {r1 - 2, r1 - 1, r1 - 1}, ks[3] = {V, V, H};
      su = rows_of(js, ks, 3, lo, nx, n1, ny_global);
    }
    if (down) {
      const int jr[3] = {r0 - 2, r0 - 1, r0 - 1}, kr[3] = {V, V, H};
      rd = rows_of(jr, kr, 3, lo, nx, n1, ny_global);
    }
  }
  for (const HaloRows* r : {&sd, &rd, &su, &ru})
    for (int q = 0; q < r->n; ++q) {
      const int jl = r->jl[q];
      if (r->is_h[q] ? (jl < 1 || jl > nyl - 1) : (jl < 0 || jl >= nyl))
        return fail(HDG_EINVAL, "dist_halo: the window lacks a ghost row this exchange touches");
    }
  const size_t need = (size_t)3 * nx * n1;
  int rc = ensure(d, need);
  if (rc) return rc;
  cudaStream_t s = S(stream);
  const long long nh = win->nh;
  auto copy = [&](const HaloRows& r, double* msg, int to_msg) {
    const int n = r.off[r.n];
    if (n > 0) halo_copy_kernel<<<(n + 255) / 256, 256, 0, s>>>(x, msg, nx, nyl, n1, nh, r, to_msg);
  };
  copy(sd, d->buf[0], 1);
  copy(su, d->buf[2], 1);
  NcclApi& N = nccl();
  ncclResult_t e = N.GroupStart();
  auto post = [&](bool send, const HaloRows& r, double* msg, int peer) {
    const size_t n = (size_t)r.off[r.n];
    if (n == 0 || e != ncclSuccess) return;
    e = send ? N.Send(msg, n, ncclDouble, peer, d->comm, s) : N.Recv(msg, n, ncclDouble, peer, d->comm, s);
  };
  // sends first, then the receives in the order that pairs them when both neighbours are this rank
  // (loopback self-test: my send-down meets my receive-from-above); with distinct peers the order
  // within the group does not matter
  post(true, sd, d->buf[0], pd);
  post(true, su, d->buf[2], pu);
  post(false, ru, d->buf[3], pu);
  post(false, rd, d->buf[1], pd);
  const ncclResult_t e2 = N.GroupEnd();
  if (e != ncclSuccess || e2 != ncclSuccess)
    return fail(HDG_ECUDA, std::string("nccl: ") + N.GetErrorString(e != ncclSuccess ? e : e2));
  copy(rd, d->buf[1], 0);
  copy(ru, d->buf[3], 0);
  CKL();
  return 0;
}

int hdg_dist_allreduce_sum(hdg_dist* d, double* v, int count, void* stream) {
  if (!d || !v || count < 1) return fail(HDG_EINVAL, "dist_allreduce: bad argument");
  NcclApi& N = nccl();
  const ncclResult_t e = N.AllReduce(v, v, (size_t)count, ncclDouble, ncclSum, d->comm, S(stream));
  if (e != ncclSuccess) return fail(HDG_ECUDA, std::string("nccl: ") + N.GetErrorString(e));
  return 0;
}

}  // extern "C"
