// hdg_setup.cu - hand-written batched kernels for the steps either side of the solve
// (SURVEY section 8(f) ranks 1 and 4): per-element local condensation for element-wise constant
// coefficients (local.py:133-237 restated by the flux-first elimination of
// discretization.PiecewiseCondenser), element-form Galerkin products (multigrid.py:328-334 in the
// form of SURVEY F4), volume reconstruction / postprocessing products (trace.py:171-185,
// local.py:240-299) and the owner sum of the condensed loads (trace.py:67).  All fp64.
#include "hdg_internal.h"

#include <cstring>

namespace {

// ------------------------------------------------------------------------------------------
// H(K) = Stab + kx Lap0 + ky Lap1 (nb x nb, SPD) eliminated without pivoting on the augmented
// matrix [H | B] held in shared memory, one CTA per element; threads (ty, tx): tx walks a row
// (conflict-free), ty the rows below the pivot.  Returns false on a non-positive pivot.
// PK = true keeps only the upper triangle of H (row i: columns j >= i, then B), which is all the
// elimination of a symmetric matrix needs (multiplier l_ik = A_ki / d_k): nb ncol - nb (nb - 1) / 2
// doubles instead of nb ncol, so p = 12 (169 x 221) fits in 227 KB.
template <bool PK>
__device__ __forceinline__ int row_base(int i, int ld, int ncol) {
  return PK ? i * ncol - (i * (i + 1)) / 2 : i * ld;
}

template <bool PK>
__device__ __forceinline__ bool eliminate(double* A, int nb, int ncol, int ld, double* dinv) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, nty = blockDim.x >> 5;
  bool ok = true;
  for (int k = 0; k < nb; ++k) {
    const double* rk = A + row_base<PK>(k, ld, ncol);
    const double d = rk[k];
    if (!(d > 0.0)) ok = false;
    const double inv = 1.0 / d;
    if (threadIdx.x == 0) dinv[k] = inv;
    for (int i = k + 1 + ty; i < nb; i += nty) {
      double* ri = A + row_base<PK>(i, ld, ncol);
      const double l = (PK ? rk[i] : ri[k]) * inv;
      for (int j = (PK ? i : k + 1) + tx; j < ncol; j += 32) ri[j] = fma(-l, rk[j], ri[j]);
    }
    __syncthreads();
  }
  return ok;
}

// S_e = kx A00 + ky A01 + Ms - B^T H^-1 B,  B = Tu - kx G0 - ky G1   (C = -B^T: Fq = Tq^T, Fu = -Tu^T)
template <bool PK>
__global__ void __launch_bounds__(1024) condense_kernel(int nb, int m, long long E, const double* __restrict__ kx,
                                                       const double* __restrict__ ky, const double* __restrict__ stab,
                                                       const double* __restrict__ lap0, const double* __restrict__ lap1,
                                                       const double* __restrict__ tu, const double* __restrict__ g0,
                                                       const double* __restrict__ g1, const double* __restrict__ a00,
                                                       const double* __restrict__ a01, const double* __restrict__ ms,
                                                       double* __restrict__ S, int* __restrict__ status) {
  extern __shared__ __align__(16) double sm[];
  const int ncol = nb + m, ld = ncol | 1;
  double* A = sm;
  double* dinv = sm + (PK ? (size_t)nb * ncol - (size_t)nb * (nb - 1) / 2 : (size_t)nb * ld);
  for (long long e = blockIdx.x; e < E; e += gridDim.x) {
    const double a = kx[e], b = ky[e];
    for (int t = threadIdx.x; t < nb * nb; t += blockDim.x) {
      const int i = t / nb, j = t - i * nb;
      if (!PK || j >= i) A[row_base<PK>(i, ld, ncol) + j] = stab[t] + a * lap0[t] + b * lap1[t];
    }
    for (int t = threadIdx.x; t < nb * m; t += blockDim.x) {
      const int i = t / m, j = t - i * m;
      A[row_base<PK>(i, ld, ncol) + nb + j] = tu[t] - a * g0[t] - b * g1[t];
    }
    __syncthreads();
    if (!eliminate<PK>(A, nb, ncol, ld, dinv) && threadIdx.x == 0) atomicExch(status, 1);
    double* out = S + e * (long long)m * m;
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
      const int r = t / m, c = t - r * m;
      double acc = 0.0;
      for (int k = 0; k < nb; ++k) {
        const double* bk = A + row_base<PK>(k, ld, ncol) + nb;
        acc = fma(bk[r] * dinv[k], bk[c], acc);
      }
      out[t] = a * a00[t] + b * a01[t] + ms[t] - acc;
    }
    __syncthreads();
  }
}

// u_e = H(K_e)^-1 rhs_e in place (rhs: E x nb)
template <bool PK>
__global__ void __launch_bounds__(256) usolve_kernel(int nb, long long E, const double* __restrict__ kx,
                                                     const double* __restrict__ ky, const double* __restrict__ stab,
                                                     const double* __restrict__ lap0, const double* __restrict__ lap1,
                                                     double* __restrict__ rhs, int* __restrict__ status) {
  extern __shared__ __align__(16) double sm[];
  const int ncol = nb + 1, ld = ncol | 1;
  double* A = sm;
  double* dinv = sm + (PK ? (size_t)nb * ncol - (size_t)nb * (nb - 1) / 2 : (size_t)nb * ld);
  for (long long e = blockIdx.x; e < E; e += gridDim.x) {
    const double a = kx[e], b = ky[e];
    for (int t = threadIdx.x; t < nb * nb; t += blockDim.x) {
      const int i = t / nb, j = t - i * nb;
      if (!PK || j >= i) A[row_base<PK>(i, ld, ncol) + j] = stab[t] + a * lap0[t] + b * lap1[t];
    }
    for (int t = threadIdx.x; t < nb; t += blockDim.x) A[row_base<PK>(t, ld, ncol) + nb] = rhs[e * nb + t];
    __syncthreads();
    if (!eliminate<PK>(A, nb, ncol, ld, dinv) && threadIdx.x == 0) atomicExch(status, 1);
    // back substitution on the upper triangle, one warp: u_k = (y_k - sum_{j > k} U_kj u_j) / U_kk
    if (threadIdx.x < 32) {
      for (int k = nb - 1; k >= 0; --k) {
        double* rk = A + row_base<PK>(k, ld, ncol);
        double s = 0.0;
        for (int j = k + 1 + (int)threadIdx.x; j < nb; j += 32) s = fma(rk[j], A[row_base<PK>(j, ld, ncol) + nb], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) rk[nb] = (rk[nb] - s) * dinv[k];
        __syncwarp();
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nb; t += blockDim.x) rhs[e * nb + t] = A[row_base<PK>(t, ld, ncol) + nb];
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// C[e, i] = beta C[e, i] + alpha rs[e] sum_j (A[e, j] cs[j] / ad[e, j]) B[i, j]   (tall-skinny: E rows,
// I, J a few hundred at most).  64 x 64 output tiles, 16-deep panels, 4 x 4 register blocks.
constexpr int GT = 64, GK = 16;

__global__ void __launch_bounds__(256) gemm_nt_kernel(long long E, int I, int J, const double* __restrict__ A, int lda,
                                                      const double* __restrict__ B, double* __restrict__ C, int ldc,
                                                      const double* __restrict__ rs, const double* __restrict__ cs,
                                                      const double* __restrict__ ad, int ldad, double alpha,
                                                      double beta) {
  __shared__ double As[GK][GT + 1], Bs[GK][GT + 1];
  const long long e0 = (long long)blockIdx.x * GT;
  const int i0 = blockIdx.y * GT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  for (int j0 = 0; j0 < J; j0 += GK) {
    for (int t = threadIdx.x; t < GT * GK; t += 256) {
      const int r = t / GK, jj = t - r * GK, j = j0 + jj;
      const long long e = e0 + r;
      double v = 0.0;
      if (e < E && j < J) {
        v = A[e * lda + j];
        if (cs) v *= cs[j];
        if (ad) v /= ad[e * ldad + j];
      }
      As[jj][r] = v;
      const int i = i0 + r;
      Bs[jj][r] = (i < I && j < J) ? B[(long long)i * J + j] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < GK; ++jj) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { av[u] = As[jj][ty + 16 * u]; bv[u] = Bs[jj][tx + 16 * u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const long long e = e0 + ty + 16 * u;
    if (e >= E) continue;
    const double s = alpha * (rs ? rs[e] : 1.0);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = i0 + tx + 16 * v;
      if (i >= I) continue;
      double* c = C + e * ldc + i;
      *c = beta == 0.0 ? s * acc[u][v] : fma(beta, *c, s * acc[u][v]);
    }
  }
}

// out[e, :] = beta out[e, :] + alpha M[cls[e]] in[e, :]   (class-indexed matrices, one warp per element)
__global__ void class_gemv_kernel(long long E, int I, int J, const long long* __restrict__ cls,
                                  const double* __restrict__ M, const double* __restrict__ in, int ldi,
                                  double* __restrict__ out, int ldo, double alpha, double beta) {
  const long long e = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= E) return;
  const double* Me = M + cls[e] * (long long)I * J;
  const double* x = in + e * ldi;
  for (int i = 0; i < I; ++i) {
    double s = 0.0;
    for (int j = lane; j < J; j += 32) s = fma(Me[(long long)i * J + j], x[j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[e * ldo + i] = beta == 0.0 ? alpha * s : fma(beta, out[e * ldo + i], alpha * s);
  }
}

// ------------------------------------------------------------------------------------------
// S_c = Q^T S Q with Q = I_4 (x) V (multigrid.py:328-334 in element form): block (a, b) of S_c is
// V^T S_ab V.  One CTA per element, S and S Q staged in shared memory.
__global__ void __launch_bounds__(128) galerkin_p_kernel(long long E, int n1, int n1c, const double* __restrict__ S,
                                                         const double* __restrict__ V, double* __restrict__ Sc) {
  extern __shared__ __align__(16) double sm[];
  const int m = 4 * n1, mc = 4 * n1c;
  double* Ss = sm;                 // m x m
  double* Ts = Ss + m * m;         // m x mc  (S Q)
  double* Vs = Ts + m * mc;        // n1 x n1c
  for (int t = threadIdx.x; t < n1 * n1c; t += blockDim.x) Vs[t] = V[t];
  for (long long e = blockIdx.x; e < E; e += gridDim.x) {
    const double* Se = S + e * (long long)m * m;
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) Ss[t] = Se[t];
    __syncthreads();
    for (int t = threadIdx.x; t < m * mc; t += blockDim.x) {
      const int r = t / mc, c = t - r * mc, sb = c / n1c, kc = c - sb * n1c;
      double acc = 0.0;
      for (int k = 0; k < n1; ++k) acc = fma(Ss[r * m + sb * n1 + k], Vs[k * n1c + kc], acc);
      Ts[t] = acc;
    }
    __syncthreads();
    double* out = Sc + e * (long long)mc * mc;
    for (int t = threadIdx.x; t < mc * mc; t += blockDim.x) {
      const int r = t / mc, c = t - r * mc, sa = r / n1c, ka = r - sa * n1c;
      double acc = 0.0;
      for (int k = 0; k < n1; ++k) acc = fma(Vs[k * n1c + ka], Ts[(sa * n1 + k) * mc + c], acc);
      out[t] = acc;
    }
    __syncthreads();
  }
}

// S_c = sum_k Q_k^T S_k Q_k over the 4 children (8 x 8 blocks, p = 1).  64 threads per coarse element.
__global__ void __launch_bounds__(64) galerkin_h_kernel(long long C, const double* __restrict__ Sch,
                                                        const double* __restrict__ Q, int shared_q,
                                                        double* __restrict__ Sc) {
  __shared__ double Ss[4][64], Qs[4][64], Ts[4][64];
  const int t = threadIdx.x, r = t >> 3, c = t & 7;
  for (long long e = blockIdx.x; e < C; e += gridDim.x) {
    const double* q = Q + (shared_q ? 0 : e * 256);
    for (int k = 0; k < 4; ++k) { Ss[k][t] = Sch[e * 256 + k * 64 + t]; Qs[k][t] = q[k * 64 + t]; }
    __syncthreads();
    for (int k = 0; k < 4; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = fma(Ss[k][r * 8 + j], Qs[k][j * 8 + c], acc);
      Ts[k][t] = acc;
    }
    __syncthreads();
    double acc = 0.0;
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = fma(Qs[k][i * 8 + r], Ts[k][i * 8 + c], acc);
    Sc[e * 64 + t] = acc;
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// element trace values (E, 4 n1), sides (bottom, right, top, left), 0 on Dirichlet sides (trace.py:81-85)
__global__ void gather_elements_kernel(int nx, int ny, int n1, long long nh, const double* __restrict__ lam,
                                       double* __restrict__ lam_e) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)nx * ny * 4 * n1;
  if (t >= total) return;
  const int k = (int)(t % n1), s = (int)((t / n1) & 3);
  const long long e = t / (4 * n1);
  const int i = (int)(e % nx), j = (int)(e / nx);
  long long blk = -1;
  if (s == 0 && j >= 1) blk = (long long)(j - 1) * nx + i;
  if (s == 2 && j + 1 <= ny - 1) blk = (long long)j * nx + i;
  if (s == 3 && i >= 1) blk = nh + (long long)(i - 1) * ny + j;
  if (s == 1 && i + 1 <= nx - 1) blk = nh + (long long)i * ny + j;
  lam_e[t] = blk >= 0 ? lam[blk * n1 + k] : 0.0;
}

// rhs_f = cl[E1, side1] + cl[E2, side2], slot-0 owner (below / left) first (trace.py:67, 73-79)
__global__ void sum_owners_kernel(int nx, int ny, int n1, long long nh, const double* __restrict__ cl,
                                  double* __restrict__ rhs, long long ndof) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ndof) return;
  const long long blk = t / n1;
  const int k = (int)(t % n1);
  long long e1, e2;
  int s1, s2;
  if (blk < nh) {
    const int j = (int)(blk / nx) + 1, i = (int)(blk % nx);
    e1 = (long long)(j - 1) * nx + i; s1 = 2;      // element below, its TOP side
    e2 = (long long)j * nx + i; s2 = 0;            // element above, its BOTTOM side
  } else {
    const long long u = blk - nh;
    const int i = (int)(u / ny) + 1, j = (int)(u % ny);
    e1 = (long long)j * nx + i - 1; s1 = 1;        // element left, its RIGHT side
    e2 = (long long)j * nx + i; s2 = 3;            // element right, its LEFT side
  }
  const int m = 4 * n1;
  rhs[t] = cl[e1 * m + s1 * n1 + k] + cl[e2 * m + s2 * n1 + k];
}

int grid_for_elements(long long E, int per_sm) {
  const long long g = (long long)sm_count() * per_sm;
  return (int)(E < g ? (E < 1 ? 1 : E) : g);
}

}  // namespace

extern "C" {

int hdg_condense_piecewise(int nb, int m, int64_t E, const double* kx, const double* ky, const double* stab,
                           const double* lap0, const double* lap1, const double* tu, const double* g0,
                           const double* g1, const double* a00, const double* a01, const double* ms, double* S_out,
                           int* status, void* stream) {
  if (nb < 1 || m < 1 || E < 0 || !kx || !ky || !S_out || !status) return fail(HDG_EINVAL, "condense: bad argument");
  if (E == 0) return 0;
  const int ld = (nb + m) | 1;
  size_t smem = sizeof(double) * ((size_t)nb * ld + nb);
  const bool packed = smem > 227 * 1024;                     // p = 12: upper triangle of H only
  if (packed) smem = sizeof(double) * ((size_t)nb * (nb + m) - (size_t)nb * (nb - 1) / 2 + nb);
  if (smem > 227 * 1024) return fail(HDG_EINVAL, "condense: the augmented element matrix exceeds shared memory (p > 12)");
  auto kern = packed ? condense_kernel<true> : condense_kernel<false>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  // one resident CTA per SM (p >= 10) gets 32 warps; with two or more, 8 warps each measured fastest
  // (profiles/condense_threads_r02.txt: p = 8 24.6 / 36.9 / 32.6 ms at 256 / 512 / 1024; p = 11 192 / 124 / 111)
  const int threads = (227 * 1024) / smem >= 2 ? 256 : 1024;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  kern<<<grid_for_elements(E, occ < 1 ? 1 : occ), threads, smem, S(stream)>>>(
      nb, m, E, kx, ky, stab, lap0, lap1, tu, g0, g1, a00, a01, ms, S_out, status);
  CKL();
  return 0;
}

int hdg_piecewise_usolve(int nb, int64_t E, const double* kx, const double* ky, const double* stab,
                         const double* lap0, const double* lap1, double* rhs, int* status, void* stream) {
  if (nb < 1 || E < 0 || !kx || !ky || !rhs || !status) return fail(HDG_EINVAL, "usolve: bad argument");
  if (E == 0) return 0;
  const int ld = (nb + 1) | 1;
  size_t smem = sizeof(double) * ((size_t)nb * ld + nb);
  const bool packed = smem > 227 * 1024;                     // p = 12: upper triangle of H only
  if (packed) smem = sizeof(double) * ((size_t)nb * (nb + 1) - (size_t)nb * (nb - 1) / 2 + nb);
  if (smem > 227 * 1024) return fail(HDG_EINVAL, "usolve: the element matrix exceeds shared memory (p > 15)");
  auto kern = packed ? usolve_kernel<true> : usolve_kernel<false>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
  kern<<<grid_for_elements(E, occ < 1 ? 1 : occ), 256, smem, S(stream)>>>(nb, E, kx, ky, stab, lap0, lap1, rhs, status);
  CKL();
  return 0;
}

int hdg_gemm_nt(int64_t E, int I, int J, const double* A, int lda, const double* B, double* C, int ldc,
                const double* rowscale, const double* colscale, const double* adiv, int ldad, double alpha,
                double beta, void* stream) {
  if (E < 0 || I < 1 || J < 1 || !A || !B || !C) return fail(HDG_EINVAL, "gemm_nt: bad argument");
  if (E == 0) return 0;
  dim3 grid((unsigned)((E + GT - 1) / GT), (unsigned)((I + GT - 1) / GT));
  gemm_nt_kernel<<<grid, 256, 0, S(stream)>>>(E, I, J, A, lda, B, C, ldc, rowscale, colscale, adiv, ldad, alpha,
                                               beta);
  CKL();
  return 0;
}

int hdg_class_gemv(int64_t E, int I, int J, const int64_t* cls, const double* M, const double* in, int ldi,
                   double* out, int ldo, double alpha, double beta, void* stream) {
  if (E < 0 || I < 1 || J < 1 || !cls || !M || !in || !out) return fail(HDG_EINVAL, "class_gemv: bad argument");
  if (E == 0) return 0;
  class_gemv_kernel<<<(unsigned)((E + 3) / 4), 128, 0, S(stream)>>>(E, I, J, (const long long*)cls, M, in, ldi, out,
                                                                     ldo, alpha, beta);
  CKL();
  return 0;
}

int hdg_galerkin_p(int64_t E, int n1, int n1c, const double* S_in, const double* V, double* Sc, void* stream) {
  if (E < 0 || n1 < 2 || n1c < 1 || !S_in || !V || !Sc) return fail(HDG_EINVAL, "galerkin_p: bad argument");
  if (E == 0) return 0;
  const int m = 4 * n1, mc = 4 * n1c;
  const size_t smem = sizeof(double) * ((size_t)m * m + (size_t)m * mc + (size_t)n1 * n1c);
  CK(cudaFuncSetAttribute(galerkin_p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, galerkin_p_kernel, 128, smem);
  galerkin_p_kernel<<<grid_for_elements(E, occ < 1 ? 1 : occ), 128, smem, S(stream)>>>(E, n1, n1c, S_in, V, Sc);
  CKL();
  return 0;
}

int hdg_galerkin_h(int64_t C, const double* S_children, const double* Q, int shared_q, double* Sc, void* stream) {
  if (C < 0 || !S_children || !Q || !Sc) return fail(HDG_EINVAL, "galerkin_h: bad argument");
  if (C == 0) return 0;
  galerkin_h_kernel<<<grid_for_elements(C, 16), 64, 0, S(stream)>>>(C, S_children, Q, shared_q, Sc);
  CKL();
  return 0;
}

int hdg_gather_elements(int nx, int ny, int p, const double* lam, double* lam_e, void* stream) {
  if (nx < 1 || ny < 1 || p < 1 || !lam_e) return fail(HDG_EINVAL, "gather_elements: bad argument");
  const int n1 = p + 1;
  const long long total = (long long)nx * ny * 4 * n1;
  gather_elements_kernel<<<(unsigned)((total + 255) / 256), 256, 0, S(stream)>>>(nx, ny, n1, (long long)nx * (ny - 1),
                                                                                  lam, lam_e);
  CKL();
  return 0;
}

int hdg_sum_owners(int nx, int ny, int p, const double* cl, double* rhs, void* stream) {
  if (nx < 1 || ny < 1 || p < 1 || !cl) return fail(HDG_EINVAL, "sum_owners: bad argument");
  const int n1 = p + 1;
  const long long nh = (long long)nx * (ny - 1), ndof = (nh + (long long)(nx - 1) * ny) * n1;
  if (ndof == 0) return 0;
  if (!rhs) return fail(HDG_EINVAL, "sum_owners: null output");
  sum_owners_kernel<<<(unsigned)((ndof + 255) / 256), 256, 0, S(stream)>>>(nx, ny, n1, nh, cl, rhs, ndof);
  CKL();
  return 0;
}

}  // extern "C"
