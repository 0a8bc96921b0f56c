// Experiment harness for the facet-record apply (hdg_soa.cuh): times kernel variants on the same
// random records (rotating buffers > L2, CUDA events, back to back) and checks that every
// variant writes the same y as the product kernel.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1705_09907_b200/csrc \
//        -o build/soa_lab tools/soa_lab.cu && build/soa_lab n J reps
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <random>

#include "hdg_soa.cuh"

using namespace hdg;

#define CHECK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int N1 = LAB_N1;

template <int MC>
static float run(const SoaArgs<N1>& a0, std::vector<double*>& xs, std::vector<double*>& ys, int reps, int nwarps) {
  const int wpb = SoaCfg<N1>::NTH / 32;
  const int grid = (nwarps + wpb - 1) / wpb;
  const int smem = soa_smem_bytes<N1>();
  CHECK(cudaFuncSetAttribute(soa_apply_kernel<N1, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid; cfg.blockDim = SoaCfg<N1>::NTH; cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = 0;
  const int NB = (int)xs.size();
  SoaArgs<N1> a = a0;
  for (int k = 0; k < 20; ++k) {
    a.x = xs[k % NB]; a.y = ys[k % NB];
    CHECK(cudaLaunchKernelEx(&cfg, soa_apply_kernel<N1, MC>, a));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int k = 0; k < reps; ++k) {
    a.x = xs[k % NB]; a.y = ys[k % NB];
    CHECK(cudaLaunchKernelEx(&cfg, soa_apply_kernel<N1, MC>, a));
  }
  cudaEventRecord(e1);
  CHECK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / reps;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1024;
  int J = argc > 2 ? atoi(argv[2]) : 0;
  const int reps = argc > 3 ? atoi(argv[3]) : 200;
  const int nx = argc > 4 ? atoi(argv[4]) : n, ny = n;
  const int W = (nx + 30) / 31;
  int occ = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  CHECK(cudaFuncSetAttribute(soa_apply_kernel<N1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, soa_smem_bytes<N1>()));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, soa_apply_kernel<N1, 0>, SoaCfg<N1>::NTH, soa_smem_bytes<N1>());
  if (J <= 0) {
    long long resident = (long long)sms * occ * (SoaCfg<N1>::NTH / 32);
    long long nseg = std::max(1LL, resident / W);
    J = (int)((ny + nseg - 1) / nseg);
  }
  const int nseg = (ny + J - 1) / J;
  const long long len = (long long)(ny + 1) * W * SoaCfg<N1>::ENT;
  const long long ndof = (long long)N1 * (2LL * nx * ny - nx - ny);
  int NB = (int)std::ceil(700e6 / (16.0 * ndof));
  if (NB < 2) NB = 2;
  std::vector<double*> xs(NB), ys(NB);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(-1, 1);
  // records: random values in real facet slots, zeros in boundary / pad slots (as packed)
  std::vector<double> h(len, 0.0);
  constexpr int ENT = SoaCfg<N1>::ENT, VOFF = N1 * 32, VW = SoaCfg<N1>::VW;
  for (long long t = 0; t < len; ++t) {
    const long long rw = t / ENT;
    const int o = (int)(t % ENT);
    const int R = (int)(rw / W), w = (int)(rw % W);
    if (o < VOFF) {
      const int col = 31 * w - 1 + o % 32;
      if (R >= 1 && R <= ny - 1 && col >= 0 && col < nx) h[t] = U(rng);
    } else {
      const int j = (o - VOFF) % VW, line = 31 * w - 1 + j, r = R - 1;
      if (j < 33 && r >= 0 && line >= 1 && line <= nx - 1) h[t] = U(rng);
    }
  }
  // duplicated slots must agree with their owners: take them from the owning tile
  for (int R = 0; R <= ny; ++R)
    for (int w = 0; w < W; ++w)
      for (int k = 0; k < N1; ++k) {
        double* rec = h.data() + ((long long)R * W + w) * ENT;
        if (w > 0) rec[k * 32] = h[((long long)R * W + w - 1) * ENT + k * 32 + 31];          // H col 31w-1
        if (w > 0) rec[VOFF + k * VW] = h[((long long)R * W + w - 1) * ENT + VOFF + k * VW + 31];
        if (w + 1 < W) rec[VOFF + k * VW + 32] = h[((long long)R * W + w + 1) * ENT + VOFF + k * VW + 1];
      }
  for (int b = 0; b < NB; ++b) {
    CHECK(cudaMalloc(&xs[b], len * 8));
    CHECK(cudaMalloc(&ys[b], len * 8));
    CHECK(cudaMemcpy(xs[b], h.data(), len * 8, cudaMemcpyHostToDevice));
    CHECK(cudaMemset(ys[b], 0, len * 8));
  }
  SoaArgs<N1> a{};
  a.nx = nx; a.ny = ny; a.W = W; a.J = J; a.nseg = nseg;
  // symmetric class blocks
  {
    using C = SoaCfg<N1>;
    const int sz[4] = {C::A0, C::A1, C::A2, C::A3};
    int mo = 0;
    for (int c = 0; c < 4; ++c) {
      for (int i = 0; i < sz[c]; ++i)
        for (int j = i; j < sz[c]; ++j) {
          const double v = U(rng) + (i == j ? 4.0 : 0.0);
          a.M[mo + i * sz[c] + j] = v;
          a.M[mo + j * sz[c] + i] = v;
        }
      mo += sz[c] * sz[c];
    }
  }
  const int nwarps = W * nseg;
  std::vector<double> y0(len), y1(len);
  float t0 = run<0>(a, xs, ys, reps, nwarps);
  CHECK(cudaMemcpy(y0.data(), ys[0], len * 8, cudaMemcpyDeviceToHost));
  float t1 = run<1>(a, xs, ys, reps, nwarps);
  CHECK(cudaMemcpy(y1.data(), ys[0], len * 8, cudaMemcpyDeviceToHost));
  double dmax = 0, ymax = 0;
  for (long long t = 0; t < len; ++t) { dmax = std::fmax(dmax, std::fabs(y0[t] - y1[t])); ymax = std::fmax(ymax, std::fabs(y0[t])); }
  const double alg = 16.0 * ndof;
  printf("{\"nx\": %d, \"n\": %d, \"N1\": %d, \"J\": %d, \"occ\": %d, \"ring\": %d, \"rot\": %d, \"smem_us\": %.2f, \"const_us\": %.2f, "
         "\"smem_frac\": %.3f, \"const_frac\": %.3f, \"rel_diff\": %.2e}\n",
         nx, n, N1, J, occ, SoaCfg<N1>::RING, NB, t0, t1, alg / (t0 * 1e3) / 6521.4, alg / (t1 * 1e3) / 6521.4, dmax / ymax);
  return 0;
}
