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
static float run(const SoaArgs<N1>& a0, std::vector<double*>& xs, std::vector<double*>& ys, int reps, int grid) {
  const int smem = soa_smem_bytes<N1>();
  CHECK(cudaFuncSetAttribute(soa_apply_kernel<N1, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid; cfg.blockDim = SoaCfg<N1>::NTH; cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = HDG_SOA_PDL ? 1 : 0;
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
  int nss = argc > 2 ? atoi(argv[2]) : 0;             // CTAs per tile (0: one wave)
  const int reps = argc > 3 ? atoi(argv[3]) : 200;
  const int nx = argc > 4 ? atoi(argv[4]) : n, ny = n;
  const int W = std::max(1, (nx - 1 + 30) / 31);
  int occ = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  CHECK(cudaFuncSetAttribute(soa_apply_kernel<N1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, soa_smem_bytes<N1>()));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, soa_apply_kernel<N1, 1>, SoaCfg<N1>::NTH, soa_smem_bytes<N1>());
  occ = std::min(occ, SoaCfg<N1>::MINB);
  if (nss <= 0) nss = std::max(1, sms * occ / W);
  const long long len = (long long)(ny + 1) * W * SoaCfg<N1>::ENT;
  const long long ndof = (long long)N1 * (2LL * nx * ny - nx - ny);
  int NB = (int)std::ceil(700e6 / (16.0 * ndof));
  if (NB < 2) NB = 2;
  std::vector<double*> xs(NB), ys(NB);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(-1, 1);
  // records: random values in real facet slots, zeros in boundary / pad slots (as packed)
  // records: random facet values laid out as soa_pack_kernel does (zeros in boundary / pad slots)
  std::vector<double> h(len, 0.0);
  {
    using C = SoaCfg<N1>;
    constexpr int ENT = C::ENT, VOFF = C::VOFF, EOFF = C::EOFF, EB = C::EB;
    std::vector<double> hv((size_t)(ny + 1) * nx * N1), vv((size_t)ny * (nx + 1) * N1, 0.0);
    for (int R = 0; R <= ny; ++R)
      for (int c = 0; c < nx; ++c)
        for (int k = 0; k < N1; ++k) hv[((size_t)R * nx + c) * N1 + k] = (R >= 1 && R <= ny - 1) ? U(rng) : 0.0;
    for (int r = 0; r < ny; ++r)
      for (int l = 1; l <= nx - 1; ++l)
        for (int k = 0; k < N1; ++k) vv[((size_t)r * (nx + 1) + l) * N1 + k] = U(rng);
    auto V = [&](int r, int l, int k) { return (r >= 0 && l >= 1 && l <= nx - 1) ? vv[((size_t)r * (nx + 1) + l) * N1 + k] : 0.0; };
    for (int R = 0; R <= ny; ++R)
      for (int w = 0; w < W; ++w) {
        double* rec = h.data() + ((long long)R * W + w) * ENT;
        for (int k = 0; k < N1; ++k) {
          for (int j = 0; j < 32; ++j) rec[k * 32 + j] = 31 * w + j < nx ? hv[((size_t)R * nx + 31 * w + j) * N1 + k] : 0.0;
          for (int j = 0; j < 31; ++j) rec[VOFF + k * 31 + j] = V(R - 1, 31 * w + 1 + j, k);
          rec[EOFF + k] = V(R - 1, 31 * w, k);
          rec[EOFF + EB + k] = V(R - 1, 31 * w + 32, k);
        }
      }
  }
  for (int b = 0; b < NB; ++b) {
    CHECK(cudaMalloc(&xs[b], len * 8));
    CHECK(cudaMalloc(&ys[b], len * 8));
    CHECK(cudaMemcpy(xs[b], h.data(), len * 8, cudaMemcpyHostToDevice));
    CHECK(cudaMemset(ys[b], 0, len * 8));
  }
  SoaArgs<N1> a{};
  a.nx = nx; a.ny = ny; a.W = W; a.nss = nss;
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
  const int nwarps = W * nss;   // CTAs
  std::vector<double> y0(len), y1(len);
  float t0 = run<0>(a, xs, ys, reps, nwarps);
  CHECK(cudaMemcpy(y0.data(), ys[0], len * 8, cudaMemcpyDeviceToHost));
  float t1 = run<1>(a, xs, ys, reps, nwarps);
  CHECK(cudaMemcpy(y1.data(), ys[0], len * 8, cudaMemcpyDeviceToHost));
  double dmax = 0, ymax = 0;
  for (long long t = 0; t < len; ++t) { dmax = std::fmax(dmax, std::fabs(y0[t] - y1[t])); ymax = std::fmax(ymax, std::fabs(y0[t])); }
  const double alg = 16.0 * ndof;
  printf("{\"nx\": %d, \"n\": %d, \"N1\": %d, \"nss\": %d, \"occ\": %d, \"ring\": %d, \"rot\": %d, \"smem_us\": %.2f, \"const_us\": %.2f, "
         "\"smem_frac\": %.3f, \"const_frac\": %.3f, \"rel_diff\": %.2e}\n",
         nx, n, N1, nss, occ, SoaCfg<N1>::RING, NB, t0, t1, alg / (t0 * 1e3) / 6458.7, alg / (t1 * 1e3) / 6458.7, dmax / ymax);
  return 0;
}
