// Microbenchmark: FP64 DFMA and DMMA (mma.sync m8n8k4 f64) peak on this GPU.
// Used to set the FP64 roofline denominator. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[8];
  for (int i = 0; i < 8; ++i) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int i = 0; i < 8; ++i) r[i] = fma(r[i], a, b);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += r[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 1234.5) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  double* out; cudaMalloc(&out, 8);
  int sms = prop.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int bpsm = 4; bpsm <= 8; bpsm *= 2) {
    dim3 grid(sms * bpsm), block(256);
    dfma_kernel<<<grid, block>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * grid.x * block.x;
    printf("{\"probe\":\"dfma\",\"blocks_per_sm\":%d,\"tflops\":%.2f,\"ms\":%.3f}\n", bpsm, flops / ms / 1e9, ms);
    dmma_kernel<<<grid, block>>>(out, 100);
    cudaEventRecord(e0);
    dmma_kernel<<<grid, block>>>(out, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 4 * 16 * (double)(iters / 4) * grid.x * (block.x / 32);
    printf("{\"probe\":\"dmma_m8n8k4\",\"blocks_per_sm\":%d,\"tflops\":%.2f,\"ms\":%.3f}\n", bpsm, flops / ms / 1e9, ms);
  }
  printf("{\"sms\":%d,\"clock_khz\":%d}\n", sms, prop.clockRate);
  return 0;
}
