// Probe: fp64 DMMA.8x8x4 throughput per SM with W warps per SM sub-partition
// (one CTA of 4 W warps per SM), each warp issuing 16 independent
// accumulator chains with register operands.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048;
  for (int W = 1; W <= 4; ++W) {
    const int threads = 128 * W;
    k<<<p.multiProcessorCount, threads>>>(out, iters);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); k<<<p.multiProcessorCount, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double flop = 2.0 * 8 * 8 * 4 * 16.0 * iters * (threads / 32) * p.multiProcessorCount;
    printf("W=%d warps/SMSP: %.2f TFLOP/s\n", W, flop / best / 1e9);
  }
  return 0;
}
