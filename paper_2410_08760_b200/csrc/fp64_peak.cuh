// fp64_peak.cuh — in-repo fp64 peak microbenchmark (the driver's
// MEASURED_PEAKS.json carries no fp64 figure).  Register-resident loops with
// 8 independent accumulators per thread, 148 x 4 CTAs of 256 threads:
//   DMMA: mma.sync.m8n8k4 f64 (SASS DMMA.8x8x4), 512 flop per warp-instruction
//   DFMA: scalar fma(double)
#pragma once
#include <string>
#include "common.cuh"

namespace fb {

constexpr int PK_ACC = 8;

__global__ void k_peak_dmma(double* out, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[PK_ACC][2];
#pragma unroll
  for (int i = 0; i < PK_ACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < PK_ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < PK_ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_peak_dfma(double* out, int iters, double a, double b) {
  double c[PK_ACC];
#pragma unroll
  for (int i = 0; i < PK_ACC; ++i) c[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < PK_ACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < PK_ACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

inline int fp64_peak_measure(double* dmma_tflops, double* dfma_tflops, std::string* err) {
  int dev = 0;
  cudaDeviceProp p;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
    *err = "no CUDA device";
    return 1;
  }
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) {
    *err = "cudaMalloc failed";
    return 1;
  }
  const int blocks = p.multiProcessorCount * 4, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto best = [&](auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    float b = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < b) b = ms;
    }
    return static_cast<double>(b);
  };
  const double warps = static_cast<double>(blocks) * threads / 32.0;
  const double ms_mma = best([&] { k_peak_dmma<<<blocks, threads>>>(out, iters); });
  const double ms_fma = best([&] { k_peak_dfma<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); });
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 1;
  }
  if (dmma_tflops) *dmma_tflops = warps * iters * PK_ACC * 512.0 / (ms_mma * 1e-3) / 1e12;
  if (dfma_tflops)
    *dfma_tflops = static_cast<double>(blocks) * threads * iters * PK_ACC * 2.0 / (ms_fma * 1e-3) / 1e12;
  return 0;
}

}  // namespace fb
