// Probe: is the fp64 tensor pipe shared between SMs?  Each CTA (4 warps)
// issues independent DMMA.8x8x4 streams; cycles per CTA vs the number and
// placement (%smid) of co-running CTAs.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__global__ void k(int iters, long long* cyc, int* smid, double* out, int active_mask_mod) {
  int sm; asm("mov.u32 %0, %%smid;" : "=r"(sm));
  double acc[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc[j], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; smid[blockIdx.x] = sm; }
}
int main() {
  long long* cyc; int* smid; double* out;
  cudaMalloc(&cyc, 8 * 1024); cudaMalloc(&smid, 4 * 1024); cudaMalloc(&out, 8 * 1024 * 256);
  const int iters = 2000;
  for (int nb : {1, 2, 3, 4, 8, 16, 74, 148, 296}) {
    k<<<nb, 128>>>(iters, cyc, smid, out, 0);
    cudaDeviceSynchronize();
    long long h[1024]; int s[1024];
    cudaMemcpy(h, cyc, 8 * nb, cudaMemcpyDeviceToHost);
    cudaMemcpy(s, smid, 4 * nb, cudaMemcpyDeviceToHost);
    double mx = 0, mn = 1e30;
    for (int i = 0; i < nb; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
    printf("blocks %3d: cycles/DMMA per warp min %.2f max %.2f  smids:", nb, mn / (iters * 8.0), mx / (iters * 8.0));
    for (int i = 0; i < nb && i < 8; ++i) printf(" %d", s[i]);
    printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
  }
  // 256 threads per CTA (2 warps per SMSP)
  for (int nb : {1, 2, 148}) {
    k<<<nb, 256>>>(iters, cyc, smid, out, 0);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, 8 * nb, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < nb; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("256 thr blocks %3d: cycles/DMMA per warp max %.2f\n", nb, mx / (iters * 8.0));
  }
}
