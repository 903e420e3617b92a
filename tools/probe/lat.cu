// Probe: dependent-chain latencies (cycles) of fp64 ops and shuffles on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double seed, double* out, long long* cyc) {
  const int lane = threadIdx.x;
  double a = seed + lane * 1e-3, b = 1.0000001;
  long long t0, t1;
  constexpr int N = 256;
  // DFMA chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) a = fma(a, b, 1e-9);
  t1 = clock64(); cyc[0] = (t1 - t0); out[lane] = a;
  // DMUL chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) a = a * b;
  t1 = clock64(); cyc[1] = (t1 - t0); out[lane] += a;
  // SHFL (64-bit) chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) a = __shfl_sync(0xffffffffu, a, (i + 1) & 31);
  t1 = clock64(); cyc[2] = (t1 - t0); out[lane] += a;
  // SHFL 32-bit chain
  float f = (float)a;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) f = __shfl_sync(0xffffffffu, f, (i + 1) & 31);
  t1 = clock64(); cyc[3] = (t1 - t0); out[lane] += f;
  // rsqrt chain (fp64)
  a = 2.0 + lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = rsqrt(a) + 1.5;
  t1 = clock64(); cyc[4] = (t1 - t0); out[lane] += a;
  // sqrt chain (fp64)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = sqrt(a) + 1.5;
  t1 = clock64(); cyc[5] = (t1 - t0); out[lane] += a;
  // div chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = 3.0 / a + 0.5;
  t1 = clock64(); cyc[6] = (t1 - t0); out[lane] += a;
  // LDS broadcast dependent chain (pointer chase in smem)
  __shared__ double sh[64];
  __shared__ int idx[64];
  sh[lane] = lane; sh[lane + 32] = lane; idx[lane] = (lane + 1) & 31; idx[lane+32] = (lane + 1) & 31;
  __syncwarp();
  int j = lane & 1;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) j = idx[j];
  t1 = clock64(); cyc[7] = (t1 - t0); out[lane] += j;
  // FSEL/select chain on doubles
  a = out[lane];
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) a = (lane > (i & 31)) ? a * b : a;
  t1 = clock64(); cyc[8] = (t1 - t0); out[lane] += a;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 128);
  const char* nm[] = {"dfma", "dmul", "shfl64", "shfl32", "rsqrt+add", "sqrt+add", "div+add", "lds-chase", "sel+dmul"};
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(1.0, o, c);
    long long h[16]; cudaMemcpy(h, c, 128, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 9; ++i) printf("%s %.1f  ", nm[i], h[i] / 256.0);
    printf("\n");
  }
}
