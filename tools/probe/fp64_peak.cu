// Throw-away probe: fp64 peak on B200 via DMMA (mma.sync f64) shapes and DFMA.
#include <cstdio>
#include <cuda_runtime.h>
#define NACC 8
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[NACC];
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fma(acc[i], a, b);
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[NACC][2];
  for (int i = 0; i < NACC; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_m16n8k4(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 0.5, b = 0.999;
  double c[NACC][4];
  for (int i = 0; i < NACC; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_m16n8k8(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 0.5, b0 = 0.999, b1 = 0.3;
  double c[NACC][4];
  for (int i = 0; i < NACC; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%4,%5}, {%6,%7}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0), "d"(b1));
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_m16n8k16(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = 0.5, b0 = 0.999, b1 = 0.3;
  double c[NACC][4];
  for (int i = 0; i < NACC; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%4,%5,%4,%5,%4,%5}, {%6,%7,%6,%7}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0), "d"(b1));
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}
template <typename F>
void bench(const char* name, F launch, double flop_per_launch) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  printf("%-12s %8.3f ms  %8.2f TFLOP/s  %s\n", name, best, flop_per_launch / (best * 1e-3) / 1e12, cudaGetErrorString(err));
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  int sms = p.multiProcessorCount;
  for (int bpsm : {1, 2, 4}) for (int threads : {128, 256, 512}) {
    int blocks = sms * bpsm; int iters = 4096;
    double nw = (double)blocks * threads / 32;
    char nm[64];
    snprintf(nm, 64, "dfma b%d t%d", bpsm, threads);
    bench(nm, [&] { k_dfma<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); }, (double)blocks * threads * iters * NACC * 2);
    snprintf(nm, 64, "m8n8k4 b%d t%d", bpsm, threads);
    bench(nm, [&] { k_m8n8k4<<<blocks, threads>>>(out, iters); }, nw * iters * NACC * 8 * 8 * 4 * 2);
    snprintf(nm, 64, "m16n8k4 b%d t%d", bpsm, threads);
    bench(nm, [&] { k_m16n8k4<<<blocks, threads>>>(out, iters); }, nw * iters * NACC * 16 * 8 * 4 * 2);
    snprintf(nm, 64, "m16n8k8 b%d t%d", bpsm, threads);
    bench(nm, [&] { k_m16n8k8<<<blocks, threads>>>(out, iters); }, nw * iters * NACC * 16 * 8 * 8 * 2);
    snprintf(nm, 64, "m16n8k16 b%d t%d", bpsm, threads);
    bench(nm, [&] { k_m16n8k16<<<blocks, threads>>>(out, iters / 2); }, nw * (iters / 2) * NACC * 16 * 8 * 16 * 2);
  }
  return 0;
}
