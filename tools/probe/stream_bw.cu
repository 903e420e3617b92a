// Probe: aggregate HBM streaming bandwidth when each CTA (one per SM, 1024
// threads) reads its own contiguous region (the per-client compressor shape).
// Variants: 8-byte loads, 16-byte loads, TMA bulk ring.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int UNR>
__global__ void __launch_bounds__(1024, 1) k_ld8(const double* __restrict__ D, int64_t w, double* out) {
  const double* v = D + blockIdx.x * w;
  double acc = 0;
  for (int64_t base = 0; base < w; base += UNR * 1024) {
    double x[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t t = base + u * 1024 + threadIdx.x;
      x[u] = t < w ? __ldcs(v + t) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += x[u];
  }
  if (acc == 12345.0) out[0] = acc;
}

template <int UNR>
__global__ void __launch_bounds__(1024, 1) k_ld16(const double* __restrict__ D, int64_t w, double* out) {
  const double2* v = reinterpret_cast<const double2*>(D + blockIdx.x * w);
  const int64_t w2 = w / 2;
  double acc = 0;
  for (int64_t base = 0; base < w2; base += UNR * 1024) {
    double2 x[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t t = base + u * 1024 + threadIdx.x;
      x[u] = t < w2 ? __ldcs(v + t) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += x[u].x + x[u].y;
  }
  if (acc == 12345.0) out[0] = acc;
}

template <int NST, int CH>
__global__ void __launch_bounds__(1024, 1) k_tma(const double* __restrict__ D, int64_t w, double* out) {
  extern __shared__ __align__(16) double ring[];
  __shared__ __align__(8) uint64_t full[NST];
  const double* v = D + blockIdx.x * w;
  const int nch = static_cast<int>((w + CH - 1) / CH);
  auto issue = [&](int i) {
    const int st = i % NST;
    const int64_t rem = w - (int64_t)i * CH; const int nel = (int)(rem < CH ? rem : CH);
    const uint32_t bytes = ((nel + 1) & ~1) * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                 "r"(smem_u32(ring + st * CH)), "l"(v + (int64_t)i * CH), "r"(bytes), "r"(smem_u32(&full[st])) : "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < min(NST, nch); ++i) issue(i);
  }
  __syncthreads();
  double acc = 0;
  for (int i = 0; i < nch; ++i) {
    const int st = i % NST;
    const uint32_t par = (i / NST) & 1;
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(smem_u32(&full[st])), "r"(par) : "memory");
    }
    for (int j = threadIdx.x; j < CH; j += 1024) acc += ring[st * CH + j];
    __syncthreads();
    if (threadIdx.x == 0 && i + NST < nch) issue(i + NST);
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t w = 524800;
  const int nblk = 512;
  double *D, *out;
  cudaMalloc(&D, (size_t)nblk * w * 8 + 64);
  cudaMalloc(&out, 8);
  cudaMemset(D, 0, (size_t)nblk * w * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int r = 0; r < 2; ++r) launch();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-28s %8.3f ms  %7.1f GB/s  (%s)\n", name, ms, nblk * w * 8 / (ms * 1e6),
           cudaGetErrorString(cudaGetLastError()));
  };
  run("ld8 UNR4", [&] { k_ld8<4><<<nblk, 1024>>>(D, w, out); });
  run("ld8 UNR8", [&] { k_ld8<8><<<nblk, 1024>>>(D, w, out); });
  run("ld8 UNR16", [&] { k_ld8<16><<<nblk, 1024>>>(D, w, out); });
  run("ld16 UNR4", [&] { k_ld16<4><<<nblk, 1024>>>(D, w, out); });
  run("ld16 UNR8", [&] { k_ld16<8><<<nblk, 1024>>>(D, w, out); });
  cudaFuncSetAttribute(k_tma<8, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2048 * 8);
  run("tma 8x16KB", [&] { k_tma<8, 2048><<<nblk, 1024, 8 * 2048 * 8>>>(D, w, out); });
  cudaFuncSetAttribute(k_tma<4, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 8192 * 8);
  run("tma 4x64KB", [&] { k_tma<4, 8192><<<nblk, 1024, 4 * 8192 * 8>>>(D, w, out); });
  cudaFuncSetAttribute(k_tma<12, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 2048 * 8);
  run("tma 12x16KB", [&] { k_tma<12, 2048><<<nblk, 1024, 12 * 2048 * 8>>>(D, w, out); });
  // whole-array coalesced reference: grid-stride over everything
  run("ld16 UNR8 (2 CTA/SM, 512t)", [&] { k_ld16<8><<<nblk, 1024>>>(D, w, out); });
  printf("SMs %d\n", sms);
  return 0;
}
