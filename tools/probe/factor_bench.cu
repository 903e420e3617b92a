// Probe: cycles of the warp-level 32x32 Cholesky block factor (the solve's
// per-panel critical section) in isolation: register + shuffle variant
// (as in k_chol_panels) vs a shared-memory variant.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
constexpr int NB = 32, LS = 36;

__global__ void k_shfl(const double* __restrict__ A, double* out, long long* cyc, int reps) {
  __shared__ double P[NB * LS];
  __shared__ double Tb[NB][LS];
  __shared__ double inv[NB];
  const int lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) P[(e / NB) * LS + e % NB] = A[e];
  __syncthreads();
  long long best = 1ll << 60;
  for (int rep = 0; rep < reps; ++rep) {
    if (threadIdx.x < 32) {
      const long long c0 = clock64();
      constexpr int SB = 8;
      double row[NB];
#pragma unroll
      for (int s2 = 0; s2 < NB; ++s2) row[s2] = P[lane * LS + s2];
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) {
        const int qend = (jj / SB + 1) * SB;
        const double piv = __shfl_sync(0xffffffffu, row[jj], jj);
        const bool ok = piv > 0.0 && isfinite(piv);
        const double ir = rsqrt(ok ? piv : 1.0);
        if (lane == jj) inv[jj] = ir;
        row[jj] = (lane == jj) ? piv * ir : ((lane > jj) ? row[jj] * ir : row[jj]);
#pragma unroll
        for (int kk = jj + 1; kk < qend; ++kk) {
          const double lk = __shfl_sync(0xffffffffu, row[jj], kk);
          row[kk] = (lane >= kk) ? fma(-row[jj], lk, row[kk]) : row[kk];
        }
        if (jj == qend - 1 && qend < NB) {
#pragma unroll
          for (int s2 = qend - SB; s2 < qend; ++s2) Tb[lane][s2] = row[s2];
          __syncwarp();
#pragma unroll
          for (int kk = qend; kk < NB; ++kk) {
            double acc = 0.0;
#pragma unroll
            for (int s2 = qend - SB; s2 < qend; ++s2) acc = fma(row[s2], Tb[kk][s2], acc);
            row[kk] = (lane >= kk) ? row[kk] - acc : row[kk];
          }
          __syncwarp();
        }
      }
      const long long c1 = clock64();
      if (c1 - c0 < best) best = c1 - c0;
#pragma unroll
      for (int s2 = 0; s2 < NB; ++s2) out[lane * NB + s2] = row[s2];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[0] = best;
}

// shared-memory variant: lane = row, F row-major stride 33; per pivot the
// column is scaled, then lanes update their row's trailing entries
__global__ void k_smem(const double* __restrict__ A, double* out, long long* cyc, int reps) {
  __shared__ double F[NB][NB + 1];
  __shared__ double S[NB][NB + 1];
  const int lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) S[e / NB][e % NB] = A[e];
  __syncthreads();
  long long best = 1ll << 60;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) F[e / NB][e % NB] = S[e / NB][e % NB];
    __syncthreads();
    if (threadIdx.x < 32) {
      const long long c0 = clock64();
      for (int jj = 0; jj < NB; ++jj) {
        const double piv = F[jj][jj];
        const double ir = rsqrt(piv);
        double lij = 0.0;
        if (lane > jj) { lij = F[lane][jj] * ir; F[lane][jj] = lij; }
        __syncwarp();
        if (lane == jj) F[jj][jj] = piv * ir;
        if (lane > jj)
          for (int kk = jj + 1; kk <= lane; ++kk) F[lane][kk] = fma(-lij, F[kk][jj], F[lane][kk]);
        __syncwarp();
      }
      const long long c1 = clock64();
      if (c1 - c0 < best) best = c1 - c0;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[1] = best;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) out[e] = F[e / NB][e % NB];
}


// chain-optimised register variant: every pivot updates all trailing columns
// immediately; the next pivot's diagonal is updated lane-locally so the
// critical chain per pivot is shfl + rsqrt + mul + fma.  Then the inverse
// T = L^-1 right-looking (lane = column, acc[] registers).
__global__ void k_fast(const double* __restrict__ A, double* out, double* tout, long long* cyc, int reps) {
  __shared__ double P[NB * LS];
  __shared__ double Ls[NB][NB + 1];
  __shared__ double invs[NB];
  const int lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) P[(e / NB) * LS + e % NB] = A[e];
  __syncthreads();
  long long best = 1ll << 60, bestT = 1ll << 60;
  for (int rep = 0; rep < reps; ++rep) {
    if (threadIdx.x < 32) {
      const long long c0 = clock64();
      double row[NB];
#pragma unroll
      for (int s2 = 0; s2 < NB; ++s2) row[s2] = P[lane * LS + s2];
      double dn = row[0];  // lane 0's diagonal
      double myinv = 0.0;
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) {
        const double piv = __shfl_sync(0xffffffffu, dn, jj);
        const double ir = rsqrt(piv);
        const double l = row[jj] * ir;  // L[lane][jj] for lane > jj
        if (lane == jj) myinv = ir;
        if (jj + 1 < NB) dn = fma(-l, l, row[jj + 1]);  // lane jj+1: next diagonal
        row[jj] = (lane == jj) ? piv * ir : ((lane > jj) ? l : row[jj]);
#pragma unroll
        for (int kk = jj + 1; kk < NB; ++kk) {
          const double lk = __shfl_sync(0xffffffffu, l, kk);
          row[kk] = (lane == kk) ? fma(-l, l, row[kk]) : ((lane > kk) ? fma(-l, lk, row[kk]) : row[kk]);
        }
      }
      const long long c1 = clock64();
      // inverse: lane = column c; acc[r] = delta_rc - sum_{k<r} L[r][k] t[k]
#pragma unroll
      for (int s2 = 0; s2 < NB; ++s2) Ls[lane][s2] = (s2 <= lane) ? row[s2] : 0.0;
      invs[lane] = myinv;
      __syncwarp();
      double acc[NB];
#pragma unroll
      for (int r = 0; r < NB; ++r) acc[r] = (r == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const double tk = acc[k] * invs[k];
        acc[k] = tk;
#pragma unroll
        for (int r = k + 1; r < NB; ++r) acc[r] = fma(-Ls[r][k], tk, acc[r]);
      }
      const long long c2 = clock64();
      if (c1 - c0 < best) best = c1 - c0;
      if (c2 - c1 < bestT) bestT = c2 - c1;
#pragma unroll
      for (int s2 = 0; s2 < NB; ++s2) out[lane * NB + s2] = row[s2];
#pragma unroll
      for (int r = 0; r < NB; ++r) tout[r * NB + lane] = acc[r];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { cyc[2] = best; cyc[3] = bestT; }
}

int main() {
  double h[NB * NB];
  for (int i = 0; i < NB; ++i)
    for (int j = 0; j < NB; ++j) h[i * NB + j] = (i == j ? NB + 1.0 : 0.0) + 1.0 / (1 + i + j);
  double *A, *o1, *o2;
  long long* cyc;
  cudaMalloc(&A, sizeof h);
  cudaMalloc(&o1, sizeof h);
  cudaMalloc(&o2, sizeof h);
  cudaMalloc(&cyc, 32);
  double *o3, *t3;
  cudaMalloc(&o3, sizeof h);
  cudaMalloc(&t3, sizeof h);
  cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
  for (int threads : {32, 256}) {
    k_shfl<<<1, threads>>>(A, o1, cyc, 20);
    k_smem<<<1, threads>>>(A, o2, cyc, 20);
    k_fast<<<1, threads>>>(A, o3, t3, cyc, 20);
    long long c[4];
    cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
    double r3[NB * NB], tt[NB * NB];
    cudaMemcpy(r3, o3, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(tt, t3, sizeof h, cudaMemcpyDeviceToHost);
    double r1[NB * NB], r2[NB * NB];
    cudaMemcpy(r1, o1, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(r2, o2, sizeof h, cudaMemcpyDeviceToHost);
    double md = 0;
    for (int i = 0; i < NB; ++i)
      for (int j = 0; j <= i; ++j) md = fmax(md, fabs(r1[i * NB + j] - r2[i * NB + j]));
    double md3 = 0, mi = 0;
    for (int i = 0; i < NB; ++i)
      for (int j = 0; j <= i; ++j) md3 = fmax(md3, fabs(r1[i * NB + j] - r3[i * NB + j]));
    for (int i = 0; i < NB; ++i)  // (L T)[i][j] = delta
      for (int j = 0; j < NB; ++j) {
        double sacc = 0;
        for (int k = 0; k < NB; ++k) sacc += (k <= i ? r3[i * NB + k] : 0.0) * tt[k * NB + j];
        mi = fmax(mi, fabs(sacc - (i == j)));
      }
    printf("threads %d: shfl-variant %lld cycles, smem-variant %lld cycles, max diff %.3e; fast %lld + inverse %lld cycles, diff %.3e, |LT-I| %.3e (%s)\n",
           threads, c[0], c[1], md, c[2], c[3], md3, mi, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
