// solve_big.cuh — the shifted Cholesky solve (H + shift I) z = rhs for
// d > CH_MAX_D (reference algorithms.py:361-367 option b, linalg.py:133-186),
// where the cluster solvers' panels and vectors no longer fit shared memory.
// Every BASELINE config has d <= 1024; this path lifts the envelope (the
// reference has no limit on d) with plain blocked kernels on the workspace M:
//
//   M ((d+1) x (d+1) doubles, column-major, ld = d + 1): the LOWER triangle
//   A[r][c] = H[c][r] (+ shift on the diagonal) for c <= r < d, and the
//   right-hand side as row d, A[d][c] = rhs[c] — factorising the augmented
//   matrix leaves L below the diagonal and y = L^-1 rhs in row d.
//
// Per BIG_NB-column panel p0 (right-looking):
//   k_big_panel   every CTA factors the diagonal block in shared memory
//                 (identical inputs: identical bits), CTA 0 writes L_pp back
//                 and reports the first pivot <= 0 or not finite
//                 (NotPositiveDefiniteError(index, value), pivots in index
//                 order); then each CTA solves its share of the rows below
//                 (rhs row included) against L_pp: L_ip = A_ip L_pp^-T;
//   k_big_update  the trailing update A[i][j] -= L_ip . L_jp over the lower
//                 triangle of [p1, d] in 64 x 64 tiles (rhs row included: the
//                 forward substitution rides along).
// k_big_back     one CTA: z = L^-T y block by block from the last (the
//                 later blocks' contribution as a matvec, then the block's
//                 triangular solve), then x_out per mode as k_chol_solve.
// The factorisation order differs from the reference's column loop; results
// agree to rounding (parity bar 1e-10).
#pragma once
#include "common.cuh"

namespace fb {

constexpr int BIG_NB = 64;
constexpr int BIG_THREADS = 256;
constexpr int BIG_TILE = 64;
constexpr int BIG_LDS = BIG_NB + 1;  // shared-memory row pitch of a 64-wide block

// A[r][c] (r >= c) from packed H (column-wise upper: H[c][r] at r(r+1)/2 + c)
__global__ void __launch_bounds__(BIG_THREADS) k_big_setup(const DevCtl* __restrict__ ctl, int d,
                                                           const double* __restrict__ hpk,
                                                           const double* __restrict__ shift_ptr,
                                                           const double* __restrict__ rhs,
                                                           double* __restrict__ M) {
  const int64_t ld = d + 1;
  const double shift = shift_ptr ? __ldcg(shift_ptr) : 0.0;
  // column c of A (rows c..d): packed column c of H holds H[0..c][c]; A's
  // column c below the diagonal is H's row c, i.e. packed entries of later
  // columns — read along packed columns instead: thread per (r, c <= r)
  for (int r = blockIdx.x; r <= d; r += gridDim.x) {
    if (r < d) {
      const int64_t pc = static_cast<int64_t>(r) * (r + 1) / 2;  // packed column r: H[0..r][r]
      for (int c = threadIdx.x; c <= r; c += blockDim.x) {
        double v = __ldcg(hpk + pc + c);  // H[c][r] = A[r][c]
        if (c == r) v = __dadd_rn(v, shift);
        M[r + c * ld] = v;
      }
    } else {
      for (int c = threadIdx.x; c < d; c += blockDim.x) M[d + c * ld] = __ldcg(rhs + c);
    }
  }
}

// dynamic smem: the diagonal block, BIG_NB x BIG_LDS doubles
__global__ void __launch_bounds__(BIG_THREADS) k_big_panel(DevCtl* __restrict__ ctl, int d, int p0,
                                                           double* __restrict__ M) {
  extern __shared__ double Ls[];  // Ls[r * BIG_LDS + c], r >= c
  __shared__ int s_fail;
  __shared__ double s_fval;
  if (ctl->halt) return;
  const int64_t ld = d + 1;
  const int pb = min(BIG_NB, d - p0), p1 = p0 + pb;
  const int tid = threadIdx.x;
  for (int e = tid; e < pb * pb; e += BIG_THREADS) {
    const int r = e / pb, c = e % pb;
    Ls[r * BIG_LDS + c] = c <= r ? M[(p0 + r) + static_cast<int64_t>(p0 + c) * ld] : 0.0;
  }
  if (tid == 0) s_fail = -1;
  __syncthreads();
  // right-looking factorisation of the block (column j: pivot, scale, update)
  for (int j = 0; j < pb; ++j) {
    const double piv = Ls[j * BIG_LDS + j];
    if (!(piv > 0.0 && isfinite(piv))) {  // uniform: every thread reads the same pivot
      if (tid == 0) {
        s_fail = j;
        s_fval = piv;
      }
      break;
    }
    const double ljj = sqrt(piv);
    const double inv = 1.0 / ljj;
    __syncthreads();  // every thread has read the pivot
    for (int r = j + 1 + tid; r < pb; r += BIG_THREADS) Ls[r * BIG_LDS + j] *= inv;
    if (tid == 0) Ls[j * BIG_LDS + j] = ljj;
    __syncthreads();
    const int m = pb - j - 1;  // trailing rows / columns j+1 .. pb-1
    for (int e = tid; e < m * m; e += BIG_THREADS) {
      const int r = j + 1 + e / m, c = j + 1 + e % m;
      if (c <= r) Ls[r * BIG_LDS + c] = fma(-Ls[r * BIG_LDS + j], Ls[c * BIG_LDS + j], Ls[r * BIG_LDS + c]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_fail >= 0) {
    if (blockIdx.x == 0 && tid == 0) {
      ctl->pivot_index = p0 + s_fail;
      ctl->pivot_value = s_fval;
      raise_status(ctl, ST_NOT_PD);
    }
    return;
  }
  if (blockIdx.x == 0)
    for (int e = tid; e < pb * pb; e += BIG_THREADS) {
      const int r = e / pb, c = e % pb;
      if (c <= r) M[(p0 + r) + static_cast<int64_t>(p0 + c) * ld] = Ls[r * BIG_LDS + c];
    }
  // rows i in [p1, d] (row d: the right-hand side): x L_pp^T = a, one row
  // per thread, forward substitution over the block's columns
  for (int i = p1 + blockIdx.x * BIG_THREADS + tid; i <= d; i += gridDim.x * BIG_THREADS) {
    double x[BIG_NB];
#pragma unroll
    for (int s = 0; s < BIG_NB; ++s) x[s] = s < pb ? M[i + static_cast<int64_t>(p0 + s) * ld] : 0.0;
#pragma unroll
    for (int s = 0; s < BIG_NB; ++s) {
      if (s < pb) {
        double v = x[s];
#pragma unroll
        for (int t = 0; t < s; ++t) v = fma(-x[t], Ls[s * BIG_LDS + t], v);
        x[s] = v / Ls[s * BIG_LDS + s];
      }
    }
#pragma unroll
    for (int s = 0; s < BIG_NB; ++s)
      if (s < pb) M[i + static_cast<int64_t>(p0 + s) * ld] = x[s];
  }
}

// trailing update of the lower triangle of [p1, d] x [p1, d): tile (ti, tj),
// ti >= tj, of BIG_TILE rows / columns; blockIdx.x enumerates the tiles.
// dynamic smem: the panel rows of both tiles, 2 x BIG_TILE x BIG_LDS doubles
__global__ void __launch_bounds__(BIG_THREADS) k_big_update(const DevCtl* __restrict__ ctl, int d, int p0,
                                                            double* __restrict__ M) {
  extern __shared__ double Ps[];  // Pa[r][s] rows of tile ti, Pb[r][s] rows of tile tj
  if (ctl->halt) return;
  const int64_t ld = d + 1;
  const int pb = min(BIG_NB, d - p0), p1 = p0 + pb;
  const int q = blockIdx.x;
  int ti = static_cast<int>((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
  while ((ti + 1) * (ti + 2) / 2 <= q) ++ti;
  while (ti * (ti + 1) / 2 > q) --ti;
  const int tj = q - ti * (ti + 1) / 2;
  const int r0 = p1 + ti * BIG_TILE, c0 = p1 + tj * BIG_TILE;
  double* Pa = Ps;
  double* Pb = Ps + BIG_TILE * BIG_LDS;
  const int tid = threadIdx.x;
  for (int e = tid; e < BIG_TILE * BIG_NB; e += BIG_THREADS) {
    const int r = e % BIG_TILE, s = e / BIG_TILE;  // coalesced along the rows
    const bool sv = s < pb;
    Pa[r * BIG_LDS + s] = (sv && r0 + r <= d) ? M[(r0 + r) + static_cast<int64_t>(p0 + s) * ld] : 0.0;
    Pb[r * BIG_LDS + s] = (sv && c0 + r < d) ? M[(c0 + r) + static_cast<int64_t>(p0 + s) * ld] : 0.0;
  }
  __syncthreads();
  // thread: rows ty + 16 a, columns tx + 16 b (a, b < 4)
  const int tx = tid & 15, ty = tid >> 4;
  double acc[4][4] = {};
  for (int s = 0; s < pb; ++s) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = Pa[(ty + 16 * a) * BIG_LDS + s];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = Pb[(tx + 16 * b) * BIG_LDS + s];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int j = c0 + tx + 16 * b;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = r0 + ty + 16 * a;
      if (i <= d && j < d && j <= i) {
        double* pm = M + i + static_cast<int64_t>(j) * ld;
        *pm = __dsub_rn(*pm, acc[a][b]);
      }
    }
  }
}

// z = L^-T y (y = row d of M), then the outputs (modes as k_chol_solve).
// one CTA of BIG_BACK_THREADS; dynamic smem: z (d doubles) + a 64-entry block
constexpr int BIG_BACK_THREADS = 1024;
__global__ void __launch_bounds__(BIG_BACK_THREADS) k_big_back(DevCtl* __restrict__ ctl, int d,
                                                               const double* __restrict__ M,
                                                               const double* __restrict__ x,
                                                               double* __restrict__ z,
                                                               double* __restrict__ x_out, int mode,
                                                               int ignore_halt) {
  extern __shared__ double zs[];  // [d] then t[BIG_NB]
  double* tb = zs + d;
  if (ctl->halt) {
    if (threadIdx.x == 0) tl_mark(2, true);
    return;
  }
  const int64_t ld = d + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = BIG_BACK_THREADS / 32;
  for (int i = tid; i < d; i += BIG_BACK_THREADS) zs[i] = M[d + static_cast<int64_t>(i) * ld];  // y
  __syncthreads();
  const int nblk = (d + BIG_NB - 1) / BIG_NB;
  for (int kb = nblk - 1; kb >= 0; --kb) {
    const int b0 = kb * BIG_NB, bn = min(BIG_NB, d - b0), b1 = b0 + bn;
    // t_c = y_c - sum_{k >= b1} L[k][c] z_k for the block's columns c: warp
    // per column, lanes over k (column c of M is contiguous in k)
    for (int cc = warp; cc < bn; cc += NW) {
      const int c = b0 + cc;
      const double* col = M + static_cast<int64_t>(c) * ld;
      double s = 0.0;
      for (int k = b1 + lane; k < d; k += 32) s = fma(col[k], zs[k], s);
      s = warp_sum(s);
      if (lane == 0) tb[cc] = zs[c] - s;
    }
    __syncthreads();
    // L_bb^T z_b = t: warp 0, lane = row, from the last row up
    if (warp == 0) {
      double zi0 = lane < bn ? tb[lane] : 0.0;
      double zi1 = lane + 32 < bn ? tb[lane + 32] : 0.0;
      for (int s2 = bn - 1; s2 >= 0; --s2) {
        const bool own0 = lane == s2, own1 = lane + 32 == s2;
        const double diag = M[(b0 + s2) + static_cast<int64_t>(b0 + s2) * ld];
        if (own0) zi0 /= diag;
        if (own1) zi1 /= diag;
        const double zs2 = __shfl_sync(0xffffffffu, s2 < 32 ? zi0 : zi1, s2 & 31);
        // rows r < s2: t_r -= L[s2][r] z_s2
        if (lane < s2) zi0 = fma(-M[(b0 + s2) + static_cast<int64_t>(b0 + lane) * ld], zs2, zi0);
        if (lane + 32 < s2) zi1 = fma(-M[(b0 + s2) + static_cast<int64_t>(b0 + lane + 32) * ld], zs2, zi1);
      }
      if (lane < bn) zs[b0 + lane] = zi0;
      if (lane + 32 < bn) zs[b0 + lane + 32] = zi1;
    }
    __syncthreads();
  }
  if (tid == 0) tl_mark(2, true);
  if (!ignore_halt && ctl->halt) return;
  for (int i = tid; i < d; i += BIG_BACK_THREADS) {
    const double zi = zs[i];
    z[i] = zi;
    if (mode == 0) x_out[i] = __dsub_rn(__ldcg(x + i), zi);
    else if (mode == 1) x_out[i] = zi;
  }
}

}  // namespace fb
