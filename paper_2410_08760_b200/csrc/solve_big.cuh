// solve_big.cuh — the shifted Cholesky solve (H + shift I) z = rhs for
// d > CP_MAX_D (reference algorithms.py:361-367 option b, linalg.py:133-186),
// where the panel-owning cluster solver's panels no longer fit shared memory
// (c4: d = 1024; the reference has no limit on d).  A right-looking blocked
// factorisation over global memory (the matrix lives in L2), ONE kernel per
// 32-column panel:
//
//   M ((d+1) x (d+1) doubles, column-major, ld = d + 1): the LOWER triangle
//   A[r][c] = H[c][r] (+ shift on the diagonal) for c <= r < d, and the
//   right-hand side as row d, A[d][c] = rhs[c] — factorising the augmented
//   matrix leaves y = L^-1 rhs in row d of L.
//   L (same shape, a second buffer): the factor below the diagonal blocks.
//   Tg[p] (32 x 32): T_p = L_pp^-1, the inverse of panel p's diagonal block.
//
// k_big_panel(p): one CTA per 64 x 64 tile (ti >= tj) of the trailing matrix
//   [p1, d] x [p1, d).  Every CTA factors the panel's 32 x 32 diagonal block
//   itself (identical inputs: identical bits; warp 0 the block factor with
//   lane c owning column c of the symmetric Schur complement, warp 1 the
//   inverse T one pivot behind it — the scheme of k_chol_panels), forms the
//   panel rows of BOTH its tiles, X = A_ip T^T (a 64 x 32 x 32 product:
//   cheaper than waiting for another CTA's), and applies
//   C_ij -= X_i X_j^T to its tile.  The CTAs of the diagonal tiles write their
//   X rows to L (a second buffer: other CTAs still read A's panel columns),
//   CTA 0 writes T_p.  No cross-CTA dependency inside a kernel; the next
//   panel's kernel follows in stream order.  The first pivot <= 0 or not
//   finite raises NotPositiveDefiniteError(index, value) (pivots in index
//   order).
// k_big_back: one CTA: z_b = T_b^T (y_b - sum_{k >= b1} L[k][b] z_k) block by
//   block from the last (a warp per column for the sum, then a 32 x 32
//   product), then x_out per mode as k_chol_solve.
// The factorisation order differs from the reference's column loop; results
// agree to rounding (parity bar 1e-10).
#pragma once
#include "common.cuh"

namespace fb {

constexpr int BIG_NB = 32;
constexpr int BIG_THREADS = 256;
constexpr int BIG_TILE = 64;
constexpr int BIG_LDS = BIG_NB + 1;  // shared-memory row pitch of a 32-wide block

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


struct BigSmem {
  double S[BIG_NB][BIG_LDS];     // the diagonal block (symmetric), then unused
  double R[BIG_NB][BIG_LDS];     // row j of the Schur complement at pivot j
  double T[BIG_NB][BIG_LDS];     // L_pp^-1 (lower triangular)
  double A[2][BIG_TILE][BIG_LDS];  // panel rows of tile ti / tj as loaded
  double X[2][BIG_TILE][BIG_LDS];  // A T^T
  double inv[BIG_NB];
  uint64_t barF[BIG_NB];
  int failed;
};

__global__ void __launch_bounds__(BIG_THREADS) k_big_panel(DevCtl* __restrict__ ctl, int d, int p0,
                                                           double* __restrict__ M,
                                                           double* __restrict__ L,
                                                           double* __restrict__ Tg) {
  extern __shared__ __align__(16) uint8_t big_raw[];
  BigSmem& sm = *reinterpret_cast<BigSmem*>(big_raw);
  const int64_t ld = d + 1;
  const int pb = min(BIG_NB, d - p0), p1 = p0 + pb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.x;
  int ti = static_cast<int>((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
  while ((ti + 1) * (ti + 2) / 2 <= q) ++ti;
  while (ti * (ti + 1) / 2 > q) --ti;
  const int tj = q - ti * (ti + 1) / 2;
  const int r0 = p1 + ti * BIG_TILE, c0 = p1 + tj * BIG_TILE;
  if (tid < BIG_NB) mbar_init(&sm.barF[tid], 1);
  if (tid == 0) {
    sm.failed = 0;
    fence_barrier_init();
  }
  // programmatic dependent launch: this prologue overlapped the previous
  // panel's kernel; the next panel's kernel may launch once every CTA of
  // this one is past the wait (so at most two panel kernels hold SM slots)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (ctl->halt) return;
  // diagnostics: CTA 0's phase stamps of panel p in g_dbg_span[8 p ..]
  const bool stamp_on = g_dbg_on && q == 0 && tid == 0 && p0 / BIG_NB < 128;
  auto stamp = [&](int ph) {
    if (stamp_on) g_dbg_span[8 * (p0 / BIG_NB) + ph] = globaltimer_ns();
  };
  stamp(0);
  // every global load of the CTA is issued here, before any is consumed: the
  // diagonal block (lower triangle, mirrored in shared memory; the identity
  // past pb), the panel rows of both tiles (coalesced along the rows), and
  // the trailing tile itself (kept in registers until the update: its
  // latency hides behind the block factor)
  const int tr = tid & 15, tc = tid >> 4;
  double sv[4], av[2][8], cv[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = tid + u * BIG_THREADS, r = e & (BIG_NB - 1), c = e >> 5;
    sv[u] = (c <= r && r < pb) ? __ldcg(M + (p0 + r) + static_cast<int64_t>(p0 + c) * ld) : (r == c ? 1.0 : 0.0);
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = tid + u * BIG_THREADS, r = e & (BIG_TILE - 1), s2 = e >> 6;
    const bool ok = s2 < pb;
    av[0][u] = (ok && r0 + r <= d) ? __ldcg(M + (r0 + r) + static_cast<int64_t>(p0 + s2) * ld) : 0.0;
    av[1][u] = (ok && ti != tj && c0 + r <= d) ? __ldcg(M + (c0 + r) + static_cast<int64_t>(p0 + s2) * ld) : 0.0;
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int j = c0 + tc + 16 * b;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = r0 + tr + 16 * a;
      cv[a][b] = (i <= d && j < d && j <= i) ? __ldcg(M + i + static_cast<int64_t>(j) * ld) : 0.0;
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = tid + u * BIG_THREADS, r = e & (BIG_NB - 1), c = e >> 5;
    if (c <= r) {
      sm.S[r][c] = sv[u];
      sm.S[c][r] = sv[u];
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = tid + u * BIG_THREADS, r = e & (BIG_TILE - 1), s2 = e >> 6;
    sm.A[0][r][s2] = av[0][u];
    if (ti != tj) sm.A[1][r][s2] = av[1][u];
  }
  __syncthreads();
  stamp(1);
  if (warp == 0) {
    // block factor on the symmetric Schur complement: lane c owns column c
    // (a[r] = S[r][c]); by symmetry its multiplier S[c][j] is its own a[j],
    // so per pivot only 1/sqrt(S[j][j]) crosses lanes
    double a[BIG_NB];
#pragma unroll
    for (int r = 0; r < BIG_NB; ++r) a[r] = sm.S[r][lane];
    double myir = 0.0, mypiv = 0.0;
    sm.R[0][lane] = a[0];
    {
      const double y = rsqrt_nr(a[0]);
      if (lane == 0) { sm.inv[0] = y; mypiv = a[0]; }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.barF[0]);
    double ir = sm.inv[0];
#pragma unroll
    for (int j = 0; j < BIG_NB; ++j) {
      const double* b = &sm.R[j][0];
      myir = (lane == j) ? ir : myir;
      const double ir2 = ir * ir;
      const double m = (lane > j) ? a[j] * ir2 : 0.0;  // columns < j are final
      if (j + 1 < BIG_NB) {
        a[j + 1] = fma(-m, b[j + 1], a[j + 1]);
        sm.R[j + 1][lane] = a[j + 1];
        const double y = rsqrt_nr(a[j + 1]);
        mypiv = (lane == j + 1) ? a[j + 1] : mypiv;
        if (lane == j + 1) sm.inv[j + 1] = y;
      }
#pragma unroll
      for (int r = j + 2; r < BIG_NB; ++r) a[r] = fma(-m, b[r], a[r]);
      __syncwarp();
      if (j + 1 < BIG_NB) {
        if (lane == 0) mbar_arrive(&sm.barF[j + 1]);
        ir = sm.inv[j + 1];
      }
    }
    // first pivot (in index order) that is <= 0 or not finite
    const unsigned bad = __ballot_sync(0xffffffffu, lane < pb && !(mypiv > 0.0 && isfinite(mypiv)));
    if (bad) {
      const int fail = __ffs(bad) - 1;
      const double fv = __shfl_sync(0xffffffffu, mypiv, fail);
      if (lane == 0) {
        sm.failed = 1;
        if (q == 0) {
          ctl->pivot_index = p0 + fail;
          ctl->pivot_value = fv;
          raise_status(ctl, ST_NOT_PD);
        }
      }
    }
  } else if (warp == 1) {
    // T = L^-1, right-looking, lane c owning column c, one pivot behind
    // warp 0: t_j = t[j] / L_jj, t[r] -= L[r][j] t_j with L[r][j] = R_j[r] ir_j
    double t[BIG_NB];
#pragma unroll
    for (int r = 0; r < BIG_NB; ++r) t[r] = (r == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int j = 0; j < BIG_NB; ++j) {
      mbar_wait(&sm.barF[j], 0);
      const double irj = sm.inv[j];
      const double u = t[j] * irj * irj;
      t[j] *= irj;
#pragma unroll
      for (int r = j + 1; r < BIG_NB; ++r) t[r] = fma(-u, sm.R[j][r], t[r]);
    }
#pragma unroll
    for (int r = 0; r < BIG_NB; ++r) sm.T[r][lane] = t[r];
  }
  __syncthreads();
  stamp(2);
  if (sm.failed) return;
  if (q == 0)
    for (int e = tid; e < BIG_NB * BIG_NB; e += BIG_THREADS)
      Tg[static_cast<int64_t>(p0 / BIG_NB) * BIG_NB * BIG_NB + e] = sm.T[e >> 5][e & 31];
  // X = A T^T: thread (row r, 8 columns); T's upper triangle is zero
  {
    const int r = tid & (BIG_TILE - 1), s0 = (tid >> 6) * 8;
    for (int h = 0; h < (ti != tj ? 2 : 1); ++h) {
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = 0.0;
#pragma unroll 8
      for (int t = 0; t < BIG_NB; ++t) {
        const double av = sm.A[h][r][t];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = fma(av, sm.T[s0 + u][t], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) sm.X[h][r][s0 + u] = acc[u];
    }
  }
  __syncthreads();
  stamp(3);
  const int hb = ti != tj ? 1 : 0;
  if (ti == tj)  // this tile's rows of L_p (row d: y)
    for (int e = tid; e < BIG_TILE * BIG_NB; e += BIG_THREADS) {
      const int r = e & (BIG_TILE - 1), s = e >> 6;
      if (s < pb && r0 + r <= d) L[(r0 + r) + static_cast<int64_t>(p0 + s) * ld] = sm.X[0][r][s];
    }
  // C[i][j] -= X_i . X_j: thread rows tr + 16 a (contiguous in memory), columns tc + 16 b
  double acc[4][4] = {};
#pragma unroll 4
  for (int s = 0; s < BIG_NB; ++s) {
    double xa[4], xb[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) xa[a] = sm.X[0][tr + 16 * a][s];
#pragma unroll
    for (int b = 0; b < 4; ++b) xb[b] = sm.X[hb][tc + 16 * b][s];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(xa[a], xb[b], acc[a][b]);
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int j = c0 + tc + 16 * b;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = r0 + tr + 16 * a;
      if (i <= d && j < d && j <= i) M[i + static_cast<int64_t>(j) * ld] = __dsub_rn(cv[a][b], acc[a][b]);
    }
  }
  stamp(4);
}

// z = L^-T y (y = row d of L), then the outputs (modes as k_chol_solve).
// one CTA of BIG_BACK_THREADS (a warp per column of a block);
// dynamic smem: z (d doubles, padded) + t[32] + T_b[32][33]
constexpr int BIG_BACK_THREADS = 1024;
__host__ __device__ constexpr size_t big_back_smem(int d) {
  return (static_cast<size_t>(d) + BIG_NB + BIG_NB + BIG_NB * BIG_LDS) * sizeof(double);
}
__global__ void __launch_bounds__(BIG_BACK_THREADS) k_big_back(DevCtl* __restrict__ ctl, int d,
                                                               const double* __restrict__ L,
                                                               const double* __restrict__ Tg,
                                                               const double* __restrict__ x,
                                                               double* __restrict__ z,
                                                               double* __restrict__ x_out, int mode,
                                                               int ignore_halt) {
  extern __shared__ double zs[];  // [d rounded up to 32] then t[32] then Tb[32][33]
  const int dp = (d + BIG_NB - 1) / BIG_NB * BIG_NB;
  double* tb = zs + dp;
  double* Tb = tb + BIG_NB;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (ctl->halt) {
    if (threadIdx.x == 0) tl_mark(2, true);
    return;
  }
  const int64_t ld = d + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < dp; i += BIG_BACK_THREADS) zs[i] = i < d ? __ldcg(L + d + static_cast<int64_t>(i) * ld) : 0.0;  // y
  __syncthreads();
  const int nblk = (d + BIG_NB - 1) / BIG_NB;
  for (int kb = nblk - 1; kb >= 0; --kb) {
    const int b0 = kb * BIG_NB, bn = min(BIG_NB, d - b0), b1 = b0 + bn;
    Tb[warp * BIG_LDS + lane] = __ldcg(Tg + static_cast<int64_t>(kb) * BIG_NB * BIG_NB + warp * BIG_NB + lane);
    // t_c = y_c - sum_{k >= b1} L[k][c] z_k: warp per column, lanes over k
    // (column c of L is contiguous in k), eight loads in flight
    {
      const int c = b0 + warp;
      double s = 0.0;
      if (warp < bn) {
        const double* col = L + static_cast<int64_t>(c) * ld;
        for (int k0 = b1; k0 < d; k0 += 256) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = k0 + u * 32 + lane;
            v[u] = k < d ? __ldcg(col + k) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = k0 + u * 32 + lane;
            s = fma(v[u], zs[k < d ? k : b1], s);
          }
        }
        s = warp_sum(s);
      }
      if (lane == 0) tb[warp] = warp < bn ? zs[c] - s : 0.0;
    }
    __syncthreads();
    // z_b = T_b^T t: z_r = sum_{s >= r} T[s][r] t_s
    if (warp == 0) {
      double zr = 0.0;
#pragma unroll 8
      for (int s2 = 0; s2 < BIG_NB; ++s2) zr = fma(Tb[s2 * BIG_LDS + lane], tb[s2], zr);
      if (lane < bn) zs[b0 + lane] = zr;
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
