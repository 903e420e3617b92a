// solve_kernels.cuh — master Newton step: (H + shift I) z = rhs by a blocked
// right-looking fp64 Cholesky on one thread-block cluster, then the two
// triangular solves (reference algorithms.py:361-367 option b,
// linalg.py:133-186).
//
// Workspace M (d x d, column-major, lda = d) holds the matrix in its UPPER
// triangle: M[j][i] = A[j][i] for j <= i, i.e. packed column i lands in
// column i of M (a coalesced copy).  After factorisation M[j][i] = L[i][j]:
// row i of L is column i of M, contiguous — the panel solve and the
// trailing update both read 32 contiguous doubles per row.
//
// The first pivot that is <= 0 or not finite stops the factorisation with
// NotPositiveDefiniteError(pivot_index, pivot_value) semantics
// (linalg.py:166-167); pivots are produced in index order.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace fb {
namespace cg = cooperative_groups;

constexpr int CH_NB = 32;
constexpr int CH_THREADS = 512;
constexpr int CH_PLD = CH_NB + 1;  // smem panel pitch (conflict-free rows)
constexpr int CH_MAX_CLUSTER = 8;

struct SolveSmem {
  double lpp[CH_NB][CH_PLD];
  double vec[1024 + 32];
  int failed;
  int halt;
};

// mode 0: x_out = fl(x - z)   (FedNL / LS direction, algorithms.py:385)
// mode 1: x_out = z           (FedNL-PP new point, algorithms.py:431)
// mode 2: x_out untouched     (leaf solve: z only)
// dynamic smem: panel staging (d * CH_PLD doubles) when `stage_panel`.
__global__ void __launch_bounds__(CH_THREADS, 1) k_chol_solve(
    DevCtl* __restrict__ ctl, int d, const double* __restrict__ hpk,
    const double* __restrict__ shift_ptr, const double* __restrict__ rhs,
    const double* __restrict__ x, double* __restrict__ M, double* __restrict__ z,
    double* __restrict__ x_out, int mode, int stage_panel, int ignore_halt) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ SolveSmem sm;
  extern __shared__ double pan[];  // [(d) x CH_PLD] when stage_panel
  const int rank = static_cast<int>(cluster.block_rank());
  const int cs = static_cast<int>(cluster.num_blocks());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gwarp = rank * (CH_THREADS / 32) + warp;
  const int nwarps = cs * (CH_THREADS / 32);
  const int gtid = rank * CH_THREADS + tid;
  const int gthreads = cs * CH_THREADS;

  // one consistent halt decision for the whole cluster: rank 0 reads the
  // control block and pushes the verdict into every CTA's shared memory
  if (tid == 0) { sm.failed = 0; sm.halt = 0; }
  cluster.sync();
  if (rank == 0 && tid == 0) {
    const int h = ignore_halt ? 0 : ctl->halt;
    for (int r = 0; r < cs; ++r) *cluster.map_shared_rank(&sm.halt, r) = h;
  }
  cluster.sync();
  if (sm.halt) return;
  const double shift = shift_ptr ? *shift_ptr : 0.0;

  // ---- M[j][i] = H[j][i] (+ shift on the diagonal), columns across warps
  for (int i = gwarp; i < d; i += nwarps) {
    const int64_t pc = packed_at(0, i);
    for (int j = lane; j <= i; j += 32) {
      double v = hpk[pc + j];
      if (j == i) v = __dadd_rn(v, shift);
      M[j + static_cast<int64_t>(i) * d] = v;
    }
  }
  cluster.sync();

  for (int p0 = 0; p0 < d; p0 += CH_NB) {
    const int pb = min(CH_NB, d - p0);
    const int p1 = p0 + pb;
    // ---- (A) diagonal block, rank 0 / warp 0: lane r owns row p0 + r
    if (rank == 0 && warp == 0) {
      double row[CH_NB];
#pragma unroll
      for (int s = 0; s < CH_NB; ++s)
        row[s] = (lane < pb && s <= lane) ? M[(p0 + s) + static_cast<int64_t>(p0 + lane) * d] : 0.0;
      int fail = -1;
      double fail_val = 0.0;
#pragma unroll
      for (int jj = 0; jj < CH_NB; ++jj) {
        if (jj < pb && fail < 0) {
          const double piv = __shfl_sync(0xffffffffu, row[jj], jj);
          if (!(piv > 0.0) || !isfinite(piv)) {
            fail = jj;
            fail_val = piv;
          } else {
            const double r = sqrt(piv);
            if (lane == jj) row[jj] = r;
            if (lane > jj) row[jj] = row[jj] / r;
            const double lj = row[jj];
            // rank-1 update of the remaining columns of this row
#pragma unroll
            for (int kk = jj + 1; kk < CH_NB; ++kk) {
              const double lk = __shfl_sync(0xffffffffu, lj, kk);  // L[kk][jj]
              if (lane >= kk && kk < pb) row[kk] = fma(-lj, lk, row[kk]);
            }
          }
        }
      }
      if (fail >= 0) {
        if (lane == 0) {
          for (int r = 0; r < cs; ++r) *cluster.map_shared_rank(&sm.failed, r) = 1;
          ctl->pivot_index = p0 + fail;
          ctl->pivot_value = fail_val;
          raise_status(ctl, ST_NOT_PD);
        }
      } else if (lane < pb) {
#pragma unroll
        for (int s = 0; s < CH_NB; ++s)
          if (s <= lane) M[(p0 + s) + static_cast<int64_t>(p0 + lane) * d] = row[s];
      }
    }
    cluster.sync();
    if (sm.failed) return;
    if (p1 >= d) break;
    // ---- (B) panel rows i >= p1:  L[i][p0:p1] = A[i][p0:p1] L_pp^{-T}
    for (int e = tid; e < CH_NB * CH_NB; e += CH_THREADS) {
      const int r = e / CH_NB, s = e % CH_NB;
      sm.lpp[r][s] = (r < pb && s <= r) ? M[(p0 + s) + static_cast<int64_t>(p0 + r) * d] : 0.0;
    }
    __syncthreads();
    for (int i = p1 + gtid; i < d; i += gthreads) {
      double* col = M + p0 + static_cast<int64_t>(i) * d;
      double v[CH_NB];
#pragma unroll
      for (int s = 0; s < CH_NB; ++s) v[s] = (s < pb) ? col[s] : 0.0;
#pragma unroll
      for (int jj = 0; jj < CH_NB; ++jj) {
        if (jj < pb) {
          double acc = v[jj];
#pragma unroll
          for (int s = 0; s < jj; ++s) acc = fma(-v[s], sm.lpp[jj][s], acc);
          v[jj] = acc / sm.lpp[jj][jj];
        }
      }
#pragma unroll
      for (int s = 0; s < CH_NB; ++s)
        if (s < pb) col[s] = v[s];
    }
    cluster.sync();
    // ---- (C) trailing update M[j][i] -= sum_s L[i][s] L[j][s], p1 <= j <= i
    const int m = d - p1;
    const double* P;
    int pld;
    if (stage_panel) {
      for (int e = tid; e < m * CH_NB; e += CH_THREADS) {
        const int r = e / CH_NB, s = e % CH_NB;
        pan[r * CH_PLD + s] = (s < pb) ? M[(p0 + s) + static_cast<int64_t>(p1 + r) * d] : 0.0;
      }
      __syncthreads();
      P = pan;
      pld = CH_PLD;
    } else {
      P = nullptr;
      pld = 0;
    }
    for (int r = gwarp; r < m; r += nwarps) {  // row i = p1 + r
      const int i = p1 + r;
      double li[CH_NB];
#pragma unroll
      for (int s = 0; s < CH_NB; ++s)
        li[s] = P ? P[r * pld + s] : ((s < pb) ? M[(p0 + s) + static_cast<int64_t>(i) * d] : 0.0);
      double* col = M + static_cast<int64_t>(i) * d;
      for (int jr = lane; jr <= r; jr += 32) {
        const int j = p1 + jr;
        double acc = 0.0;
        if (P) {
#pragma unroll
          for (int s = 0; s < CH_NB; ++s) acc = fma(li[s], P[jr * pld + s], acc);
        } else {
          const double* cj = M + p0 + static_cast<int64_t>(j) * d;
#pragma unroll 8
          for (int s = 0; s < pb; ++s) acc = fma(li[s], __ldcg(cj + s), acc);
        }
        col[j] = __dsub_rn(col[j], acc);
      }
    }
    cluster.sync();
  }
  if (rank != 0) return;

  // ---- triangular solves on rank 0: L y = rhs, then L^T z = y
  double* y = sm.vec;
  for (int i = tid; i < d; i += CH_THREADS) y[i] = rhs[i];
  __syncthreads();
  for (int b0 = 0; b0 < d; b0 += CH_NB) {
    const int bn = min(CH_NB, d - b0);
    if (warp == 0) {
      const int i = b0 + lane;
      double yi = (lane < bn) ? y[i] : 0.0;
      for (int s = 0; s < bn; ++s) {
        if (lane == s) yi = yi / M[i + static_cast<int64_t>(i) * d];
        const double ys = __shfl_sync(0xffffffffu, yi, s);
        if (lane > s && lane < bn) yi = fma(-M[(b0 + s) + static_cast<int64_t>(i) * d], ys, yi);
      }
      if (lane < bn) y[i] = yi;
    }
    __syncthreads();
    for (int i = b0 + bn + tid; i < d; i += CH_THREADS) {
      const double* col = M + b0 + static_cast<int64_t>(i) * d;
      double acc = y[i];
      for (int s = 0; s < bn; ++s) acc = fma(-col[s], y[b0 + s], acc);
      y[i] = acc;
    }
    __syncthreads();
  }
  // backward: z_i = (y_i - sum_{j > i} L[j][i] z_j) / L[i][i],  L[j][i] = M[i][j]
  const int nb = (d + CH_NB - 1) / CH_NB;
  for (int kb = nb - 1; kb >= 0; --kb) {
    const int b0 = kb * CH_NB, bn = min(CH_NB, d - b0);
    if (warp == 0) {
      const int i = b0 + lane;
      double zi = (lane < bn) ? y[i] : 0.0;
      for (int s = bn - 1; s >= 0; --s) {
        if (lane == s) zi = zi / M[i + static_cast<int64_t>(i) * d];
        const double zs = __shfl_sync(0xffffffffu, zi, s);
        if (lane < s) zi = fma(-M[i + static_cast<int64_t>(b0 + s) * d], zs, zi);  // L[b0+s][i]
      }
      if (lane < bn) y[i] = zi;
    }
    __syncthreads();
    for (int i = tid; i < b0; i += CH_THREADS) {
      double acc = y[i];
      for (int s = 0; s < bn; ++s) acc = fma(-M[i + static_cast<int64_t>(b0 + s) * d], y[b0 + s], acc);
      y[i] = acc;
    }
    __syncthreads();
  }
  for (int i = tid; i < d; i += CH_THREADS) {
    const double zi = y[i];
    z[i] = zi;
    if (mode == 0) x_out[i] = __dsub_rn(x[i], zi);
    else if (mode == 1) x_out[i] = zi;
  }
}

}  // namespace fb
