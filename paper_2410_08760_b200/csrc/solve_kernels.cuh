// solve_kernels.cuh — master Newton step: (H + shift I) z = rhs by a blocked
// right-looking fp64 Cholesky on one thread-block cluster (reference
// algorithms.py:361-367 option b, linalg.py:133-186).
//
// Workspace M ((d+1) x (d+1) slots, column-major, lda = d + 1) holds the
// matrix in its UPPER triangle, M[j][i] = A[j][i] for j <= i < d, i.e.
// packed column i lands in column i of M (a coalesced copy), and the
// right-hand side as an extra column M[j][d] = rhs[j].  Factorising the
// augmented matrix produces L (L y = rhs, y = "row d" of L): the forward
// substitution rides along with the panel solves and trailing updates.
// L is written to the LOWER triangle, M[i][j] = L[i][j] (i >= j), so the
// upper-triangle inputs of a panel are never overwritten while other CTAs of
// the cluster may still be reading them (panel solves are redundant per CTA
// and not separated by a barrier from the owners' write-back).
//
// Per panel of NB columns there are two cluster barriers:
//   (A) rank 0 / warp 0 factors the NB x NB diagonal block (already in its
//       shared memory) and pushes L_pp and 1/diag into every CTA's shared
//       memory over DSMEM;
//   (BC) every CTA solves ALL panel rows against L_pp into its own shared
//       panel (redundant, cheap), writes the rows it owns back to M, and
//       applies its share of the trailing update; updates that land in the
//       next diagonal block are also pushed into rank 0's shared memory.
// The backward substitution L^T z = y runs on rank 0 with the next block's
// loads issued before the current block's sequential solve.
//
// The first pivot that is <= 0 or not finite stops the factorisation with
// NotPositiveDefiniteError(pivot_index, pivot_value) semantics
// (linalg.py:166-167); pivots are produced in index order.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace fb {
namespace cg = cooperative_groups;

constexpr int CH_THREADS = 256;
constexpr int CH_MAX_CLUSTER = 8;
constexpr int CH_MAX_D = 1024;

template <int NB>
struct SolveSmem {
  double blk[NB][NB + 1];  // L_pp of the current panel (row r, col s)
  double nxt[2][NB][NB + 1];  // next diagonal block (panel parity), pushed over DSMEM
  double inv[NB];          // 1 / L[jj][jj]
  double col[NB];          // column broadcast during the block factorisation
  double vec[CH_MAX_D + 64];
  double dinv[CH_MAX_D];   // 1 / L[i][i] for the backward substitution
  int failed;
};

// panel rows p1..d during the factorisation; the inverted diagonal blocks
// (transposed, ceil(d / NB) x NB rows) during the backward substitution
template <int NB>
constexpr size_t solve_panel_bytes(int d) {
  return static_cast<size_t>((d + NB) / NB * NB + 1) * (NB + 1) * sizeof(double);
}

// mode 0: x_out = fl(x - z)   (FedNL / LS direction, algorithms.py:385)
// mode 1: x_out = z           (FedNL-PP new point, algorithms.py:431)
// mode 2: x_out untouched     (leaf solve / LS: z only)
// dynamic smem: the panel, (d + 1) x (NB + 1) doubles.
template <int NB>
__global__ void __launch_bounds__(CH_THREADS, 1) k_chol_solve(
    DevCtl* __restrict__ ctl, int d, const double* __restrict__ hpk,
    const double* __restrict__ shift_ptr, const double* __restrict__ rhs,
    const double* __restrict__ x, double* __restrict__ M, double* __restrict__ z,
    double* __restrict__ x_out, int mode, int ignore_halt, long long* __restrict__ dbg) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ SolveSmem<NB> sm;
  extern __shared__ double pan[];  // [(d + 1) x (NB + 1)]: panel rows p1..d
  constexpr int PLD = NB + 1;
  const int rank = static_cast<int>(cluster.block_rank());
  const int cs = static_cast<int>(cluster.num_blocks());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = CH_THREADS / 32;
  const int gwarp = rank * NW + warp;
  const int nwarps = cs * NW;
  const int64_t ld = d + 1;
  const int rows = d + 1;  // row d of the augmented matrix carries the rhs
  long long t_mark = clock64();
  auto mark = [&](int slot) {  // optional phase timing on rank 0 / thread 0
    if (dbg && tid == 0 && rank == 0) {
      const long long now = clock64();
      dbg[slot] += now - t_mark;
      t_mark = now;
    }
  };

  // No early exit on ctl->halt (a cluster-wide decision would cost two
  // barriers): a halted round computes on stale data and rank 0 drops the
  // outputs at the end.  sm.failed is ordered before any DSMEM push by the
  // first cluster barrier below.
  if (tid == 0) sm.failed = 0;
  const double shift = shift_ptr ? __ldcg(shift_ptr) : 0.0;

  // ---- M[j][i] = H[j][i] (+ shift on the diagonal); M[j][d] = rhs[j]
  for (int i = gwarp; i <= d; i += nwarps) {
    if (i < d) {
      const int64_t pc = packed_at(0, i);
      for (int j = lane; j <= i; j += 32) {
        double v = __ldcg(hpk + pc + j);
        if (j == i) v = __dadd_rn(v, shift);
        M[j + i * ld] = v;
      }
    } else {
      for (int j = lane; j < d; j += 32) M[j + i * ld] = __ldcg(rhs + j);
    }
  }
  // every CTA stages the first diagonal block straight from H
  {
    const int pb = min(NB, d);
    for (int e = tid; e < NB * NB; e += CH_THREADS) {
      const int r = e / NB, s = e % NB;
      double v = 0.0;
      if (r < pb && s <= r) {
        v = __ldcg(hpk + packed_at(s, r));
        if (s == r) v = __dadd_rn(v, shift);
      }
      sm.nxt[0][r][s] = v;
    }
  }
  cluster.sync();
  mark(0);

  for (int p0 = 0; p0 < d; p0 += NB) {
    const int pb = min(NB, d - p0);
    const int p1 = p0 + pb;
    // ---- (A) diagonal block, factored redundantly by warp 0 of EVERY CTA
    //      (identical inputs and instruction streams give identical bits), so
    //      no barrier or exchange is needed before the panel solve.  Lane r owns
    //      row r; SB-wide sub-blocks keep the per-pivot update loop short.
    const int par = (p0 / NB) & 1;
    if (warp == 0) {
      constexpr int SB = 8;
      double row[NB];
#pragma unroll
      for (int s2 = 0; s2 < NB; ++s2) row[s2] = sm.nxt[par][lane & (NB - 1)][s2];
      // every pivot is processed (no data-dependent exit, so row[] stays in
      // registers); the first failing pivot is remembered
      int fail = NB;
      double fail_val = 0.0;
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) {  // constant trip counts: row[] stays in registers
        const int qend = (jj / SB + 1) * SB;  // end of jj's sub-block
        const double piv = __shfl_sync(0xffffffffu, row[jj], jj);
        const bool ok = piv > 0.0 && isfinite(piv);
        if (!ok && jj < pb && fail == NB) { fail = jj; fail_val = piv; }
        const double ir = rsqrt(ok ? piv : 1.0);
        if (lane == jj) sm.inv[jj] = ir;
        row[jj] = (lane == jj) ? piv * ir : ((lane > jj) ? row[jj] * ir : row[jj]);
#pragma unroll
        for (int kk = jj + 1; kk < qend; ++kk) {
          const double lk = __shfl_sync(0xffffffffu, row[jj], kk);  // L[kk][jj]
          row[kk] = (lane >= kk) ? fma(-row[jj], lk, row[kk]) : row[kk];
        }
        if (jj == qend - 1 && qend < NB) {
          // columns [qend-SB, qend) of L update columns [qend, NB) of rows >= qend
#pragma unroll
          for (int s2 = qend - SB; s2 < qend; ++s2) sm.blk[lane & (NB - 1)][s2] = row[s2];
          __syncwarp();
#pragma unroll
          for (int kk = qend; kk < NB; ++kk) {
            double acc = 0.0;
#pragma unroll
            for (int s2 = qend - SB; s2 < qend; ++s2) acc = fma(row[s2], sm.blk[kk][s2], acc);
            row[kk] = (lane >= kk) ? row[kk] - acc : row[kk];
          }
          __syncwarp();
        }
      }
      if (fail < NB) {
        if (lane == 0) {
          sm.failed = 1;
          if (rank == 0) {
            ctl->pivot_index = p0 + fail;
            ctl->pivot_value = fail_val;
            raise_status(ctl, ST_NOT_PD);
          }
        }
      } else {
#pragma unroll
        for (int s2 = 0; s2 < NB; ++s2) sm.blk[lane & (NB - 1)][s2] = (s2 <= lane) ? row[s2] : 0.0;
        if (rank == 0 && lane < pb) {
#pragma unroll
          for (int s2 = 0; s2 < NB; ++s2)
            if (s2 <= lane) M[(p0 + lane) + (p0 + s2) * ld] = row[s2];  // L, lower storage
          sm.dinv[p0 + lane] = sm.inv[lane];
        }
      }
    }
    mark(1);
    __syncthreads();
    if (sm.failed) return;  // uniform across the cluster (identical factorisations)
    mark(3);
    // ---- (B) every CTA: all panel rows i in [p1, d] (incl. the rhs row) into
    //          its own shared panel (redundant, saves an exchange barrier):
    //          column-oriented solve against L_pp with the reciprocal diagonal
    const int m = rows - p1;
    for (int r = tid; r < m; r += CH_THREADS) {
      const int i = p1 + r;
      const double* colp = M + p0 + i * ld;
      double v[NB];
#pragma unroll
      for (int s = 0; s < NB; ++s) v[s] = (s < pb) ? __ldcg(colp + s) : 0.0;
#pragma unroll
      for (int s = 0; s < NB; ++s) {
        v[s] *= sm.inv[s < pb ? s : 0];
        if (s >= pb) v[s] = 0.0;
#pragma unroll
        for (int jj = s + 1; jj < NB; ++jj) v[jj] = fma(-v[s], sm.blk[jj][s], v[jj]);
      }
#pragma unroll
      for (int s = 0; s < NB; ++s) pan[r * PLD + s] = v[s];
    }
    mark(4);
    __syncthreads();
    // rows are owned warp-round-robin across the cluster: row r -> warp r % nwarps
    for (int r = gwarp; r < m; r += nwarps) {
      const int i = p1 + r;
      for (int s = lane; s < pb; s += 32) M[i + (p0 + s) * ld] = pan[r * PLD + s];  // L[i][p0+s]
    }
    mark(5);
    if (p1 == d) {  // only the rhs row remained: y is complete
      cluster.sync();
      break;
    }
    // ---- (C) trailing update M[j][i] -= sum_s L[i][s] L[j][s], p1 <= j <= i,
    //          rows i in [p1, d] (row d updates the right-hand side)
    const int nb_next = min(NB, d - p1);
    for (int r = gwarp; r < m; r += nwarps) {  // row i = p1 + r
      const int i = p1 + r;
      const int jmax = (i == d) ? r - 1 : r;  // the rhs row has no diagonal
      double li[NB];
#pragma unroll
      for (int s = 0; s < NB; ++s) li[s] = pan[r * PLD + s];
      double* colp = M + i * ld;
      for (int jr = lane; jr <= jmax; jr += 32) {
        const int j = p1 + jr;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const double* pj = pan + jr * PLD;
#pragma unroll
        for (int s = 0; s < NB; s += 4) {
          a0 = fma(li[s], pj[s], a0);
          a1 = fma(li[s + 1], pj[s + 1], a1);
          a2 = fma(li[s + 2], pj[s + 2], a2);
          a3 = fma(li[s + 3], pj[s + 3], a3);
        }
        const double nv = __dsub_rn(__ldcg(colp + j), (a0 + a1) + (a2 + a3));
        colp[j] = nv;
        if (r < nb_next)  // next diagonal block (row r, col jr <= r) into every CTA
          for (int q = 0; q < cs; ++q) cluster.map_shared_rank(&sm, q)->nxt[par ^ 1][r][jr] = nv;
      }
    }
    mark(6);
    cluster.sync();
    mark(7);
  }
  if (rank != 0) return;

  // ---- backward substitution on rank 0 (L[j][i] = M[i][j]; y = M[:, d]):
  //      z_b = L_bb^{-T} (y_b - sum_{c > b} L_cb^T z_c), block by block; the
  //      next block and the update operands are loaded before each block's
  //      sequential solve.
  double* y = sm.vec;
  const int nb = (d + NB - 1) / NB;
  double* stage = pan;  // two [NB][NB+1] slots: L_bb^T (row r, col s) = L[b0+s][b0+r]
  for (int i = tid; i < d; i += CH_THREADS) y[i] = __ldcg(M + d + i * ld);  // L[d][i] = y_i
  // warp 0 solves the diagonal blocks; warps 1.. stage the next block and
  // prefetch the update operands of the rows they own (rows < b0)
  auto load_block = [&](int kb, double* dst) {
    const int b0 = kb * NB, bn = min(NB, d - b0);
    for (int e = tid - 32; e < NB * NB; e += CH_THREADS - 32) {
      const int s2 = e / NB, r = e % NB;  // coalesced along r
      dst[r * (NB + 1) + s2] = (r < bn && s2 < bn && s2 >= r) ? __ldcg(M + (b0 + s2) + (b0 + r) * ld) : 0.0;
    }
  };
  constexpr int UW = CH_THREADS - 32;  // update threads
  constexpr int RPT = (CH_MAX_D + UW - 1) / UW;
  if (warp != 0) load_block(nb - 1, stage + ((nb - 1) & 1) * NB * (NB + 1));
  __syncthreads();
  for (int kb = nb - 1; kb >= 0; --kb) {
    const int b0 = kb * NB, bn = min(NB, d - b0);
    double* cur = stage + (kb & 1) * NB * (NB + 1);
    if (warp == 0) {
      double zi = (lane < bn) ? y[b0 + lane] : 0.0;
      for (int s2 = bn - 1; s2 >= 0; --s2) {
        if (lane == s2) zi *= sm.dinv[b0 + s2];
        const double zs = __shfl_sync(0xffffffffu, zi, s2);
        if (lane < s2) zi = fma(-cur[lane * (NB + 1) + s2], zs, zi);
      }
      if (lane < bn) y[b0 + lane] = zi;
      __syncthreads();
      mark(8);
      __syncthreads();
    } else {
      const int ut = tid - 32;
      double mv[NB];
      int iq = ut;  // first owned row; later rows are loaded in place
#pragma unroll
      for (int s2 = 0; s2 < NB; ++s2)
        mv[s2] = (iq < b0 && s2 < bn) ? __ldcg(M + (b0 + s2) + iq * ld) : 0.0;
      if (kb > 0) load_block(kb - 1, stage + ((kb - 1) & 1) * NB * (NB + 1));
      __syncthreads();  // z_b ready
      if (iq < b0) {
        double acc = y[iq];
#pragma unroll
        for (int s2 = 0; s2 < NB; ++s2)
          if (s2 < bn) acc = fma(-mv[s2], y[b0 + s2], acc);
        y[iq] = acc;
      }
      for (int q = 1; q < RPT; ++q) {
        const int i = ut + q * UW;
        if (i < b0) {
          double acc = y[i];
          for (int s2 = 0; s2 < bn; ++s2) acc = fma(-__ldcg(M + (b0 + s2) + i * ld), y[b0 + s2], acc);
          y[i] = acc;
        }
      }
      __syncthreads();
    }
  }
  mark(9);
  if (!ignore_halt && ctl->halt) return;
  for (int i = tid; i < d; i += CH_THREADS) {
    const double zi = y[i];
    z[i] = zi;
    if (mode == 0) x_out[i] = __dsub_rn(__ldcg(x + i), zi);
    else if (mode == 1) x_out[i] = zi;
  }
}

}  // namespace fb
