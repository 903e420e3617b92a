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
#include "round_kernels.cuh"

namespace fb {
namespace cg = cooperative_groups;

constexpr int CH_THREADS = 256;
constexpr int CH_MAX_CLUSTER = 8;
constexpr int CH_MAX_D = 1024;
constexpr int CH_DMMA_MIN_D = 256;  // trailing update on DMMA tiles above this d

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
  if (tid == 0) tl_mark(2, false);
  for (int k2 = tid; k2 < PLD; k2 += CH_THREADS) pan[(d + NB) / NB * NB * PLD + k2] = 0.0;  // zero row
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
    //          rows i in [p1, d] (row d updates the right-hand side): the
    //          lower-triangular 8 x 8 tiles (row tile ti >= column tile tj) of
    //          P P^T on DMMA.8x8x4 (P = the m x NB panel in shared memory),
    //          TB tiles per warp in flight, the M operands loaded first
    const int nb_next = min(NB, d - p1);
    if (d > CH_DMMA_MIN_D) {  // DMMA tiles (large d: c4)
      const int g = lane >> 2, tg = lane & 3;
      const int mz = (d + NB) / NB * NB;  // a panel row never written: zeros (set up front)
      const int T = (m + 7) >> 3;
      const int ntile = T * (T + 1) / 2;
      constexpr int TB = 4;
      for (int q0 = gwarp * TB; q0 < ntile; q0 += nwarps * TB) {
        int ti[TB], tj[TB];
        double mv[TB][2], acc[TB][2];
#pragma unroll
        for (int u = 0; u < TB; ++u) {
          const int q = q0 + u;
          int a2 = static_cast<int>((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
          while ((a2 + 1) * (a2 + 2) / 2 <= q) ++a2;
          while (a2 * (a2 + 1) / 2 > q) --a2;
          ti[u] = q < ntile ? a2 : -1;
          tj[u] = q - a2 * (a2 + 1) / 2;
          acc[u][0] = acc[u][1] = 0.0;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = ti[u] * 8 + g, jr = tj[u] * 8 + 2 * tg + e;
            const bool ok = ti[u] >= 0 && r < m && jr <= r && p1 + jr < d;
            mv[u][e] = ok ? __ldcg(M + (p1 + jr) + static_cast<int64_t>(p1 + r) * ld) : 0.0;
          }
        }
        const double* pa[TB];
        const double* pb2[TB];
#pragma unroll
        for (int u = 0; u < TB; ++u) {  // rows past m read the zero row past the panel
          const int ra = ti[u] * 8 + g, rb = tj[u] * 8 + g;
          pa[u] = pan + (ti[u] >= 0 && ra < m ? ra : mz) * PLD + tg;
          pb2[u] = pan + (ti[u] >= 0 && rb < m ? rb : mz) * PLD + tg;
        }
#pragma unroll
        for (int k0 = 0; k0 < NB; k0 += 4) {
          double av[TB], bv[TB];
#pragma unroll
          for (int u = 0; u < TB; ++u) {
            av[u] = pa[u][k0];
            bv[u] = pb2[u][k0];
          }
#pragma unroll
          for (int u = 0; u < TB; ++u) dmma_8x8x4_nv(acc[u], av[u], bv[u]);
        }
#pragma unroll
        for (int u = 0; u < TB; ++u) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = ti[u] * 8 + g, jr = tj[u] * 8 + 2 * tg + e;
            if (!(ti[u] >= 0 && r < m && jr <= r && p1 + jr < d)) continue;
            const double nv = __dsub_rn(mv[u][e], acc[u][e]);
            M[(p1 + jr) + static_cast<int64_t>(p1 + r) * ld] = nv;
            if (r < nb_next)  // next diagonal block (row r, col jr <= r) into every CTA
              for (int qc = 0; qc < cs; ++qc) cluster.map_shared_rank(&sm, qc)->nxt[par ^ 1][r][jr] = nv;
          }
        }
      }
    }
    else {  // small d: one warp per row, FMA dot products against the panel
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
  if (tid == 0) tl_mark(2, true);
  if (!ignore_halt && ctl->halt) return;
  for (int i = tid; i < d; i += CH_THREADS) {
    const double zi = y[i];
    z[i] = zi;
    if (mode == 0) x_out[i] = __dsub_rn(__ldcg(x + i), zi);
    else if (mode == 1) x_out[i] = zi;
  }
}

}  // namespace fb

namespace fb {

// ===========================================================================
// k_chol_panels — panel-owning blocked Cholesky for d <= CP_MAX_D.
//
// The matrix is cut into 32-column panels; panel p lives in the shared
// memory of cluster CTA p % cs (KP = 1 or 2 panels per CTA), as rows
// ("slots") i - p0 of columns [p0, p0 + 32) of the lower triangle plus the
// right-hand side as a final slot (the forward substitution rides along).
// Per panel p its owner
//   A  factors the 32 x 32 diagonal block (warp 0) and forms T = L_pp^-1,
//      while its other warps finish the pending update of the panel's lower
//      rows from panel p - 1,
//   B  solves the rows below the block, X = A T^T, on the fp64 tensor cores
//      (mma.sync m8n8k4 / DMMA), writes L_p to global memory and releases it
//      to every CTA through a cluster-scope mbarrier arrive.
// Every CTA applies L_p to its own later panels as soon as it is released
// (C_q -= L_p L_p^T restricted to panel q, DMMA, operands from L2) — the
// panel that is factored next gets its diagonal rows first (lookahead), so
// the critical path per panel is one release + 4 DMMA row tiles + the block
// factor + the TRSM.  The backward substitution runs panel by panel from the
// last: the owner of panel b forms z_b = T_b^T (y_b - w_b), where w_b was
// accumulated from the z of later panels as they were released, and pushes
// z_b into every CTA over DSMEM.
//
// The factorisation order differs from the reference's column loop
// (linalg.py:151-170); results agree to rounding (parity bar 1e-10).  The
// first pivot that is <= 0 or not finite raises NotPositiveDefiniteError
// (index, value) semantics, pivots being produced in index order.
// ===========================================================================
constexpr int CP_NB = 32;
constexpr int CP_LS = 36;  // slot stride (doubles): conflict-free DMMA fragment loads
constexpr int CP_MAXP = 16;
// warps that update the panel's lower rows while warp 0 factors its diagonal
// block: the block factor is latency-bound on shuffles, and warps sharing
// its scheduler / the smem pipe slow it (measured: excluding warp 4 cut the
// per-panel factor from 8.6 to 7.5 us)
#ifndef CP_MARKS
#define CP_MARKS 0
#endif
#ifndef CP_NO_PUSH
#define CP_NO_PUSH 0
#endif
#ifndef CP_REST_WARPS
#define CP_REST_WARPS 0xECu
#endif
constexpr int CP_MAX_D = CP_MAXP * CP_NB;
// one panel per CTA up to this many panels: a non-portable cluster (B200
// allows 16), so no CTA serves two panels (at c0's 10 panels the owner of
// two competed between its next factor and the other panel's updates)
#ifndef CP_MAX_CLUSTER
#define CP_MAX_CLUSTER 16
#endif

// The round reduction (k_reduce's outputs, round_kernels.cuh) folded into the
// solve cluster's prologue: `grad` non-null selects it.  CTA r forms gbar
// for its own panels' features (exactly the right-hand-side entries it
// holds) and the per-client scalars of client chunk r; the cluster-wide sums
// go through DSMEM in rank order, so every CTA derives the same shift.
struct CpRed {
  int n_active, n_div, nblk, n_pairs;
  const int32_t* ni;         // [n] samples per client
  const double* lam;         // [n] lambda per client
  const double* grad;        // [n][d] local gradients (Hessian pass)
  const double* loss_part;   // [n][nblk]
  const double* frob_part;   // [n][n_pairs]
  const int32_t* flags;      // [n]
  double* gbar;              // [d]
  double* f_cli;             // [n]
  double* shift_cli;         // [n]
  RoundScalars* out;
  double* row_grad;
  double* row_f;
};

struct CpSmem {
  double T[2][CP_NB][CP_LS];  // inverse diagonal blocks of the own panels
  double z[CP_MAX_D];         // solution entries released so far
  double w[2][CP_NB];         // back-substitution accumulators of the own panels
  double part[8][CP_NB];
  double inv[CP_NB];
  // slots 32..95 of L_{q-1} for the own panel q factored next, pushed over
  // DSMEM by its owner: rows 0..31 are q's diagonal rows (and the B operand
  // of every pending update of q), rows 32..63 the A operand of q's head
  double rcv[2 * CP_NB][CP_LS];
  uint64_t barL[CP_MAXP];    // L2 copy of L_p released
  uint64_t barLd[CP_MAXP];   // rcv rows 0..31 landed (transaction bytes)
  uint64_t barLd2[CP_MAXP];  // rcv rows 32..63 landed (transaction bytes)
  uint64_t barZ[CP_MAXP];    // z_b landed (transaction bytes)
  uint64_t barRF;            // the next owner's rcv is free again (second push)
  uint64_t barF[CP_NB];      // block factor: pivot j's row and 1/sqrt published
  double rpart[4];           // fused reduction: this CTA's partials (gg, fs, ss, bad)
  double gown[2 * CP_NB];    // fused reduction: gbar of the own panels' features
  double rscr[8];
  double rscr3[3 * CH_THREADS / 32];
  int rbad;
  int failed;
};

__host__ __device__ constexpr int cp_rows(int d) { return (d > CP_NB ? d : CP_NB) + 1; }
// bytes of L_p's slots [lo, lo + 32) (lo = 32: the next panel's diagonal
// rows; lo = 64: the A rows of its head update) pushed to the next owner:
// real rows plus the right-hand side slot when it falls in the range
__host__ __device__ constexpr uint32_t cp_push_bytes(int d, int p, int lo) {
  return static_cast<uint32_t>(
      ((d - p * 32 - lo < 0 ? 0 : (d - p * 32 - lo > 32 ? 32 : d - p * 32 - lo)) +
       ((d - p * 32 >= lo && d - p * 32 < lo + 32) ? 1 : 0)) * 32 * 8);
}
// dynamic shared memory for the panels: what the 227 KB per CTA leaves
// next to the static CpSmem
// diagnostics (fb_solve_phase_cycles): per-CTA timestamps staged in dynamic
// shared memory after the panels, flushed at the end (a global store per
// stamp would itself stall behind the SM's outstanding memory traffic);
// rows 0..CP_MAXP-1 per panel, row CP_MAXP for the end markers (p = 63)
constexpr size_t CP_STAMP_BYTES = (CP_MAXP + 1) * 16 * sizeof(long long);
constexpr size_t CP_DYN_SMEM_MAX = 227 * 1024 - sizeof(CpSmem) - 512 - CP_STAMP_BYTES;
__host__ __device__ constexpr size_t cp_panel_bytes(int d) {
  return static_cast<size_t>(cp_rows(d)) * CP_LS * sizeof(double);
}

// C_q[slots] -= L_p[rows] L_p[jrows]^T for q's slots in [s_lo, s_hi] (row
// tiles of 8, warps [w_lo, w_hi) round robin).  L_p is read from global
// (__ldcg: written by another SM during this launch) or from local shared
// memory.
// The receiver's diagonal-block update from the pushed rows (slots 0..31 of
// panel q, A = B = rcv rows 0..31): the four 8-row tiles in column halves
// over all eight warps (16 DMMAs each).
__device__ __forceinline__ void cp_update_diag8(const double* __restrict__ Lr, double* __restrict__ Pq,
                                                int d, int q0, int nreal_q) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = warp & 3, h = warp >> 2;
  double b[8][2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int jj = (2 * h + j) * 8 + (lane >> 2);
    const bool ok = q0 + jj < d;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) b[ks][j] = ok ? Lr[jj * CP_LS + ks * 4 + (lane & 3)] : 0.0;
  }
  const int r = tile * 8 + (lane >> 2);
  const bool rok = r < nreal_q;
  double a[8];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) a[ks] = rok ? -Lr[r * CP_LS + ks * 4 + (lane & 3)] : 0.0;
  double acc[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int cc = (2 * h + j) * 8 + 2 * (lane & 3);
    acc[j][0] = rok ? Pq[r * CP_LS + cc] : 0.0;
    acc[j][1] = rok ? Pq[r * CP_LS + cc + 1] : 0.0;
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[j], a[ks], b[ks][j]);
  if (rok) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int cc = (2 * h + j) * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(Pq + r * CP_LS + cc) = make_double2(acc[j][0], acc[j][1]);
    }
  }
}

template <bool GLOBAL>
__device__ __forceinline__ void cp_update(const double* __restrict__ Lp, int p, int q,
                                          double* __restrict__ Pq, int d, int s_lo, int s_hi,
                                          int w_lo, int w_hi, int src_slot_off = 0,
                                          uint32_t warp_mask = 0xffu) {
  const int warp_id = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // participating warps: [w_lo, w_hi) intersected with warp_mask, renumbered densely
  const uint32_t part = warp_mask & (((1u << w_hi) - 1u) & ~((1u << w_lo) - 1u));
  if (!((part >> warp_id) & 1u)) return;
  const int warp = w_lo + __popc(part & ((1u << warp_id) - 1u));
  w_hi = w_lo + __popc(part);
  const int p0 = p * CP_NB, q0 = q * CP_NB;
  const int nreal_q = d - q0, rs_q = max(nreal_q, CP_NB), rs_p = max(d - p0, CP_NB);
  const int off = q0 - p0;
  auto ld = [&](int slot, int col) -> double {
    const double* a = Lp + static_cast<int64_t>(slot - src_slot_off) * CP_LS + col;
    return GLOBAL ? __ldcg(a) : *a;
  };
  // B fragments: b = L_p[j][k], j = q0 + 8 ct + (lane >> 2), k = 4 ks + (lane & 3)
  double b[8][4];
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) {
    const int jj = ct * 8 + (lane >> 2);
    const bool ok = q0 + jj < d;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) b[ks][ct] = ok ? ld(off + jj, ks * 4 + (lane & 3)) : 0.0;
  }
  const int t_lo = s_lo >> 3, t_hi = s_hi >> 3;
  for (int tile = t_lo + (warp - w_lo); tile <= t_hi; tile += (w_hi - w_lo)) {
    const int r = tile * 8 + (lane >> 2);  // this lane's A row slot
    int src = -1;
    if (r >= s_lo && r <= s_hi) {
      if (r < nreal_q) src = r + off;
      else if (r == rs_q) src = rs_p;
    }
    double a[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) a[ks] = src >= 0 ? -ld(src, ks * 4 + (lane & 3)) : 0.0;
    // C fragments: rows tile*8 + (lane >> 2), cols 8 ct + 2 (lane & 3) + {0, 1}
    const int cr = tile * 8 + (lane >> 2);
    const bool cok = cr >= s_lo && cr <= s_hi && (cr < nreal_q || cr == rs_q);
    double acc[4][2];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int cc = ct * 8 + 2 * (lane & 3);
      acc[ct][0] = cok ? Pq[cr * CP_LS + cc] : 0.0;
      acc[ct][1] = cok ? Pq[cr * CP_LS + cc + 1] : 0.0;
    }
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) dmma_8x8x4(acc[ct], a[ks], b[ks][ct]);
    if (cok) {
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) {
        const int cc = ct * 8 + 2 * (lane & 3);
        Pq[cr * CP_LS + cc] = acc[ct][0];
        Pq[cr * CP_LS + cc + 1] = acc[ct][1];
      }
    }
  }
}

// One 8-row tile (slots 8 tile ..) of panel q -= L_pp[A rows] (L_pp slots
// 32..63)^T, pp = q - 1: the A rows (slots + 32, the right-hand side slot
// mapped to L_pp's) come from the released L2 copy of L_pp, the B rows from
// this CTA's pushed copy `Bs` (rcv rows 0..31).  One warp.
__device__ __forceinline__ void cp_tile_update_l2(const double* __restrict__ Lsrc,
                                                  const double* __restrict__ Bs, double* __restrict__ Pq,
                                                  int tile, int d, int q0, int nreal_q, int rs_q, int rs_pp) {
  const int lane = threadIdx.x & 31;
  const int r = tile * 8 + (lane >> 2);
  int src = -1;
  if (r < nreal_q) src = r + CP_NB;
  else if (r == rs_q) src = rs_pp;
  double a[8];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
    a[ks] = src >= 0 ? -__ldcg(Lsrc + static_cast<int64_t>(src) * CP_LS + ks * 4 + (lane & 3)) : 0.0;
  const bool cok = r < nreal_q || r == rs_q;
  double acc[4][2];
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) {
    const int cc = ct * 8 + 2 * (lane & 3);
    acc[ct][0] = cok ? Pq[r * CP_LS + cc] : 0.0;
    acc[ct][1] = cok ? Pq[r * CP_LS + cc + 1] : 0.0;
  }
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) {
    const int jj = ct * 8 + (lane >> 2);
    const bool ok = q0 + jj < d;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      dmma_8x8x4(acc[ct], a[ks], ok ? Bs[jj * CP_LS + ks * 4 + (lane & 3)] : 0.0);
  }
  if (cok) {
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
      const int cc = ct * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(Pq + r * CP_LS + cc) = make_double2(acc[ct][0], acc[ct][1]);
    }
  }
}

template <int KP>
__global__ void __launch_bounds__(CH_THREADS, 1) k_chol_panels(
    DevCtl* __restrict__ ctl, int d, const double* __restrict__ hpk,
    const double* __restrict__ shift_ptr, const double* __restrict__ rhs,
    const double* __restrict__ x, double* __restrict__ Lg, double* __restrict__ z,
    double* __restrict__ x_out, int mode, int ignore_halt, long long* __restrict__ dbg, CpRed red) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ CpSmem sm;
  extern __shared__ __align__(16) double cpan[];
  const int rank = static_cast<int>(cluster.block_rank());
  const int cs = static_cast<int>(cluster.num_blocks());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npan = (d + CP_NB - 1) / CP_NB;
  const int RS = cp_rows(d);
  if (tid == 0) tl_mark(2, false);
  long long t_mark = clock64();
  auto mark = [&](int slot) {
    if (CP_MARKS && dbg && tid == 0 && rank == 0) {
      const long long now = clock64();
      dbg[slot] += now - t_mark;
      t_mark = now;
    }
  };
  auto P = [&](int k) { return cpan + static_cast<size_t>(k) * RS * CP_LS; };
  // diagnostics: per-panel global timestamps (fb_debug_counters)
  long long* stamps = reinterpret_cast<long long*>(cpan + static_cast<size_t>(KP) * RS * CP_LS);
  auto srow = [&](int p) { return p < CP_MAXP ? p : (p == 63 ? CP_MAXP : -1); };
  // a predicated store, not a branch: a branch taken by one lane would leave
  // the warp split for the code that follows (twice the issue slots)
  // (also in the production round while g_dbg_on: to g_dbg_cta, row p = panel)
  const bool stamping = dbg != nullptr || g_dbg_on;
  auto stamp_if = [&](bool on, int p, int k) {
    if (stamping) {
      const long long tv = globaltimer_ns();
      const int row = srow(p);
      const uint32_t addr = smem_u32(stamps + (row < 0 ? 0 : row) * 16 + k);
      asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u64 [%0], %1;\n\t}" ::"r"(addr),
                   "l"(tv), "r"(static_cast<uint32_t>(on && row >= 0))
                   : "memory");
    }
  };
  auto stamp = [&](int p, int k) { stamp_if(tid == 0, p, k); };  // dbg[16 + 16 p + k], thread 0
  auto stamp_w = [&](int p, int k, int w) { stamp_if(tid == 32 * w, p, k); };  // lane 0 of warp w
  if (stamping)
    for (int i = tid; i < (CP_MAXP + 1) * 16; i += CH_THREADS) stamps[i] = 0;
  auto Lglob = [&](int p) { return Lg + static_cast<size_t>(p) * RS * CP_LS; };
  const int last_own = rank + ((npan - 1 - rank) / cs) * cs;  // highest own panel (rank < npan)
  int fac_uses = 0;  // block factors done by this CTA (parity of sm.barF)
  // per own panel: bit p' = L_{p'} still owed to it (deferred by the apply
  // step while the CTA's next panel was two steps away)
  uint32_t pend[2] = {0u, 0u};

  if (tid == 0) {
    for (int p = 0; p < npan; ++p) {
      mbar_init(&sm.barL[p], 1);
      mbar_init(&sm.barLd[p], 1);
      mbar_init(&sm.barLd2[p], 1);
      mbar_init(&sm.barZ[p], 1);
    }
    mbar_init(&sm.barRF, 1);
    for (int j = 0; j < CP_NB; ++j) mbar_init(&sm.barF[j], 1);
    fence_barrier_init();
    sm.rbad = 0x7fffffff;
    // the backward substitution's z_b arrives by st.async (complete_tx): this
    // CTA's single arrival on barZ[b] is the byte count it expects
    for (int b = 0; b < npan; ++b)
      if (rank < b && rank != b % cs)
        mbar_arrive_expect_tx(&sm.barZ[b], static_cast<uint32_t>(min(CP_NB, d - b * CP_NB)) * 8u);
    // likewise L_p's slots 32..95 pushed to the next owner in step B of p
    for (int p = 0; p + 1 < npan; ++p)
      if ((p + 1) % cs == rank) {
        mbar_arrive_expect_tx(&sm.barLd[p], cp_push_bytes(d, p, 32));
        mbar_arrive_expect_tx(&sm.barLd2[p], cp_push_bytes(d, p, 64));
      }
    sm.failed = 0;
  }
  // ---- own panels from packed H (A[i][j] = H[min][max]), + shift
  //      on the diagonal, identity padding, right-hand side as the last slot
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int q = rank + k * cs;
    if (q >= npan) break;
    const int q0 = q * CP_NB, nreal = d - q0, rs = max(nreal, CP_NB), pb = min(CP_NB, nreal);
    double* Pq = P(k);
    // 8 independent loads in flight per thread (the setup is on the critical
    // path and H^k is usually not in L2 after the Hessian pass)
    constexpr int UL = 8;
    const int n_el = (rs + 1) * CP_NB;
    for (int e0 = tid; e0 < n_el; e0 += UL * CH_THREADS) {
      double v[UL];
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        const int e = e0 + u * CH_THREADS;
        const int r = e / CP_NB, c = e % CP_NB;
        double vv = 0.0;
        if (e < n_el) {
          if (r == rs) {
            vv = 0.0;  // right-hand side: after the dependency wait below
          } else if (r < nreal) {
            // the diagonal block in full (the block factor reads it as
            // symmetric columns), the rows below as the lower triangle
            const int i = q0 + r, j = q0 + c;
            const int hi = max(i, j), lo = min(i, j);
            if (c < pb) vv = __ldcg(hpk + static_cast<int64_t>(hi) * (hi + 1) / 2 + lo);
          } else {
            vv = (r == c) ? 1.0 : 0.0;  // padding of the last panel's diagonal block
          }
        }
        v[u] = vv;
      }
#pragma unroll
      for (int u = 0; u < UL; ++u) {
        const int e = e0 + u * CH_THREADS;
        if (e < n_el) Pq[(e / CP_NB) * CP_LS + e % CP_NB] = v[u];
      }
    }
  }
  // H^k is ready before the round reduction finishes (programmatic dependent
  // launch: this kernel may start while k_reduce still runs); the shift and
  // the right-hand side come from k_reduce, so wait for it here.  Without a
  // programmatic dependency the wait returns at once.
  if (tid == 0) tl_mark(3, false);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tid == 0) tl_mark(3, true);
  double shift = 0.0;
  const bool fused = red.grad != nullptr;
  bool skip_solve = false;  // fused reduction found a non-finite client (uniform)
  if (fused) {
    // ---- the round reduction (k_reduce), cluster-parallel
    const int n = red.n_active;
    double(*rwork)[2 * CP_NB] = reinterpret_cast<double(*)[2 * CP_NB]>(&sm.T[0][0][0]);  // free until the factor
    // (a) gbar of the own panels' features: warp w sums clients w, w + 8, ..
    //     for features lo + lane (+ 32), coalesced; then the 8 warps in order
    const int q_lo = rank;  // own panels rank, rank + cs (feature slots 0..63)
    double acc0 = 0.0, acc1 = 0.0;
    const int a0 = q_lo * CP_NB + lane;
    const int a1 = (KP > 1 && q_lo + cs < npan) ? (q_lo + cs) * CP_NB + lane : d;
    constexpr int GU = 18;  // clients per warp and batch: n <= 144 in one round trip
    // Every load of the reduction is issued before any is consumed: a
    // dependent round trip costs 1-2 us while the compressor streams D.
    // (b) staging: this CTA's client chunk's loss / Frobenius partials and
    // lambda / n_i / flags, in the rcv buffer (free until panel 0's push)
    const int cpc = (n + cs - 1) / cs;
    const int c_lo = min(n, rank * cpc), c_hi = min(n, c_lo + cpc);
    const int per_c = red.nblk + red.n_pairs;
    const int per_s = per_c + 3;
    double* stage = &sm.rcv[0][0];
    const int chunk = max(1, (2 * CP_NB * CP_LS) / per_s);
    auto stage_chunk = [&](int i0, int nc) {
      for (int e = tid; e < nc * per_s; e += CH_THREADS) {
        const int ii = e / per_s, r = e - ii * per_s, c = i0 + ii;
        double v;
        if (r < red.nblk) v = __ldcg(red.loss_part + static_cast<int64_t>(c) * red.nblk + r);
        else if (r < per_c) v = __ldcg(red.frob_part + static_cast<int64_t>(c) * red.n_pairs + (r - red.nblk));
        else if (r == per_c) v = red.lam[c];
        else if (r == per_c + 1) v = static_cast<double>(red.ni[c]);
        else v = static_cast<double>(__ldcg(red.flags + c));
        stage[e] = v;
      }
    };
    double v0[GU], v1[GU];
    for (int c0 = warp; c0 < n; c0 += 8 * GU) {
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int c = c0 + 8 * u;
        v0[u] = (c < n && a0 < d) ? __ldcg(red.grad + static_cast<int64_t>(c) * d + a0) : 0.0;
        v1[u] = (c < n && a1 < d) ? __ldcg(red.grad + static_cast<int64_t>(c) * d + a1) : 0.0;
      }
      if (c0 == warp) {  // with the first gradient batch in flight
        stage_chunk(c_lo, min(chunk, c_hi - c_lo));
      }
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        acc0 = __dadd_rn(acc0, v0[u]);
        acc1 = __dadd_rn(acc1, v1[u]);
      }
    }
    if (n <= warp) stage_chunk(c_lo, min(chunk, c_hi - c_lo));  // (no gradient batch on this warp)
    if (tid == 0) tl_mark(9, true);
    rwork[warp][lane] = acc0;
    rwork[warp][CP_NB + lane] = acc1;
    double xx_p = 0.0;
    for (int a = tid; a < d; a += CH_THREADS) xx_p = fma(x[a], x[a], xx_p);
    double fs_t = 0.0, ss_t = 0.0;
    int bad_t = 0x7fffffff;
    __syncthreads();
    const double xx = block_sum(xx_p, sm.rscr);
    if (tid < 2 * CP_NB) {
      double t2 = 0.0;
#pragma unroll
      for (int w2 = 0; w2 < 8; ++w2) t2 = __dadd_rn(t2, rwork[w2][tid]);
      sm.gown[tid] = __ddiv_rn(t2, static_cast<double>(red.n_div));
    }
    // per-client scalars: thread per client, the partials summed in order
    for (int i0 = c_lo; i0 < c_hi; i0 += chunk) {
      const int nc = min(chunk, c_hi - i0);
      if (i0 != c_lo) {
        __syncthreads();
        stage_chunk(i0, nc);
        __syncthreads();
      }
      for (int ii = tid; ii < nc; ii += CH_THREADS) {
        const int c = i0 + ii;
        const double* st = stage + ii * per_s;
        double ls = 0.0, fp = 0.0;
        for (int r = 0; r < red.nblk; ++r) ls = __dadd_rn(ls, st[r]);
        for (int r = red.nblk; r < per_c; ++r) fp = __dadd_rn(fp, st[r]);
        const double reg = __dmul_rn(__dmul_rn(0.5, st[per_c]), xx);
        const double fc = __dadd_rn(__ddiv_rn(ls, st[per_c + 1]), reg);
        const double sc = sqrt(fp);
        red.f_cli[c] = fc;
        red.shift_cli[c] = sc;
        fs_t += fc;
        ss_t += sc;
        if (static_cast<int>(st[per_c + 2]) & 1) bad_t = min(bad_t, c);
      }
    }
    __syncthreads();
    if (tid == 0) tl_mark(10, true);
    double gg_t = 0.0;
    if (tid < 2 * CP_NB) {
      const int a = tid < CP_NB ? a0 - lane + tid : (a1 < d ? a1 - lane + tid - CP_NB : d);
      if (a < d) {
        const double g = sm.gown[tid];
        red.gbar[a] = g;
        gg_t = g * g;
      }
    }
    double gg = gg_t, fs = fs_t, ss = ss_t;
    block_sum3(gg, fs, ss, sm.rscr3);
    bad_t = __reduce_min_sync(0xffffffffu, bad_t);
    if (lane == 0 && bad_t != 0x7fffffff) atomicMin(&sm.rbad, bad_t);
    __syncthreads();
    if (tid == 0) {
      sm.rpart[0] = gg;
      sm.rpart[1] = fs;
      sm.rpart[2] = ss;
      sm.rpart[3] = static_cast<double>(sm.rbad);
      sm.rscr[0] = xx;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int q = rank + k * cs;
    if (q >= npan) break;
    const int q0 = q * CP_NB, nreal = d - q0, rs = max(nreal, CP_NB), pb = min(CP_NB, nreal);
    double* Pq = P(k);
    if (tid < CP_NB)
      Pq[rs * CP_LS + tid] = tid < pb ? (fused ? sm.gown[k * CP_NB + tid] : __ldcg(rhs + q0 + tid)) : 0.0;
  }
  if (tid == 0) tl_mark(11, false);
  cluster.sync();  // barriers initialised and reduction partials published cluster-wide
  if (tid == 0) tl_mark(11, true);
  if (fused) {
    // cluster sums in rank order (identical in every CTA)
    double gg = 0.0, fs = 0.0, ss = 0.0, bad = 2147483647.0;
    for (int r2 = 0; r2 < cs; ++r2) {
      const double* rp = cluster.map_shared_rank(&sm.rpart[0], r2);
      gg += rp[0];
      fs += rp[1];
      ss += rp[2];
      bad = fmin(bad, rp[3]);
    }
    shift = __ddiv_rn(ss, static_cast<double>(red.n_div));
    if (rank == 0 && tid == 0) {
      red.out->grad_norm = sqrt(gg);
      red.out->f_mean = __ddiv_rn(fs, static_cast<double>(red.n_div));
      red.out->shift_mean = shift;
      red.out->xx = sm.rscr[0];
      const int slot = ctl->round - ctl->row_base;
      if (red.row_grad) red.row_grad[slot] = red.out->grad_norm;
      if (red.row_f) red.row_f[slot] = red.out->f_mean;
      if (bad < 2147483647.0) {
        ctl->bad_client = static_cast<int32_t>(bad);
        raise_status(ctl, ST_NONFINITE);
      }
    }
    skip_solve = bad < 2147483647.0;  // the same partials in every CTA: no solve this round
  } else {
    shift = shift_ptr ? __ldcg(shift_ptr) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int q = rank + k * cs;
    if (q >= npan) break;
    const int pb = min(CP_NB, d - q * CP_NB);
    double* Pq = P(k);
    if (tid < pb) Pq[tid * CP_LS + tid] = __dadd_rn(Pq[tid * CP_LS + tid], shift);
  }
  __syncthreads();
  if (tid == 0) tl_mark(7, true);
  // the compressor may start streaming D now (k_wait_reduce): released by a
  // warp that is idle while panel 0 is factored (the fence is cumulative over
  // the reduction's writes this thread observed through the barrier)
  if (fused && rank == 0 && tid == CH_THREADS - 32) {
    __threadfence();
    atomicExch(&ctl->red_gate, ctl->round + 1);
  }
  mark(0);

  // ---- factorisation.  Panel p - 1's owner pushes L_{p-1}'s slots 32..95
  //      into panel p's owner (rcv): rows 0..31 give p's diagonal block its
  //      last update (barLd), rows 32..63 the update of p's head slots
  //      32..63 (barLd2) — the rows whose TRSM p pushes on in turn — so the
  //      chain from factor to factor never waits for an L2 round trip.  The
  //      rest of p's rows take L_{p-1} from its L2 copy (barL), fused with
  //      their TRSM in step B.  cs >= 4 here: consecutive panels always have
  //      different owners.
  for (int p = 0; p < npan && !skip_solve; ++p) {
    const int owner = p % cs, kp = p / cs;
    const int p0 = p * CP_NB;
    if (rank == owner) {
      double* Pp = P(kp);
      const int nreal = d - p0, rs = max(nreal, CP_NB), pb = min(CP_NB, nreal);
      const int t_lo = CP_NB / 8, t_hi = rs / 8;
      // (A) warp 0: diagonal block; warp 1: T = L_pp^-1 alongside; the rest:
      //     the head slots' pending update from the pushed rows
      stamp(p, 0);
      if (warp == 0) {
        // Block factor on the symmetric Schur complement, lane c owning
        // column c (a[r] = S[r][c]).  By symmetry lane c's multiplier
        // S[c][j] is its own a[j], so per pivot only 1/sqrt(S[j][j]) crosses
        // lanes (shared memory, no shuffle); row j of S is published (in the
        // T buffer, which warp 1 overwrites only after reading every row)
        // for the trailing updates and for warp 1.
        double* rows = &sm.T[kp][0][0];
        double a[CP_NB];
#pragma unroll
        for (int r = 0; r < CP_NB; ++r) a[r] = Pp[r * CP_LS + lane];
        double myir = 0.0, mypiv = 0.0;
        rows[lane] = a[0];
        {
          const double y = rsqrt_nr(a[0]);
          if (lane == 0) { sm.inv[0] = y; mypiv = a[0]; }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.barF[0]);
        double ir = sm.inv[0];
#pragma unroll
        for (int j = 0; j < CP_NB; ++j) {
          const double* b = rows + j * CP_LS;
          myir = (lane == j) ? ir : myir;
          const double ir2 = ir * ir;
          const double m = (lane > j) ? a[j] * ir2 : 0.0;  // columns < j are final
          if (j + 1 < CP_NB) {
            a[j + 1] = fma(-m, b[j + 1], a[j + 1]);
            rows[(j + 1) * CP_LS + lane] = a[j + 1];
            const double y = rsqrt_nr(a[j + 1]);
            mypiv = (lane == j + 1) ? a[j + 1] : mypiv;
            if (lane == j + 1) sm.inv[j + 1] = y;
          }
#pragma unroll
          for (int r = j + 2; r < CP_NB; ++r) a[r] = fma(-m, b[r], a[r]);
          __syncwarp();
          if (j + 1 < CP_NB) {
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
            ctl->pivot_index = p0 + fail;
            ctl->pivot_value = fv;
            raise_status(ctl, ST_NOT_PD);
          }
        } else {
#pragma unroll
          for (int r = 0; r < CP_NB; ++r) Pp[r * CP_LS + lane] = (r >= lane) ? a[r] * myir : 0.0;
        }
        mark(3);
        stamp(p, 1);
      } else if (warp == 1) {
        // T = L^-1, right-looking, lane c owning column c, one pivot behind
        // warp 0: t_j = t[j] / L_jj, t[r] -= L[r][j] t_j with L[r][j] = S_j[r] ir_j
        const double* rows = &sm.T[kp][0][0];
        const uint32_t par = static_cast<uint32_t>(fac_uses & 1);
        double t[CP_NB];
#pragma unroll
        for (int r = 0; r < CP_NB; ++r) t[r] = (r == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int j = 0; j < CP_NB; ++j) {
          mbar_wait(&sm.barF[j], par);
          const double irj = sm.inv[j];
          const double u = t[j] * irj * irj;
          t[j] *= irj;
#pragma unroll
          for (int r = j + 1; r < CP_NB; ++r) t[r] = fma(-u, rows[j * CP_LS + r], t[r]);
        }
        __syncwarp();  // every lane's last row read precedes the first T store
#pragma unroll
        for (int r = 0; r < CP_NB; ++r) sm.T[kp][r][lane] = t[r];
      } else if (p > 0 && ((CP_REST_WARPS >> warp) & 1u)) {
        // head slots 32..63: A = L_{p-1} slots 64..95 (rcv rows 32..63),
        // B = L_{p-1} slots 32..63 (rcv rows 0..31)
        mbar_wait_cluster(&sm.barLd2[p - 1], 0);
        cp_update<false>(&sm.rcv[0][0], p - 1, p, Pp, d, CP_NB, min(2 * CP_NB - 1, rs), 1, 8, CP_NB,
                         CP_REST_WARPS);
      }
      __syncthreads();
      ++fac_uses;
      stamp(p, 2);
      mark(4);
      if (sm.failed) {
        // release every waiter with the failure flag set
        if (tid < cs && tid != rank) {
          int* rf = cluster.map_shared_rank(&sm.failed, tid);
          *rf = 1;
          fence_cluster();
          for (int q = p; q < npan; ++q) {
            mbar_arrive_remote(&sm.barL[q], static_cast<uint32_t>(tid));
            // the next owner's barLd / barLd2 wait for transaction bytes
            if (q + 1 < npan && (q + 1) % cs == tid) {
              mbar_complete_tx_remote(mapa_u32(&sm.barLd[q], static_cast<uint32_t>(tid)), cp_push_bytes(d, q, 32));
              mbar_complete_tx_remote(mapa_u32(&sm.barLd2[q], static_cast<uint32_t>(tid)), cp_push_bytes(d, q, 64));
            }
          }
        }
        break;
      }
      // (B) rows below the block: X = A T^T (in place), 8-row tiles.  Warps
      //     0..3 take the head tiles (slots 32..63, already updated), warps
      //     4..7 the next four (slots 64..95: their L_{p-1} update first);
      //     both go to the next owner as st.async stores completing its
      //     barLd / barLd2.  Then every warp takes the remaining tiles, each
      //     updated from L_{p-1}'s L2 copy and solved in one pass.  Every
      //     solved tile is also written to L_p's L2 copy.
      {
        const int nxt_owner = (p + 1) % cs;
        const bool push = !CP_NO_PUSH && p + 1 < npan;
        // the next owner's rcv is free once it finished the panel it last
        // received for (its panel p + 1 - cs)
        if (push && p + 1 >= cs) mbar_wait_cluster(&sm.barRF, 0);
        const uint32_t rcv_r = push ? mapa_u32(&sm.rcv[0][0], static_cast<uint32_t>(nxt_owner)) : 0u;
        const uint32_t bar_r = push ? mapa_u32(&sm.barLd[p], static_cast<uint32_t>(nxt_owner)) : 0u;
        const uint32_t bar2_r = push ? mapa_u32(&sm.barLd2[p], static_cast<uint32_t>(nxt_owner)) : 0u;
        double bt[8][4];
#pragma unroll
        for (int ct = 0; ct < 4; ++ct)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) bt[ks][ct] = sm.T[kp][ct * 8 + (lane >> 2)][ks * 4 + (lane & 3)];
        double* G = (p < npan - 1 && cs > 1) ? Lglob(p) : nullptr;
        const double* Lprev = p > 0 ? Lglob(p - 1) : nullptr;
        const int rs_prev = p > 0 ? max(d - (p - 1) * CP_NB, CP_NB) : 0;
        bool prev_ready = p == 0;
        auto update_from_l2 = [&](int tile) {
          if (p == 0) return;
          if (!prev_ready) {
            mbar_wait_cluster(&sm.barL[p - 1], 0);  // L_{p-1}'s L2 copy
            prev_ready = true;
          }
          cp_tile_update_l2(Lprev, &sm.rcv[0][0], Pp, tile, d, p0, nreal, rs, rs_prev);
          __syncwarp();
        };
        auto do_tile = [&](int tile) {
          const int r = tile * 8 + (lane >> 2);
          const bool ok = r < nreal || r == rs;
          double a[8];
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) a[ks] = ok ? Pp[r * CP_LS + ks * 4 + (lane & 3)] : 0.0;
          double acc[4][2] = {};
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int ct = 0; ct < 4; ++ct) dmma_8x8x4(acc[ct], a[ks], bt[ks][ct]);
          __syncwarp();
          if (ok) {
            const bool to_next = push && r < 3 * CP_NB;
            const uint32_t bar = r < 2 * CP_NB ? bar_r : bar2_r;
#pragma unroll
            for (int ct = 0; ct < 4; ++ct) {
              const int cc = ct * 8 + 2 * (lane & 3);
              const double2 v2 = make_double2(acc[ct][0], acc[ct][1]);
              *reinterpret_cast<double2*>(Pp + r * CP_LS + cc) = v2;
              if (to_next)
                st_async_v2f64(rcv_r + static_cast<uint32_t>(((r - CP_NB) * CP_LS + cc) * 8), bar, v2.x, v2.y);
              if (G) __stcg(reinterpret_cast<double2*>(G + r * CP_LS + cc), v2);
            }
          }
        };
        // the head tiles on all eight warps (column halves: 16 DMMAs each)
        {
          const int tile = t_lo + (warp & 3), h = warp >> 2;
          if (tile <= t_hi) {
            const int r = tile * 8 + (lane >> 2);
            double acc[2][2] = {};
            const bool ok = r < nreal || r == rs;
            double a[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) a[ks] = ok ? Pp[r * CP_LS + ks * 4 + (lane & 3)] : 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
#pragma unroll
              for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[j], a[ks], h ? bt[ks][2 + j] : bt[ks][j]);
            asm volatile("bar.sync 1, 256;" ::: "memory");  // both halves read the rows first
            if (ok) {
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int cc = (2 * h + j) * 8 + 2 * (lane & 3);
                const double2 v2 = make_double2(acc[j][0], acc[j][1]);
                *reinterpret_cast<double2*>(Pp + r * CP_LS + cc) = v2;
                if (push) st_async_v2f64(rcv_r + static_cast<uint32_t>(((r - CP_NB) * CP_LS + cc) * 8), bar_r, v2.x, v2.y);
                if (G) __stcg(reinterpret_cast<double2*>(G + r * CP_LS + cc), v2);
              }
            }
          } else {
            asm volatile("bar.sync 1, 256;" ::: "memory");
          }
          stamp(p, 3);
        }
        if (warp >= 4) {
          const int tile = t_lo + warp;  // slots 64 + 8 (warp - 4) ..
          if (tile <= t_hi) {
            update_from_l2(tile);
            do_tile(tile);
          }
          stamp_w(p, 5, 4);
        }
        for (int t2 = t_lo + 8 + warp; t2 <= t_hi; t2 += 8) {
          update_from_l2(t2);
          do_tile(t2);
        }
        stamp(p, 6);
        stamp_w(p, 7, 4);
      }
      __syncthreads();
      stamp(p, 4);
      mark(5);
      // release L_p's L2 copy (the CTA barrier orders every warp's stores
      // before thread 0's cluster-scope release)
      if (tid == 0) {
        if (p < npan - 1 && cs > 1)
          for (int r2 = 0; r2 < cs; ++r2)
            if (r2 != rank && r2 + ((npan - 1 - r2) / cs) * cs > p)  // r2 owns a later panel
              mbar_arrive_remote(&sm.barL[p], static_cast<uint32_t>(r2));
        // rcv is no longer needed: its next push (for panel p + cs) may come
        if (p + cs < npan)
          mbar_arrive_remote(&sm.barRF, static_cast<uint32_t>((p + cs - 1) % cs));
      }
      mark(6);
      stamp(p, 14);
      // updates from L_{p-1} deferred by the lookahead (own panels after p)
      if (p > 0 && last_own > p) {
        const int pp = p - 1;
        mbar_wait_cluster(&sm.barL[pp], 0);  // (complete: re-checked per warp)
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int q = rank + k * cs;
          if (q <= p || q >= npan) continue;
          const int rs_q = max(d - q * CP_NB, CP_NB);
          cp_update<true>(Lglob(pp), pp, q, P(k), d, 0, rs_q, 0, 8);
          for (uint32_t m = pend[k]; m; m &= m - 1) {
            const int pq = __ffs(m) - 1;
            cp_update<true>(Lglob(pq), pq, q, P(k), d, 0, rs_q, 0, 8);
          }
          pend[k] = 0u;
        }
        __syncthreads();
      }
      stamp(p, 15);
    } else if (last_own > p) {
      if (!CP_NO_PUSH && (p + 1) % cs == rank) {
        // our panel is next: its diagonal rows from the pushed rows of L_p
        mbar_wait_cluster(&sm.barLd[p], 0);
        if (sm.failed) break;
        cp_update_diag8(&sm.rcv[0][0], P((p + 1) / cs), d, (p + 1) * CP_NB, d - (p + 1) * CP_NB);
        __syncthreads();
      } else {
        mbar_wait_cluster(&sm.barL[p], 0);
      }
      mark(7);
      if (sm.failed) break;
    }
    // apply L_p to the own panels after p.  Lookahead: if the next panel is
    // ours, its diagonal rows were updated from the push above and its other
    // rows follow in its own steps A / B; the other own panels' updates are
    // deferred until that panel is factored and released.
    // Two panels before the next own panel, the other own panels' updates
    // are owed (pend) until after that panel's step B: this CTA must be free
    // when the next panel's diagonal rows arrive.
    const bool next_mine = p + 1 < npan && (p + 1) % cs == rank;
    const int nq = rank > p ? rank : rank + cs;  // next own panel
    const bool urgent = rank != owner && nq == p + 2 && nq < npan;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int q = rank + k * cs;
      if (q <= p || q >= npan) continue;
      if (next_mine) continue;
      if (urgent && q != nq) {
        pend[k] |= 1u << p;
        continue;
      }
      const int rs_q = max(d - q * CP_NB, CP_NB);
      if (rank == owner)
        cp_update<false>(P(kp), p, q, P(k), d, 0, rs_q, 0, 8);
      else
        cp_update<true>(Lglob(p), p, q, P(k), d, 0, rs_q, 0, 8);
    }
    __syncthreads();
    mark(8);
  }
  mark(1);
  if (tid == 0) tl_mark(8, true);
  if (rank == 0) stamp(63, 0);
  cluster.sync();  // failure flags settled cluster-wide
  if (rank == 0) stamp(63, 1);
  if (!sm.failed && !skip_solve) {
    // ---- backward substitution: L^T z = y, panel by panel from the last.
    //      Warp k runs own panel q_k = rank + k cs alone: for every later
    //      panel b it waits for z_b (barZ[b]: st.async bytes from b's owner,
    //      or the local arrive of the warp owning b) and accumulates
    //      w = sum_b L_{q_k}[rows b]^T z_b; then z_{q_k} = T^T (y - w) goes to
    //      the earlier CTAs as st.async stores.  No CTA-wide barrier per panel.
    if (warp < KP && rank + warp * cs < npan) {
      const int k = warp, q = rank + k * cs, q0 = q * CP_NB;
      const double* Pq = P(k);
      double wacc = 0.0;
      for (int b = npan - 1; b > q; --b) {
        const int b0 = b * CP_NB, bn = min(CP_NB, d - b0);
        mbar_wait_cluster(&sm.barZ[b], 0);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
        for (int i = 0; i < CP_NB; ++i)
          if (i < bn) acc[i & 3] = fma(Pq[(b0 + i - q0) * CP_LS + lane], sm.z[b0 + i], acc[i & 3]);
        wacc += (acc[0] + acc[1]) + (acc[2] + acc[3]);
      }
      const int bn = min(CP_NB, d - q0), rs = max(d - q0, CP_NB);
      // r_t = y_t - w_t;  z_s = sum_{t >= s} T[t][s] r_t
      sm.part[warp][lane] = (lane < bn) ? __dsub_rn(Pq[rs * CP_LS + lane], wacc) : 0.0;
      __syncwarp();
      double zacc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
      for (int t2 = 0; t2 < CP_NB; ++t2)
        if (t2 >= lane) zacc[t2 & 3] = fma(sm.T[k][t2][lane], sm.part[warp][t2], zacc[t2 & 3]);
      const double zs = (zacc[0] + zacc[1]) + (zacc[2] + zacc[3]);
      stamp_if(lane == 0, q, 10);
      if (lane < bn) {
        sm.z[q0 + lane] = zs;
        for (int r2 = 0; r2 < cs; ++r2)  // CTAs owning a panel before q
          if (r2 != rank && r2 < q) st_async_f64(&sm.z[q0 + lane], &sm.barZ[q], static_cast<uint32_t>(r2), zs);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.barZ[q]);  // this CTA's other warp (an earlier own panel)
      stamp_if(lane == 0, q, 11);
    }
    __syncthreads();
    mark(2);
    if (rank == 0) stamp(63, 2);
    // ---- outputs of the own panels
    if (ignore_halt || !ctl->halt) {
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int q = rank + k * cs;
        if (q >= npan) break;
        const int q0 = q * CP_NB, bn = min(CP_NB, d - q0);
        if (tid < bn) {
          const int i = q0 + tid;
          const double zi = sm.z[i];
          z[i] = zi;
          if (mode == 0) x_out[i] = __dsub_rn(__ldcg(x + i), zi);
          else if (mode == 1) x_out[i] = zi;
        }
      }
    }
  }
  cluster.sync();  // no CTA leaves while its shared memory may be addressed
  if (tid == 0) tl_mark(2, true);
  if (stamping)
    for (int i = tid; i < (CP_MAXP + 1) * 16; i += CH_THREADS) {
      const int row = i / 16, k = i % 16;
      if (!stamps[i]) continue;
      if (dbg) dbg[16 + (row < CP_MAXP ? row : 63) * 16 + k] = stamps[i];
      else g_dbg_cta[(row < CP_MAXP ? row : 63) * 16 + k] = stamps[i];
    }
}

}  // namespace fb
