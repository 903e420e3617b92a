// hessian_dmma.cuh — batched upper-triangular Hessian on fp64 tensor cores,
// fused with the FedNL shift difference (reference oracle.py:124-139,
// algorithms.py:228-231, linalg.py:139-148).
//
// For every client c and every 64x64 tile pair (I <= J) of its upper
// triangle:
//     S[a][b] = sum_j Bt[c][a][j] * h_c[j] * Bt[c][b][j]      (DMMA.8x8x4)
//     H       = S (+ lam on the diagonal)
//     D[c][t] = H - Hest[c][t]            packed t = b(b+1)/2 + a, a <= b
//     frob_part[c][pair] = sum wt * D^2   (wt = 1 diagonal, 2 off-diagonal)
//     flags[c] |= 1 (non-finite D) | 2 (nonzero D)
// Optionally H itself is written (`hess_out`, FedNL-PP / exact init).
//
// Operands are staged by TMA: box {16 samples, 64 features} per operand and
// stage, SWIZZLE_128B, NSTAGE-deep mbarrier ring; the h chunk rides on the
// same barrier as a 128 B bulk copy.  Each of the 4 warps owns a 32x32
// quadrant as 4x4 m8n8k4 fragments (32 fp64 accumulators per thread).  The
// A fragment is scaled by h_j in registers (one DMUL per 16 DMMA).
#pragma once
#include "common.cuh"

namespace fb {

constexpr int HT = 64;          // tile edge (features)
constexpr int HKC = 16;         // samples per stage (128 B rows)
constexpr int HSTAGE = 4;       // pipeline depth
constexpr int HCONS = 4;        // consumer (DMMA) warps, one 32x32 quadrant each
constexpr int HTHREADS = (HCONS + 1) * 32;  // + one TMA producer warp
constexpr int HC_LD = HT + 1;   // epilogue staging pitch

struct HessSmem {
  double a[HSTAGE][HT * HKC];  // 8 KB per stage, 1024 B aligned (swizzle-128B)
  double b[HSTAGE][HT * HKC];
  double h[HSTAGE][HKC];
  double gc[HSTAGE][HKC];      // gradient coefficients (fused gradient, diagonal tiles)
  uint64_t full[HSTAGE];       // TMA -> consumers (transaction count)
  uint64_t empty[HSTAGE];      // consumers -> producer (one arrive per active warp)
  double red[HTHREADS / 32];
  int flag_or;
};
constexpr size_t HESS_SMEM = sizeof(HessSmem) + 1024;  // + alignment slack

// The consumers hand a ring slot back to the TMA with an mbarrier arrive
// whose address depends (through `zero_mask`: a kernel argument that is 0 at
// run time but unknown to ptxas) on every fragment value the warp loaded
// from the slot.  Without that dependency ptxas hoists the arrive above the
// stage's last fragment loads, and the next TMA fill of the slot races them.
__device__ __forceinline__ void mbar_arrive_dep(uint64_t* bar, uint32_t dep, uint32_t zero_mask) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar) + (dep & zero_mask))
               : "memory");
}
__device__ __forceinline__ uint32_t dep_of(double v) {
  return static_cast<uint32_t>(__double2hiint(v));
}

// element (r, s) of a [64 rows][16 doubles] SWIZZLE_128B tile, in doubles
__device__ __forceinline__ int swz(int r, int s) {
  return r * HKC + ((((s >> 1) ^ (r & 7)) << 1) | (s & 1));
}


// One consumer warp's mainloop over all K-chunks, specialised at compile time
// for its 32x32 quadrant: MR x NC valid 8x8 fragments (rows / columns past d
// in the last tile are skipped, rounded up to 2 or 4) and TRI = a diagonal
// quadrant, whose fragments strictly below the diagonal are skipped.  No
// runtime branch sits between the DMMAs.
template <int MR, int NC, bool TRI>
__device__ __forceinline__ void hess_consume(HessSmem& sm, bool diag, int nk, int rowbase,
                                             int colbase, int g, int t, int lane,
                                             uint32_t zero_mask, double (&acc)[4][4][2]) {
  for (int it = 0; it < nk; ++it) {
    const int s2 = it % HSTAGE;
    mbar_wait(&sm.full[s2], (it / HSTAGE) & 1);
    const double* sa = sm.a[s2];
    const double* sb = diag ? sm.a[s2] : sm.b[s2];
    uint32_t ldep = 0;  // every value loaded from the slot feeds the release
#pragma unroll
    for (int kk = 0; kk < HKC / 4; ++kk) {
      // k-step kk reads samples {2kk, 2kk+1, 2kk+8, 2kk+9}: with the 128B
      // swizzle every half-warp then touches 16 distinct bank pairs
      const int ks = 2 * kk + (t & 1) + 8 * (t >> 1);
      const double hv = sm.h[s2][ks];
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < MR; ++mi) af[mi] = sa[swz(rowbase + 8 * mi + g, ks)] * hv;
#pragma unroll
      for (int nj = 0; nj < NC; ++nj) bf[nj] = sb[swz(colbase + 8 * nj + g, ks)];
#pragma unroll
      for (int q = 0; q < MR; ++q) ldep ^= dep_of(af[q]);
#pragma unroll
      for (int q = 0; q < NC; ++q) ldep ^= dep_of(bf[q]);
#pragma unroll
      for (int mi = 0; mi < MR; ++mi)
#pragma unroll
        for (int nj = 0; nj < NC; ++nj)
          if (!TRI || mi <= nj) dmma_8x8x4(acc[mi][nj], af[mi], bf[nj]);
    }
    // release the slot once every fragment load of this stage completed
    if (lane == 0) mbar_arrive_dep(&sm.empty[s2], ldep, zero_mask);
  }
}

// grid (n_pairs, n_active), block HTHREADS, dynamic smem HESS_SMEM.
// Warps 0..3 compute (warp q owns quadrant rows 32*(q&1), cols 32*(q>>1));
// warp 4 is the TMA producer.  Stage s is refilled once every active
// consumer warp has arrived on empty[s] (no CTA-wide barrier per stage).
// MINB = CTAs per SM the register budget is cut for (2 is used).
template <int MINB>
__global__ void __launch_bounds__(HTHREADS, MINB) k_hessian(
    const __grid_constant__ CUtensorMap tmap_b, const DevCtl* __restrict__ ctl, int d,
    const int32_t* __restrict__ ni_arr, int ldh, const double* __restrict__ hcoef,
    const double* __restrict__ lam_arr, const int32_t* __restrict__ clients,
    const double* __restrict__ hest, int64_t hest_stride, double* __restrict__ D,
    double* __restrict__ hess_out, double* __restrict__ frob_part, int32_t* __restrict__ flags,
    uint32_t zero_mask, const double* __restrict__ gcoef, const double* __restrict__ x,
    double* __restrict__ grad, const int32_t* __restrict__ pair_order, int n_pairs_arg, int grp,
    const int32_t* __restrict__ dispatch) {
  // the round reduction may launch now (it waits for this pass)
  asm volatile("griddepcontrol.launch_dependents;");
  if (ctl && ctl->halt) return;
  extern __shared__ uint8_t smem_raw[];
  HessSmem& sm = *reinterpret_cast<HessSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));

  // 1-D grid over (client group, pair, client): groups of `grp` clients in
  // order (a group's B rows stay in L2 while its tiles run); inside a group
  // the tile pairs go costliest first (`pair_order`), so every wave — the
  // last one included — ends on the cheap diagonal / edge tiles
  const int n_pairs = n_pairs_arg;
  const int n_act = static_cast<int>(gridDim.x) / n_pairs;
  const int L = blockIdx.x;
  const int g0 = (L / (grp * n_pairs)) * grp;  // first client of the group
  const int gs = min(grp, n_act - g0);
  const int rem = L - g0 * n_pairs;
  int slot = g0 + rem % gs;
  int pair = pair_order[rem / gs];
  if (dispatch) {  // explicit (pair << 16 | client slot) per CTA
    const int v = dispatch[L];
    slot = v & 0xFFFF;
    pair = v >> 16;
  }
  const int c = client_of(clients, slot);
  // pair -> (I, J), I <= J, column-wise like the packed layout
  int J = static_cast<int>((sqrtf(8.0f * pair + 1.0f) - 1.0f) * 0.5f);
  while ((J + 1) * (J + 2) / 2 <= pair) ++J;
  while (J * (J + 1) / 2 > pair) --J;
  const int I = pair - J * (J + 1) / 2;
  const bool diag = (I == J);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int rowbase = 32 * (warp & 1), colbase = 32 * (warp >> 1);
  // on a diagonal tile the lower-left quadrant is entirely below the diagonal;
  // with `grad` set that warp computes the local gradient of the tile's 64
  // features from the same stages instead (oracle.py:108-121, fused: B is
  // streamed once for the Hessian and the gradient)
  const bool fuse_grad = diag && grad != nullptr;
  const int n_active_warps = (diag && !fuse_grad) ? HCONS - 1 : HCONS;
  const bool consumer = warp < HCONS && !(diag && rowbase > colbase);
  const bool grad_warp = fuse_grad && warp < HCONS && rowbase > colbase;

  const int nk = (ni_arr[c] + HKC - 1) / HKC;  // this client's samples (ragged shards)
  const double lam = lam_arr[c];
  const double* hrow = hcoef + static_cast<int64_t>(c) * ldh;
  const double* grow = fuse_grad ? gcoef + static_cast<int64_t>(c) * ldh : nullptr;
  const uint32_t stage_bytes =
      (diag ? 1u : 2u) * HT * HKC * 8u + HKC * 8u + (fuse_grad ? HKC * 8u : 0u);

  const long long t_start = clock64();
  if (tid == 0) {
    tma_prefetch_desc(&tmap_b);
    for (int s2 = 0; s2 < HSTAGE; ++s2) {
      mbar_init(&sm.full[s2], 1);
      mbar_init(&sm.empty[s2], n_active_warps);
    }
    fence_barrier_init();
    sm.flag_or = 0;
  }
  __syncthreads();

  double acc[4][4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 4; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;

  if (warp == HCONS) {
    // ---------------- TMA producer
    if (lane == 0) {
      // programmatic dependent launch: the margins kernel's coefficients
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int it = 0; it < nk; ++it) {
        const int s2 = it % HSTAGE;
        if (it >= HSTAGE) mbar_wait(&sm.empty[s2], ((it / HSTAGE) - 1) & 1);
        mbar_arrive_expect_tx(&sm.full[s2], stage_bytes);
        tma_load_3d(sm.a[s2], &tmap_b, &sm.full[s2], it * HKC, I * HT, c);
        if (!diag) tma_load_3d(sm.b[s2], &tmap_b, &sm.full[s2], it * HKC, J * HT, c);
        bulk_load(sm.h[s2], hrow + it * HKC, HKC * 8, &sm.full[s2]);
        if (fuse_grad) bulk_load(sm.gc[s2], grow + it * HKC, HKC * 8, &sm.full[s2]);
      }
    }
  } else if (grad_warp) {
    // ---------------- fused gradient: lane owns features r = lane, lane + 32
    double g0 = 0.0, g1 = 0.0;
    for (int it = 0; it < nk; ++it) {
      const int s2 = it % HSTAGE;
      mbar_wait(&sm.full[s2], (it / HSTAGE) & 1);
      const double* sa = sm.a[s2];
      uint32_t ldep = 0;
#pragma unroll
      for (int k2 = 0; k2 < HKC; ++k2) {
        const double gk = sm.gc[s2][k2];
        const double v0 = sa[swz(lane, k2)], v1 = sa[swz(lane + 32, k2)];
        ldep ^= dep_of(v0) ^ dep_of(v1) ^ dep_of(gk);
        g0 = fma(v0, gk, g0);
        g1 = fma(v1, gk, g1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_dep(&sm.empty[s2], ldep, zero_mask);
    }
    const double* xc = x;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int a = I * HT + lane + 32 * h2;
      if (a < d)
        grad[static_cast<int64_t>(c) * d + a] = __dadd_rn(h2 ? g1 : g0, __dmul_rn(lam, xc[a]));
    }
  } else if (consumer) {
    // ---------------- DMMA consumers, specialised per quadrant shape
    const int vr = (d - (I * HT + rowbase) + 7) / 8, vc = (d - (J * HT + colbase) + 7) / 8;
    const int mr = vr >= 3 ? 4 : 2, nc = vc >= 3 ? 4 : 2;  // vr, vc >= 1 for an active quadrant
    const bool tri = diag && rowbase == colbase;
    if (tri) {
      if (mr == 4) hess_consume<4, 4, true>(sm, diag, nk, rowbase, colbase, g, t, lane, zero_mask, acc);
      else hess_consume<2, 2, true>(sm, diag, nk, rowbase, colbase, g, t, lane, zero_mask, acc);
    } else if (mr == 4 && nc == 4) {
      hess_consume<4, 4, false>(sm, diag, nk, rowbase, colbase, g, t, lane, zero_mask, acc);
    } else if (mr == 4) {
      hess_consume<4, 2, false>(sm, diag, nk, rowbase, colbase, g, t, lane, zero_mask, acc);
    } else if (nc == 4) {
      hess_consume<2, 4, false>(sm, diag, nk, rowbase, colbase, g, t, lane, zero_mask, acc);
    } else {
      hess_consume<2, 2, false>(sm, diag, nk, rowbase, colbase, g, t, lane, zero_mask, acc);
    }
  }
  __syncthreads();  // all stages consumed; the ring is free for the epilogue
  const long long t_main = clock64();

  // ---- epilogue: stage the tile column-major, then stream packed columns
  double* cs = &sm.a[0][0];  // [64 cols][HC_LD] — reuses the pipeline ring
  if (consumer) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int nj = 0; nj < 4; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = rowbase + 8 * mi + g;
          const int col = colbase + 8 * nj + 2 * t + e;
          cs[col * HC_LD + r] = acc[mi][nj][e];
        }
  }
  __syncthreads();

  const double* hest_c = hest + static_cast<int64_t>(c) * hest_stride;
  const int64_t w = packed_len(d);
  double* Dc = D + static_cast<int64_t>(c) * w;
  double* Hc = hess_out ? hess_out + static_cast<int64_t>(slot) * w : nullptr;
  double part = 0.0;
  int fl = 0;
  // every warp (producer included) streams columns col = warp, warp + 5, ...;
  // the H_i^k operands of all its (column, row) pairs are loaded first so
  // the global-memory latency is paid once per warp, not once per column
  constexpr int NW = HTHREADS / 32;
  constexpr int MAXC = (HT + NW - 1) / NW;  // columns per warp
  double hk[MAXC][2];
#pragma unroll
  for (int q = 0; q < MAXC; ++q) {
    const int col = warp + q * NW;
    const int b = J * HT + col;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int a = I * HT + lane + 32 * h2;
      const bool ok = col < HT && b < d && a <= b && a < d;
      hk[q][h2] = ok ? __ldg(hest_c + packed_at(a, b)) : 0.0;
    }
  }
#pragma unroll
  for (int q = 0; q < MAXC; ++q) {
    const int col = warp + q * NW;
    const int b = J * HT + col;
    if (col >= HT || b >= d) continue;
    const int64_t cbase = packed_at(0, b);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int r = lane + 32 * h2;
      const int a = I * HT + r;
      if (a > b || a >= d) continue;
      const int64_t tt = cbase + a;
      double hv = cs[col * HC_LD + r];
      if (a == b) hv = __dadd_rn(hv, lam);
      const double dv = __dsub_rn(hv, hk[q][h2]);
      Dc[tt] = dv;
      if (Hc) Hc[tt] = hv;
      const double wt = (a == b) ? 1.0 : 2.0;
      part = fma(__dmul_rn(wt, dv), dv, part);
      if (!isfinite(dv)) fl |= 1;
      if (dv != 0.0) fl |= 2;
    }
  }
  const double tot = block_sum(part, sm.red);
  if (fl) atomicOr(&sm.flag_or, fl);
  __syncthreads();
  if (tid == 0) {
    frob_part[static_cast<int64_t>(c) * n_pairs + pair] = tot;
    if (sm.flag_or) atomicOr(&flags[c], sm.flag_or);
    if (g_dbg_on) {  // diagnostics: CTA-summed mainloop / epilogue cycles
      const long long t_end = clock64();
      atomicAdd(reinterpret_cast<unsigned long long*>(&g_dbg[20]), static_cast<unsigned long long>(t_main - t_start));
      atomicAdd(reinterpret_cast<unsigned long long*>(&g_dbg[21]), static_cast<unsigned long long>(t_end - t_main));
      atomicAdd(reinterpret_cast<unsigned long long*>(&g_dbg[22]), 1ull);
    }
  }
}

}  // namespace fb
