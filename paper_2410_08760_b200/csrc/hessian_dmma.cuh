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
// stage, SWIZZLE_128B, HW_STAGE-deep mbarrier ring; the h chunk rides on the
// same barrier as a 128 B bulk copy.  A tile's 8x8 fragments (m8n8k4 DMMA)
// are split between four warps in balanced blocks of up to 4x4 (32 fp64
// accumulators per thread); the A fragment is scaled by h_j in registers.
#pragma once
#include "common.cuh"

namespace fb {

constexpr int HT = 64;          // tile edge (features)
constexpr int HKC = 16;         // samples per stage (128 B rows)


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


// ===================================================================
// Persistent, warp-specialised variant (the production kernel).
//
// A one-tile-per-CTA kernel (round 1) paid, per 64x64 tile, the TMA pipeline
// fill and an epilogue (stage -> H_i^k loads -> D / Frobenius) during which
// its DMMA warps idle.  Here one CTA per SM runs two independent tile
// pipes, each with its own stage ring and hand-off buffer, and every pipe
// loops over tiles (items) with its roles running concurrently:
//   4 DMMA warps   the current item (on a diagonal tile the lower-left warp
//                  forms the fused local gradient), then hand the
//                  accumulators to the epilogue through `cs` and go on;
//   1 TMA warp     streams the stages of item j+1 while the DMMA warps
//                  finish item j (the ring never drains between items);
//   1 epilogue     item j-1: H_i^k loads, D in packed column segments, the
//     warp         Frobenius partial and the flags.
// Two pipes per CTA (not two CTAs per SM) so that the DMMA warps get 168
// registers (a whole stage's fragments in flight) under one launch bound.
// Items are (client slot, tile pair) in the order of the one-tile grid
// (client groups, costliest tile pairs first); a pipe's producer claims the
// next one with an atomic ticket and publishes it to its DMMA and epilogue
// warps through a small queue in shared memory (the stage barrier it arms
// next orders the write), so the pipes stay balanced to the last item.  The
// hand-off pitch 66 makes the accumulator stores conflict-free.
constexpr int HW_PIPES = 2;
constexpr int HW_MMA = 4;  // DMMA warps per pipe
constexpr int HW_THREADS = HW_PIPES * (HW_MMA + 2) * 32;
constexpr int HW_LD = HT + 2;
constexpr int HW_STAGE = 4;
// the producer runs at most HW_STAGE items ahead of the DMMA warps, which
// run at most one item ahead of the epilogue: a queue of 16 never wraps
constexpr int HW_QUEUE = 16;

struct __align__(1024) HwPipe {
  double a[HW_STAGE][HT * HKC];  // 1024 B aligned (swizzle-128B)
  double b[HW_STAGE][HT * HKC];
  double h[HW_STAGE][HKC];
  double gc[HW_STAGE][HKC];
  double cs[HT * HW_LD];         // accumulator hand-off (column-major, pitch HW_LD)
  uint64_t full[HW_STAGE];
  uint64_t empty[HW_STAGE];
  uint64_t cs_full;              // 4 DMMA warps -> epilogue warp
  uint64_t cs_empty;             // epilogue warp -> DMMA warps
  int32_t itemq[HW_QUEUE];       // claimed item of the pipe's j-th tile (-1: no more)
  int32_t solo_item;             // solo mode: the tile the pipe's five warps finish together
  double solo_part[HW_MMA + 1];  // solo mode: per-warp Frobenius partials (summed in warp order)
};
constexpr size_t HESS_WS_SMEM = HW_PIPES * sizeof(HwPipe) + 1024;

struct HwItem {
  int slot, c, pair, I, J, nk;
  bool diag;
};
__device__ __forceinline__ HwItem hw_item(int L, int n_pairs, int n_act, int grp,
                                          const int32_t* __restrict__ pair_order,
                                          const int32_t* __restrict__ clients,
                                          const int32_t* __restrict__ ni_arr) {
  HwItem it;
  const int g0 = (L / (grp * n_pairs)) * grp;  // first client of the group
  const int gs = min(grp, n_act - g0);
  const int rem = L - g0 * n_pairs;
  it.slot = g0 + rem % gs;
  it.pair = pair_order[rem / gs];
  it.c = client_of(clients, it.slot);
  int J = static_cast<int>((sqrtf(8.0f * it.pair + 1.0f) - 1.0f) * 0.5f);
  while ((J + 1) * (J + 2) / 2 <= it.pair) ++J;
  while (J * (J + 1) / 2 > it.pair) --J;
  it.J = J;
  it.I = it.pair - J * (J + 1) / 2;
  it.diag = it.I == J;
  it.nk = (ni_arr[it.c] + HKC - 1) / HKC;
  return it;
}

// One DMMA warp's mainloop of one item over the pipe's global stages
// [g0, g0 + nk): its task is the MR x NC block of 8x8 fragments at fragment
// row r0, column c0 (TRI: only the fragments on or above the diagonal).
// GRAD: also the fused local gradient of the block's rows from the same A
// values (before their h scaling): gpart[mi] accumulates row 8(r0+mi)+g over
// this lane's samples; the 4 lanes of a row are summed at the end.
template <int MR, int NC, bool TRI, bool GRAD>
__device__ __forceinline__ void hw_consume(HwPipe& sm, bool diag, int nk, int g0, int r0, int c0,
                                           int g, int t, int lane, uint32_t zero_mask,
                                           double (&acc)[4][4][2], double (&gpart)[4]) {
  for (int it = 0; it < nk; ++it) {
    const int gsn = g0 + it;
    const int s2 = gsn % HW_STAGE;
    mbar_wait(&sm.full[s2], (gsn / HW_STAGE) & 1);
    const double* sa = sm.a[s2];
    const double* sb = diag ? sm.a[s2] : sm.b[s2];
    uint32_t ldep = 0;
#pragma unroll
    for (int kk = 0; kk < HKC / 4; ++kk) {
      const int ks = 2 * kk + (t & 1) + 8 * (t >> 1);
      const double hv = sm.h[s2][ks];
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < MR; ++mi) {
        const double raw = sa[swz(8 * (r0 + mi) + g, ks)];
        if (GRAD) gpart[mi] = fma(raw, sm.gc[s2][ks], gpart[mi]);
        af[mi] = raw * hv;
      }
#pragma unroll
      for (int nj = 0; nj < NC; ++nj) bf[nj] = sb[swz(8 * (c0 + nj) + g, ks)];
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
    if (lane == 0) mbar_arrive_dep(&sm.empty[s2], ldep, zero_mask);
  }
}

// the (MR, NC, TRI, GRAD) instantiation of a task (MR, NC in 1..4)
template <bool TRI, bool GRAD>
__device__ __forceinline__ void hw_consume_any(int mr, int nc, HwPipe& sm, bool diag, int nk, int g0,
                                               int r0, int c0, int g, int t, int lane,
                                               uint32_t zero_mask, double (&acc)[4][4][2],
                                               double (&gpart)[4]) {
#define HW_CASE(M, N)                                                                          \
  case (M) * 8 + (N):                                                                          \
    hw_consume<M, N, TRI, GRAD>(sm, diag, nk, g0, r0, c0, g, t, lane, zero_mask, acc, gpart); \
    break;
  if (TRI) {
    switch (mr * 9) {  // square blocks only
      HW_CASE(1, 1) HW_CASE(2, 2) HW_CASE(3, 3) HW_CASE(4, 4)
    }
  } else {
    switch (mr * 8 + nc) {
      HW_CASE(1, 1) HW_CASE(1, 2) HW_CASE(1, 3) HW_CASE(1, 4)
      HW_CASE(2, 1) HW_CASE(2, 2) HW_CASE(2, 3) HW_CASE(2, 4)
      HW_CASE(3, 1) HW_CASE(3, 2) HW_CASE(3, 3) HW_CASE(3, 4)
      HW_CASE(4, 1) HW_CASE(4, 2) HW_CASE(4, 3) HW_CASE(4, 4)
    }
  }
#undef HW_CASE
}

// The fragment task of DMMA warp q (0..3) of an item, balanced so that the
// four warps — one per SM sub-partition, whose DMMA pipes are separate —
// carry equal shares (an edge or diagonal tile otherwise leaves one pipe
// idle and another full).  nv = valid 8-row fragments of the tile's rows
// (diagonal) or columns (off-diagonal).
//   diagonal:     t1 = ceil(nv / 2): q0 = tri [0, t1), q3 = tri [t1, nv),
//                 q1 / q2 = the rectangle rows [0, t1) x cols [t1, nv),
//                 split by columns; q0 and q3 also form the gradient
//   off-diagonal: rows 0..3 / 4..7 (q0, q1 | q2, q3) x cols split at
//                 ceil(nv / 2)
struct HwTask {
  int r0, c0, mr, nc;
  bool tri, grad;
};
__device__ __forceinline__ HwTask hw_task(int q, bool diag, int nv) {
  HwTask k;
  k.tri = false;
  k.grad = false;
  if (diag) {
    const int t1 = (nv + 1) / 2, t2 = nv - t1;
    const int ca = (t2 + 1) / 2, cb = t2 - ca;
    if (q == 0) { k.r0 = 0; k.c0 = 0; k.mr = t1; k.nc = t1; k.tri = true; k.grad = true; }
    else if (q == 3) { k.r0 = t1; k.c0 = t1; k.mr = t2; k.nc = t2; k.tri = true; k.grad = true; }
    else if (q == 1) { k.r0 = 0; k.c0 = t1; k.mr = t1; k.nc = ca; }
    else { k.r0 = 0; k.c0 = t1 + ca; k.mr = t1; k.nc = cb; }
  } else {
    const int ca = (nv + 1) / 2;
    k.r0 = (q & 1) * 4;
    k.mr = 4;
    k.c0 = (q >> 1) ? ca : 0;
    k.nc = (q >> 1) ? nv - ca : ca;
  }
  return k;
}

// release a pipe's stages [g0, g0 + nk) without reading them
__device__ __forceinline__ void hw_skip(HwPipe& sm, int nk, int g0, int lane) {
  for (int it = 0; it < nk; ++it) {
    const int gsn = g0 + it, s2 = gsn % HW_STAGE;
    mbar_wait(&sm.full[s2], (gsn / HW_STAGE) & 1);
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s2]);
  }
}

// The epilogue of a tile over columns c0, c0 + step, ... (the epilogue warp
// alone: 0, 1; in solo mode each of the pipe's five warps: r, 5): D = H (+ lam
// on the diagonal) - H_i^k in packed column segments (H too when
// requested); returns the warp's Frobenius partial (all lanes), ORs flags.
// H_i^k operands are loaded 8 columns at a time, the next 8 in flight.
//
// The FP64 pipe is the DMMA pipe: every DADD / DMUL here waits behind the
// DMMA warps' issue, and one warp runs a whole tile's epilogue, so the loop is
// kept to two FP64 instructions per element (the difference, one FMA into
// the Frobenius partial) and a few integer ones.  On a diagonal tile lam is
// first added to this warp's diagonal entries of `cs` (column c of the tile
// holds (c, c) at row c); every term is weighted 2 in the loop and the
// diagonal terms' surplus is taken back after it.  Flags: non-finite iff the
// largest |high word| reaches the exponent mask; nonzero iff any bit of
// |dv| is set (so -0.0 counts as zero, NaN as nonzero, like dv != 0.0).
template <bool DIAG>
__device__ __forceinline__ double hw_epi_body(HwPipe& sm, const HwItem& itm, int c0, int step, int nmine, int ncol,
                                              const double* __restrict__ hest_c, double* __restrict__ Dc,
                                              double* __restrict__ Hc, double lam, int lane, uint32_t& hmax,
                                              uint32_t& nzb) {
  constexpr int ECH = 8;  // columns per chunk: 16 loads in flight per lane
  const int a0 = itm.I * HT + lane;
  double hk[ECH][2];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int q = 0; q < ECH; ++q) {
      const int col = c0 + (k0 + q) * step, b = itm.J * HT + col;
      const int cb = b * (b + 1) / 2;  // packed column start (< 2^31 for d <= 46340)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int a = a0 + 32 * h2;
        hk[q][h2] = (col < ncol && (!DIAG || a <= b)) ? __ldcs(hest_c + cb + a) : 0.0;
      }
    }
  };
  if (DIAG) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int cc = lane + 32 * h2;
      if (cc < ncol && cc >= c0 && (cc - c0) % step == 0)
        sm.cs[cc * HW_LD + cc] = __dadd_rn(sm.cs[cc * HW_LD + cc], lam);
    }
    __syncwarp();
  }
  load_chunk(0);
  double po = 0.0;
  for (int k0 = 0; k0 < nmine; k0 += ECH) {
    double hv[ECH][2];
#pragma unroll
    for (int q = 0; q < ECH; ++q) {
      const int col = min(c0 + (k0 + q) * step, HT - 1);
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) hv[q][h2] = sm.cs[col * HW_LD + lane + 32 * h2];
    }
    double hkc[ECH][2];
#pragma unroll
    for (int q = 0; q < ECH; ++q) hkc[q][0] = hk[q][0], hkc[q][1] = hk[q][1];
    if (k0 + ECH < nmine) load_chunk(k0 + ECH);  // the next chunk's loads in flight
#pragma unroll
    for (int q = 0; q < ECH; ++q) {
      const int col = c0 + (k0 + q) * step, b = itm.J * HT + col;
      if (col >= ncol) continue;
      const int cb = b * (b + 1) / 2;
      double* dcol = Dc + cb + a0;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        if (DIAG && a0 + 32 * h2 > b) continue;
        const double h = hv[q][h2];
        const double dv = __dsub_rn(h, hkc[q][h2]);
        __stcs(dcol + 32 * h2, dv);
        if (Hc) Hc[cb + a0 + 32 * h2] = h;
        po = fma(dv, dv, po);
        const uint32_t habs = static_cast<uint32_t>(__double2hiint(dv)) & 0x7fffffffu;
        hmax = max(hmax, habs);
        nzb |= habs | static_cast<uint32_t>(__double2loint(dv));
      }
    }
  }
  double part = 2.0 * po;
  if (DIAG) {  // the diagonal terms count once: take one of the two back
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int cc = lane + 32 * h2, a = a0 + 32 * h2;
      if (cc < ncol && cc >= c0 && (cc - c0) % step == 0) {
        const double dv = __dsub_rn(sm.cs[cc * HW_LD + cc], __ldg(hest_c + a * (a + 1) / 2 + a));
        part = fma(-dv, dv, part);
      }
    }
  }
  return part;
}

__device__ __forceinline__ double hw_epi_cols(HwPipe& sm, const HwItem& itm, int c0, int step, int d,
                                              int64_t w, const double* __restrict__ hest, int64_t hest_stride,
                                              const double* __restrict__ lam_arr, double* __restrict__ D,
                                              double* __restrict__ hess_out, int32_t* __restrict__ flags,
                                              int lane, uint64_t* release = nullptr) {
  const double* hest_c = hest + static_cast<int64_t>(itm.c) * hest_stride;
  const double lam = lam_arr[itm.c];
  double* Dc = D + static_cast<int64_t>(itm.c) * w;
  double* Hc = hess_out ? hess_out + static_cast<int64_t>(itm.slot) * w : nullptr;
  const int ncol = min(HT, d - itm.J * HT);
  const int nmine = ncol > c0 ? (ncol - c0 + step - 1) / step : 0;  // this warp's columns
  uint32_t hmax = 0, nzb = 0;
  double part = itm.diag ? hw_epi_body<true>(sm, itm, c0, step, nmine, ncol, hest_c, Dc, Hc, lam, lane, hmax, nzb)
                         : hw_epi_body<false>(sm, itm, c0, step, nmine, ncol, hest_c, Dc, Hc, lam, lane, hmax, nzb);
  if (release) {  // every read of `cs` is done: hand it back before the sums
    __syncwarp();
    if (lane == 0) mbar_arrive(release);
  }
  part = warp_sum(part);
  const int fl = __reduce_or_sync(0xffffffffu, (hmax >= 0x7ff00000u ? 1 : 0) | (nzb != 0 ? 2 : 0));
  if (lane == 0 && fl) atomicOr(&flags[itm.c], fl);
  return part;
}

template <bool solo>
__global__ void __launch_bounds__(HW_THREADS, 1) k_hessian_ws(
    const __grid_constant__ CUtensorMap tmap_b, const DevCtl* __restrict__ ctl, int d,
    const int32_t* __restrict__ ni_arr, int ldh, const double* __restrict__ hcoef,
    const double* __restrict__ lam_arr, const int32_t* __restrict__ clients,
    const double* __restrict__ hest, int64_t hest_stride, double* __restrict__ D,
    double* __restrict__ hess_out, double* __restrict__ frob_part, int32_t* __restrict__ flags,
    uint32_t zero_mask, const double* __restrict__ gcoef, const double* __restrict__ x,
    double* __restrict__ grad, const int32_t* __restrict__ pair_order, int n_pairs, int n_act,
    int grp, int32_t* __restrict__ sched, int b_evict_first) {
  // sched[0]: next unclaimed item, sched[1]: producers finished (the last
  // one re-arms both for the next launch)
  // the round reduction may launch now (it waits for this pass)
  asm volatile("griddepcontrol.launch_dependents;");
  if (ctl && ctl->halt) return;
  if (threadIdx.x == 0) tl_mark(1, false);
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared array (keeps the
  // shared address space: LDS with 32-bit addresses, not generic loads)
  HwPipe* pipes = reinterpret_cast<HwPipe*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = n_act * n_pairs;
  if (tid < HW_PIPES) {
    HwPipe& pp = pipes[tid];
    for (int s2 = 0; s2 < HW_STAGE; ++s2) {
      mbar_init(&pp.full[s2], 1);
      mbar_init(&pp.empty[s2], HW_MMA);
    }
    mbar_init(&pp.cs_full, HW_MMA);
    mbar_init(&pp.cs_empty, 1);
    if (tid == 0) tma_prefetch_desc(&tmap_b);
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t w = packed_len(d);
  // warps [0, 8): DMMA (pipe = warp / 4); 8, 9: TMA of pipe 0, 1; 10, 11: epilogue of pipe 0, 1
  const int pipe = warp < HW_PIPES * HW_MMA ? warp / HW_MMA : (warp - HW_PIPES * HW_MMA) % HW_PIPES;
  HwPipe& sm = pipes[pipe];

  if (warp >= HW_PIPES * HW_MMA && warp < HW_PIPES * HW_MMA + HW_PIPES) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // margins' coefficients
      int gsn = 0;
      const uint64_t pol = b_evict_first ? l2_evict_first_policy() : l2_evict_normal_policy();
      for (int j = 0;; ++j) {
        int L = atomicAdd(&sched[0], 1);
        if (L >= total) L = -1;
        sm.itemq[j % HW_QUEUE] = L;
        if (L < 0) {  // publish the end through the next stage barrier
          const int s2 = gsn % HW_STAGE;
          if (gsn >= HW_STAGE) mbar_wait(&sm.empty[s2], ((gsn / HW_STAGE) - 1) & 1);
          mbar_arrive(&sm.full[s2]);
          break;
        }
        const HwItem itm = hw_item(L, n_pairs, n_act, grp, pair_order, clients, ni_arr);
        const bool fuse_grad = itm.diag && grad != nullptr;
        const uint32_t stage_bytes =
            (itm.diag ? 1u : 2u) * HT * HKC * 8u + HKC * 8u + (fuse_grad ? HKC * 8u : 0u);
        const double* hrow = hcoef + static_cast<int64_t>(itm.c) * ldh;
        const double* grow = gcoef + static_cast<int64_t>(itm.c) * ldh;
        for (int it = 0; it < itm.nk; ++it, ++gsn) {
          const int s2 = gsn % HW_STAGE;
          if (gsn >= HW_STAGE) mbar_wait(&sm.empty[s2], ((gsn / HW_STAGE) - 1) & 1);
          mbar_arrive_expect_tx(&sm.full[s2], stage_bytes);
          tma_load_3d_hint(sm.a[s2], &tmap_b, &sm.full[s2], it * HKC, itm.I * HT, itm.c, pol);
          if (!itm.diag) tma_load_3d_hint(sm.b[s2], &tmap_b, &sm.full[s2], it * HKC, itm.J * HT, itm.c, pol);
          bulk_load(sm.h[s2], hrow + it * HKC, HKC * 8, &sm.full[s2]);
          if (fuse_grad) bulk_load(sm.gc[s2], grow + it * HKC, HKC * 8, &sm.full[s2]);
        }
      }
      __threadfence();
      if (atomicAdd(&sched[1], 1) == HW_PIPES * static_cast<int>(gridDim.x) - 1) {
        atomicExch(&sched[0], 0);  // every producer has claimed its last item
        atomicExch(&sched[1], 0);
      }
    }
    return;
  }

  if (warp < HW_PIPES * HW_MMA) {
    // ------------------------------------------------------ DMMA warps
    // Task -> sub-partition placement (warp k of either pipe runs on
    // sub-partition k; the epilogue warps sit on sub-partitions 2 and 3, the
    // idle-most TMA warps on 0 and 1).  A diagonal tile has two 10-fragment
    // triangle tasks (which also form the gradient) and two 8-fragment
    // rectangles.  Few tiles per dimension (d <= 512, where diagonal tiles
    // are a third of the items): both triangles on sub-partitions 0 and 1,
    // away from the epilogue warps' FP64 / issue load (c0 195.3 -> 188.8 us).
    // Many tiles (c4): the second pipe takes the tasks pairwise swapped, so
    // triangles meet the other pipe's rectangles (c4 34.57 -> 34.49 ms).
    const int q4 = n_pairs <= 36 ? ((0x2130 >> (4 * (warp % HW_MMA))) & 3) : ((warp % HW_MMA) ^ (pipe & 1));
    const int g = lane >> 2, t = lane & 3;
    int gsn = 0;
    for (int j = 0;; ++j) {
      mbar_wait(&sm.full[gsn % HW_STAGE], (gsn / HW_STAGE) & 1);  // the item's first stage (or the end)
      const int L = sm.itemq[j % HW_QUEUE];
      if (L < 0) {  // tell the epilogue, once it has taken the last tile
        if constexpr (solo) {
          if (q4 == 0 && lane == 0) sm.solo_item = -1;
          asm volatile("bar.sync %0, %1;" ::"r"(1 + pipe), "r"((HW_MMA + 1) * 32) : "memory");
          break;
        }
        if (j > 0) mbar_wait(&sm.cs_empty, (j - 1) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.cs_full);
        break;
      }
      const HwItem itm = hw_item(L, n_pairs, n_act, grp, pair_order, clients, ni_arr);
      const bool fuse_grad = itm.diag && grad != nullptr;
      const int nv = min(8, (d - itm.J * HT + 7) / 8);
      const HwTask tk = hw_task(q4, itm.diag, nv);
      double acc[4][4][2];
      double gpart[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
      const bool active = tk.mr > 0 && tk.nc > 0;
      if (!active) {
        hw_skip(sm, itm.nk, gsn, lane);
      } else if (tk.tri) {
        if (fuse_grad)
          hw_consume_any<true, true>(tk.mr, tk.nc, sm, true, itm.nk, gsn, tk.r0, tk.c0, g, t, lane, zero_mask, acc, gpart);
        else
          hw_consume_any<true, false>(tk.mr, tk.nc, sm, true, itm.nk, gsn, tk.r0, tk.c0, g, t, lane, zero_mask, acc, gpart);
      } else {
        hw_consume_any<false, false>(tk.mr, tk.nc, sm, itm.diag, itm.nk, gsn, tk.r0, tk.c0, g, t, lane, zero_mask, acc,
                                     gpart);
      }
      gsn += itm.nk;
      if (fuse_grad && tk.grad) {  // local gradient rows 8 r0 .. (oracle.py:108-121)
        const double lam = lam_arr[itm.c];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          double v = gpart[mi];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          const int a = itm.I * HT + 8 * (tk.r0 + mi) + g;
          if (mi < tk.mr && t == 0 && a < d)
            grad[static_cast<int64_t>(itm.c) * d + a] = __dadd_rn(v, __dmul_rn(lam, x[a]));
        }
      }
      // hand the accumulators to the epilogue once it has read the last tile
      if (j > 0 && !solo) mbar_wait(&sm.cs_empty, (j - 1) & 1);
      if (active) {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj)
            if (mi < tk.mr && nj < tk.nc)
#pragma unroll
              for (int e = 0; e < 2; ++e)
                sm.cs[(8 * (tk.c0 + nj) + 2 * t + e) * HW_LD + 8 * (tk.r0 + mi) + g] = acc[mi][nj][e];
      }
      if constexpr (solo) {  // few tiles per pipe: the five warps finish this one together
        if (q4 == 0 && lane == 0) sm.solo_item = L;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + pipe), "r"((HW_MMA + 1) * 32) : "memory");
        const double part = hw_epi_cols(sm, itm, q4, HW_MMA + 1, d, w, hest, hest_stride, lam_arr, D,
                                        hess_out, flags, lane);
        if (lane == 0) sm.solo_part[q4] = part;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + pipe), "r"((HW_MMA + 1) * 32) : "memory");
        continue;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.cs_full);
    }
    return;
  }

  // ------------------------------------------------------------ epilogue
  if constexpr (solo) {
    for (;;) {
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pipe), "r"((HW_MMA + 1) * 32) : "memory");
      const int L = sm.solo_item;
      if (L < 0) break;
      const HwItem itm = hw_item(L, n_pairs, n_act, grp, pair_order, clients, ni_arr);
      const double part = hw_epi_cols(sm, itm, HW_MMA, HW_MMA + 1, d, w, hest, hest_stride, lam_arr, D,
                                      hess_out, flags, lane);
      if (lane == 0) sm.solo_part[HW_MMA] = part;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pipe), "r"((HW_MMA + 1) * 32) : "memory");
      if (lane == 0) {
        double tot = 0.0;
#pragma unroll
        for (int q = 0; q <= HW_MMA; ++q) tot += sm.solo_part[q];
        frob_part[static_cast<int64_t>(itm.c) * n_pairs + itm.pair] = tot;
      }
    }
  } else {
    for (int j = 0;; ++j) {
      mbar_wait(&sm.cs_full, j & 1);
      const int L = sm.itemq[j % HW_QUEUE];
      if (L < 0) break;
      const HwItem itm = hw_item(L, n_pairs, n_act, grp, pair_order, clients, ni_arr);
      const double part = hw_epi_cols(sm, itm, 0, 1, d, w, hest, hest_stride, lam_arr, D, hess_out, flags, lane,
                                      &sm.cs_empty);  // (the DMMA warps may stage the next tile)
      if (lane == 0) frob_part[static_cast<int64_t>(itm.c) * n_pairs + itm.pair] = part;
    }
  }
  if (lane == 0) tl_mark(1, true);
}

}  // namespace fb
