// compress_kernels.cuh — Hessian-shift compressors on packed differences
// (reference compressors.py:132-370).
//
// Output of every kind, per client c:
//   bitmap[c][wb]   selected packed positions (bit t%32 of word t/32)
//   count[c]        number of entries (0 for an all-zero difference: no draws)
//   idx/val lists   ascending positions and their values (values scaled by
//                   w/k for the Rand kinds), capacity `cap` per client
//   draws[c]        u64 draws consumed from the client's round stream
// Dense kinds (identity, natural) set count = w and leave the bitmap unused.
//
// Bit-exactness notes:
//  * TopK ranks |v| (or wt v v), descending, ties to the smaller position
//    (np.lexsort, compressors.py:139-141).  |v| >= 0 doubles order like their
//    63-bit patterns, so an exact radix select over (key, position) is used.
//  * TopLEK replicates numpy's pairwise np.sum over the sorted energies and
//    the sequential cumsum / division / searchsorted of toplek_plan.
//  * Rand values are fl(v * (w / k)) with w / k a correctly rounded double.
#pragma once
#include "common.cuh"

namespace fb {

constexpr int TK_THREADS = 1024;
constexpr int TK_NW = TK_THREADS / 32;

// energy = (wt * v) * v exactly as numpy evaluates weights * packed * packed
__device__ __forceinline__ double energy_of(double v, int64_t t) {
  const double wt = packed_is_diag_fast(t) ? 1.0 : 2.0;
  return __dmul_rn(__dmul_rn(wt, v), v);
}
__device__ __forceinline__ uint64_t rank_key(double v, int64_t t, int weighted) {
  if (weighted) return static_cast<uint64_t>(__double_as_longlong(energy_of(v, t)));
  return static_cast<uint64_t>(__double_as_longlong(v)) & 0x7FFFFFFFFFFFFFFFull;
}

// exclusive block scan of ints (blockDim.x a multiple of 32, <= 1024);
// the block total is returned through `total`.  ws: 64 ints of smem.
__device__ __forceinline__ int block_excl_scan(int v, int* ws, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = (lane < nw) ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    ws[32 + lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const int before = (wid == 0) ? 0 : ws[32 + wid - 1];
  *total = ws[32 + nw - 1];
  return before + x - v;
}

// What a compressor emits besides its (idx, val) list:
//  * the client's shift update Hest[c][t] = fl(Hest + fl(alpha v)) at every
//    selected position (compressors.py:373-393, algorithms.py:234) when hest
//    is non-null, and
//  * range starts rs[c][r] = #entries with position < r * FOLD_RANGE
//    (r = 0..nr) so the master fold can slice every client's list by range.
constexpr int FOLD_RANGE = 256;
struct Emit {
  double* hest;
  int64_t hest_stride;
  double alpha;
  int32_t* rs;
  int nr;
};
__device__ __forceinline__ void emit_entry(const Emit& em, int c, int64_t t, double v) {
  if (em.hest) {
    double* hp = em.hest + static_cast<int64_t>(c) * em.hest_stride + t;
    *hp = __dadd_rn(*hp, __dmul_rn(em.alpha, v));
  }
}

__device__ __forceinline__ void emit_empty(const Emit& em, int c) {
  if (em.rs)
    for (int r = threadIdx.x; r <= em.nr; r += blockDim.x) em.rs[static_cast<int64_t>(c) * (em.nr + 1) + r] = 0;
}

__device__ __forceinline__ void clear_row(uint32_t* row, int wb) {
  for (int q = threadIdx.x; q < wb; q += blockDim.x) row[q] = 0u;
}

// Compact a bitmap row into ascending (idx, val) lists; val = fl(v * scale)
// when scale != 1 (Rand kinds).  Emits the client update and range starts.
// Whole block, any blockDim multiple of 32.
__device__ void compact_bitmap(const uint32_t* __restrict__ row, int wb,
                               const double* __restrict__ v, double scale, uint32_t* idx,
                               double* val, int* ws, const Emit& em, int c) {
  int carry = 0;
  int32_t* rsc = em.rs ? em.rs + static_cast<int64_t>(c) * (em.nr + 1) : nullptr;
  for (int base = 0; base < wb; base += blockDim.x) {
    const int q = base + threadIdx.x;
    const uint32_t word = (q < wb) ? row[q] : 0u;
    int total;
    int off = block_excl_scan(__popc(word), ws, &total) + carry;
    if (rsc && q < wb && (q % (FOLD_RANGE / 32)) == 0) rsc[q / (FOLD_RANGE / 32)] = off;
    uint32_t m = word;
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      const int64_t t = static_cast<int64_t>(q) * 32 + bit;
      const double x = (scale == 1.0) ? v[t] : __dmul_rn(v[t], scale);
      idx[off] = static_cast<uint32_t>(t);
      val[off] = x;
      emit_entry(em, c, t, x);
      ++off;
    }
    carry += total;
    __syncthreads();
  }
  if (rsc && threadIdx.x == 0) rsc[em.nr] = carry;
}

// ------------------------------------------------------------------- TopK
// grid n_active, block 1024.
__global__ void __launch_bounds__(TK_THREADS) k_topk(
    const DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int wb, int k,
    int weighted, const int32_t* __restrict__ clients, const int32_t* __restrict__ flags,
    uint32_t* __restrict__ bitmap, int32_t* __restrict__ count, uint32_t* __restrict__ idx_list,
    double* __restrict__ val_list, int cap, int32_t* __restrict__ draws, Emit em) {
  if (ctl && ctl->halt) return;
  __shared__ uint32_t hist[2048];
  __shared__ int ws[64];
  __shared__ int s_digit, s_above;
  const int c = client_of(clients, blockIdx.x);
  const double* v = D + static_cast<int64_t>(c) * w;
  uint32_t* brow = bitmap + static_cast<int64_t>(c) * wb;
  if (threadIdx.x == 0 && draws) draws[c] = 0;
  if (!(flags[c] & 2)) {  // all-zero difference: empty delta, no draws
    clear_row(brow, wb);
    emit_empty(em, c);
    if (threadIdx.x == 0) count[c] = 0;
    return;
  }
  const int lane = threadIdx.x & 31;
  constexpr int LO[6] = {52, 41, 30, 19, 8, 0};
  constexpr int BITS[6] = {11, 11, 11, 11, 11, 8};
  uint64_t prefix = 0;  // selected digits so far (key >> (LO[L] + BITS[L]))
  int need = k;
  bool take_all = false;
  int lo = 0;
  for (int L = 0; L < 6; ++L) {
    lo = LO[L];
    const int bits = BITS[L];
    const int hi = lo + bits;
    const uint32_t mask = (1u << bits) - 1u;
    for (int i = threadIdx.x; i < 2048; i += TK_THREADS) hist[i] = 0u;
    __syncthreads();
    for (int64_t base = 0; base < w; base += TK_THREADS) {
      const int64_t t = base + threadIdx.x;
      uint32_t dig = 0xFFFFFFFFu;
      if (t < w) {
        const uint64_t key = rank_key(v[t], t, weighted);
        if ((hi >= 64 ? 0ull : (key >> hi)) == prefix) dig = static_cast<uint32_t>(key >> lo) & mask;
      }
      const uint32_t peers = __match_any_sync(0xffffffffu, dig);
      if (dig != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[dig], __popc(peers));
    }
    __syncthreads();
    // locate the digit holding the need-th largest key: bins scanned from the top
    {
      const int b0 = 2047 - 2 * threadIdx.x, b1 = b0 - 1;  // descending pair
      const int c0 = static_cast<int>(hist[b0]), c1 = static_cast<int>(hist[b1]);
      int total;
      const int above0 = block_excl_scan(c0 + c1, ws, &total);
      const int above1 = above0 + c0;
      if (above0 < need && need <= above0 + c0) { s_digit = b0; s_above = above0; }
      if (c1 > 0 && above1 < need && need <= above1 + c1) { s_digit = b1; s_above = above1; }
    }
    __syncthreads();
    const int dg = s_digit;
    need -= s_above;
    prefix = (prefix << bits) | static_cast<uint64_t>(dg);
    const bool all = (static_cast<int>(hist[dg]) == need);
    __syncthreads();
    if (all) { take_all = true; break; }
  }
  // final pass: ascending compaction of {key > T} U {first `need` of key == T}
  int carry_sel = 0, carry_eq = 0;
  uint32_t* il = idx_list + static_cast<int64_t>(c) * cap;
  double* vl = val_list + static_cast<int64_t>(c) * cap;
  for (int64_t base = 0; base < w; base += TK_THREADS) {
    const int64_t t = base + threadIdx.x;
    int gt = 0, eq = 0;
    double vt = 0.0;
    if (t < w) {
      vt = v[t];
      const uint64_t hk = rank_key(vt, t, weighted) >> lo;
      gt = hk > prefix;
      eq = hk == prefix;
    }
    int sel = gt | eq;
    if (!take_all) {
      int tot_eq;
      const int r = block_excl_scan(eq, ws, &tot_eq) + carry_eq;
      carry_eq += tot_eq;
      sel = gt | (eq & (r < need));
    }
    int tot_sel;
    const int pos = block_excl_scan(sel, ws, &tot_sel) + carry_sel;
    carry_sel += tot_sel;
    if (em.rs && t < w && (t % FOLD_RANGE) == 0)
      em.rs[static_cast<int64_t>(c) * (em.nr + 1) + t / FOLD_RANGE] = pos;
    if (sel) {
      il[pos] = static_cast<uint32_t>(t);
      vl[pos] = vt;
      emit_entry(em, c, t, vt);
    }
    const uint32_t word = __ballot_sync(0xffffffffu, sel);
    if (lane == 0 && t < w + 31) {
      const int64_t q = t >> 5;
      if (q < wb) brow[q] = word;
    }
  }
  if (threadIdx.x == 0) {
    count[c] = carry_sel;
    if (em.rs) em.rs[static_cast<int64_t>(c) * (em.nr + 1) + em.nr] = carry_sel;
  }
}

// ------------------------------------------------- TopK, shared-memory path
// For w <= TKS_MAXW the upper 32 bits of every key stay in shared memory
// after ONE coalesced pass over D (which also builds the first histogram);
// the remaining radix levels on those bits run out of shared memory, and only
// the group tied on the upper 32 bits is re-read from global memory to
// resolve the low 31 bits; its members' verdicts (greater / tied) are kept
// as bitmasks so the selection sweeps never touch global memory.  The
// selection rule is identical to k_topk (descending key, ties to the smaller
// position).
//
// dynamic shared memory: hi[w] u32 | gtm[wb] u32 | eqm[wb] u32 | scratch
// (histogram + candidates during selection, the position list afterwards)
constexpr int TKS_MAXW = 46000;
constexpr int TKS_CAND = 1024;
constexpr int TKS_SCRATCH = 16384;  // bytes
constexpr int TKS_POS = TKS_SCRATCH / 4;
__host__ __device__ constexpr size_t tks_smem_bytes(int64_t w) {
  return static_cast<size_t>(w) * 4 + 3 * static_cast<size_t>((w + 31) / 32) * 4 + TKS_SCRATCH;
}
constexpr size_t TKS_SMEM = tks_smem_bytes(TKS_MAXW);

// Radix digit search over hist[0, nbins): the digit holding the need-th
// largest element (counting from the top bin).  Whole block; returns digit
// and the count strictly above it through shared scalars.
__device__ __forceinline__ void tks_find_digit(const uint32_t* hist, int nbins, int need, int* ws,
                                               int* s_digit, int* s_above) {
  const int b0 = nbins - 1 - 2 * static_cast<int>(threadIdx.x), b1 = b0 - 1;
  const int c0 = (b0 >= 0) ? static_cast<int>(hist[b0]) : 0;
  const int c1 = (b1 >= 0) ? static_cast<int>(hist[b1]) : 0;
  int total;
  const int above0 = block_excl_scan(c0 + c1, ws, &total);
  const int above1 = above0 + c0;
  if (c0 > 0 && above0 < need && need <= above0 + c0) { *s_digit = b0; *s_above = above0; }
  if (c1 > 0 && above1 < need && need <= above1 + c1) { *s_digit = b1; *s_above = above1; }
  __syncthreads();
}

// Histogram increment with a warp-uniform fast path (tie-heavy inputs put
// whole warps in one bin): one atomic of the population instead of 32.
__device__ __forceinline__ void tks_add(uint32_t* hist, uint32_t dig, int lane) {
  const uint32_t valid = __ballot_sync(0xffffffffu, dig != 0xFFFFFFFFu);
  if (!valid) return;
  const uint32_t first = __shfl_sync(0xffffffffu, dig, __ffs(valid) - 1);
  if (__all_sync(0xffffffffu, dig == first || dig == 0xFFFFFFFFu)) {
    if (lane == 0) atomicAdd(&hist[first], __popc(valid));
  } else if (dig != 0xFFFFFFFFu) {
    atomicAdd(&hist[dig], 1u);
  }
}

__device__ __forceinline__ uint32_t lo_key(const double* v, int t, int weighted) {
  return static_cast<uint32_t>(rank_key(__ldg(v + t), t, weighted) & 0x7FFFFFFFull);
}
// low 31 key bits, skipping the global re-read when they are known to be zero
__device__ __forceinline__ uint32_t lo_key_m(const double* v, int t, int weighted,
                                             const uint32_t* lzm) {
  return ((lzm[t >> 5] >> (t & 31)) & 1u) ? 0u : lo_key(v, t, weighted);
}

__global__ void __launch_bounds__(TK_THREADS, 1) k_topk_smem(
    const DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int wb, int k,
    int weighted, const int32_t* __restrict__ clients, const int32_t* __restrict__ flags,
    uint32_t* __restrict__ bitmap, int32_t* __restrict__ count, uint32_t* __restrict__ idx_list,
    double* __restrict__ val_list, int cap, int32_t* __restrict__ draws, Emit em) {
  if (ctl && ctl->halt) return;
  PhaseClock pc;
  const long long gt_start = globaltimer_ns();
  extern __shared__ uint32_t tks_dyn[];
  const int wi = static_cast<int>(w);
  uint32_t* hi_s = tks_dyn;                  // [wi]
  uint32_t* gtm = tks_dyn + wi;              // [wb] tie group: key greater than threshold
  uint32_t* eqm = gtm + wb;                  // [wb] tie group: key equal to threshold
  uint32_t* lzm = eqm + wb;                  // [wb] low 31 key bits are zero (no re-read)
  uint32_t* scratch = lzm + wb;              // TKS_SCRATCH bytes
  uint32_t* hist = scratch;                  // [2048]
  uint32_t* cand_lo = scratch + 2048;        // [TKS_CAND]
  int32_t* cand_t = reinterpret_cast<int32_t*>(scratch + 2048 + TKS_CAND);  // [TKS_CAND]
  int32_t* pos_list = reinterpret_cast<int32_t*>(scratch);                   // [TKS_POS] later
  __shared__ int ws[64];
  __shared__ int s_digit, s_above, s_ncand;
  __shared__ int w_gt[TK_NW], w_eq[TK_NW], w_sel_pre[TK_NW], w_eq_pre[TK_NW];
  const int c = client_of(clients, blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* v = D + static_cast<int64_t>(c) * w;
  uint32_t* brow = bitmap + static_cast<int64_t>(c) * wb;
  if (tid == 0 && draws) draws[c] = 0;
  if (!(flags[c] & 2)) {
    clear_row(brow, wb);
    emit_empty(em, c);
    if (tid == 0) count[c] = 0;
    return;
  }
  // ---- pass 0: keys' upper halves into smem + histogram of hi bits [21, 32)
  for (int i = tid; i < 2048; i += TK_THREADS) hist[i] = 0u;
  for (int i = tid; i < wb; i += TK_THREADS) { gtm[i] = 0u; eqm[i] = 0u; lzm[i] = 0u; }
  if (tid == 0) s_ncand = 0;
  __syncthreads();
  constexpr int UNR = 8;  // loads in flight per thread
  for (int base = 0; base < wi; base += UNR * TK_THREADS) {
    double x[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = base + u * TK_THREADS + tid;
      x[u] = (t < wi) ? __ldg(v + t) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = base + u * TK_THREADS + tid;
      uint32_t dig = 0xFFFFFFFFu;
      bool lz = false;
      if (t < wi) {
        const uint64_t key = rank_key(x[u], t, weighted);
        const uint32_t hi = static_cast<uint32_t>(key >> 31);
        hi_s[t] = hi;
        dig = hi >> 21;
        lz = (key & 0x7FFFFFFFull) == 0;
      }
      const uint32_t lzb = __ballot_sync(0xffffffffu, lz);
      if (lane == 0 && t < wi) lzm[t >> 5] = lzb;
      tks_add(hist, dig, lane);
    }
  }
  __syncthreads();
  pc.mark(0);
  // ---- radix levels on the upper 32 bits (all in shared memory)
  constexpr int HSH[3] = {21, 10, 0};
  constexpr int HBI[3] = {11, 11, 10};
  uint32_t prefix = 0;
  int need = k;
  int level_shift = 0;     // shift of the prefix that decides the selection
  bool take_all = false;   // every element with that prefix is selected
  for (int L = 0; L < 3; ++L) {
    if (L > 0) {
      for (int i = tid; i < 2048; i += TK_THREADS) hist[i] = 0u;
      __syncthreads();
      const int hsh = HSH[L - 1];
      const uint32_t dmask = (1u << HBI[L]) - 1u;
      for (int base = 0; base < wi; base += TK_THREADS) {
        const int t = base + tid;
        uint32_t dig = 0xFFFFFFFFu;
        if (t < wi) {
          const uint32_t hi = hi_s[t];
          if ((hi >> hsh) == prefix) dig = (hi >> HSH[L]) & dmask;
        }
        tks_add(hist, dig, lane);
      }
      __syncthreads();
    }
    tks_find_digit(hist, 1 << HBI[L], need, ws, &s_digit, &s_above);
    const int dg = s_digit;
    need -= s_above;
    prefix = (L == 0) ? static_cast<uint32_t>(dg) : ((prefix << HBI[L]) | static_cast<uint32_t>(dg));
    level_shift = HSH[L];
    const bool all = (static_cast<int>(hist[dg]) == need);
    __syncthreads();
    if (all) { take_all = true; break; }
  }
  pc.mark(1);
  // ---- low 31 bits among the elements tied on all 32 upper bits; their
  //      verdicts go to the gt / eq bitmasks
  const uint32_t T_hi = prefix;  // meaningful when !take_all (level_shift == 0)
  if (!take_all) {
    // gather the tie group (warp-aggregated: one shared atomic per warp) and
    // count members whose low key bits are not known to be zero
    __shared__ int s_nnz;
    if (tid == 0) s_nnz = 0;
    __syncthreads();
    for (int base = 0; base < wi; base += TK_THREADS) {
      const int t = base + tid;
      const bool in = t < wi && hi_s[t] == T_hi;
      const bool nz = in && !((lzm[t >> 5] >> (t & 31)) & 1u);
      const uint32_t inb = __ballot_sync(0xffffffffu, in), nzb = __ballot_sync(0xffffffffu, nz);
      int wbase = 0;
      if (lane == 0 && inb) {
        wbase = atomicAdd(&s_ncand, __popc(inb));
        if (nzb) atomicAdd(&s_nnz, __popc(nzb));
      }
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      if (in) {
        const int slot = wbase + __popc(inb & ((1u << lane) - 1u));
        if (slot < TKS_CAND) {
          cand_t[slot] = t;
          cand_lo[slot] = nz ? lo_key(v, t, weighted) : 0u;
        }
      }
    }
    __syncthreads();
    const int ncand = s_ncand;
    if (s_nnz == 0) {
      // every tied key is exactly T_hi << 31: the whole group is "equal";
      // the first `need` of them by position are taken in the sweeps
      for (int base = 0; base < wi; base += TK_THREADS) {
        const int t = base + tid;
        const uint32_t eb = __ballot_sync(0xffffffffu, t < wi && hi_s[t] == T_hi);
        if (lane == 0 && t < wi) eqm[t >> 5] = eb;
      }
      __syncthreads();
    } else {
      const bool in_smem = ncand <= TKS_CAND;
      uint32_t lo_prefix = 0;
      int lo_shift = 0;
      bool lo_all = false;
      constexpr int LSH[3] = {20, 10, 0};
      constexpr int LBI[3] = {11, 10, 10};
      for (int L = 0; L < 3; ++L) {
        for (int i = tid; i < 2048; i += TK_THREADS) hist[i] = 0u;
        __syncthreads();
        const int upper = L == 0 ? 31 : LSH[L - 1];
        const uint32_t dmask = (1u << LBI[L]) - 1u;
        const int lim = in_smem ? ncand : wi;
        for (int base = 0; base < lim; base += TK_THREADS) {
          const int e = base + tid;
          uint32_t dig = 0xFFFFFFFFu;
          bool have = false;
          uint32_t lo = 0;
          if (e < lim) {
            if (in_smem) { lo = cand_lo[e]; have = true; }
            else if (hi_s[e] == T_hi) { lo = lo_key_m(v, e, weighted, lzm); have = true; }
          }
          if (have && (upper >= 31 ? 0u : (lo >> upper)) == lo_prefix) dig = (lo >> LSH[L]) & dmask;
          tks_add(hist, dig, lane);
        }
        __syncthreads();
        tks_find_digit(hist, 1 << LBI[L], need, ws, &s_digit, &s_above);
        const int dg = s_digit;
        need -= s_above;
        lo_prefix = (L == 0) ? static_cast<uint32_t>(dg) : ((lo_prefix << LBI[L]) | static_cast<uint32_t>(dg));
        lo_shift = LSH[L];
        const bool all = (static_cast<int>(hist[dg]) == need);
        __syncthreads();
        if (all) { lo_all = true; break; }
      }
      // verdicts of the tie group
      if (in_smem) {
        for (int e = tid; e < ncand; e += TK_THREADS) {
          const int t = cand_t[e];
          const uint32_t lp = cand_lo[e] >> lo_shift;
          if (lp > lo_prefix || (lo_all && lp == lo_prefix)) atomicOr(&gtm[t >> 5], 1u << (t & 31));
          else if (lp == lo_prefix) atomicOr(&eqm[t >> 5], 1u << (t & 31));
        }
      } else {  // large tie group: warp-aligned sweep, one word per warp ballot
        for (int base = 0; base < wi; base += TK_THREADS) {
          const int t = base + tid;
          int g_ = 0, e_ = 0;
          if (t < wi && hi_s[t] == T_hi) {
            const uint32_t lp = lo_key_m(v, t, weighted, lzm) >> lo_shift;
            g_ = lp > lo_prefix || (lo_all && lp == lo_prefix);
            e_ = !g_ && lp == lo_prefix;
          }
          const uint32_t gb = __ballot_sync(0xffffffffu, g_), eb = __ballot_sync(0xffffffffu, e_);
          if (lane == 0 && t < wi) { gtm[t >> 5] = gb; eqm[t >> 5] = eb; }
        }
      }
      __syncthreads();
    }
  }
  pc.mark(2);
  // ---- final selection, ascending positions.  Warp w owns the contiguous
  //      segment [w*S, (w+1)*S) (S a multiple of 32): a counting sweep, one
  //      scan over the 32 warp totals, then an emitting sweep.
  auto classify = [&](int t, uint32_t& gt_bits, uint32_t& eq_bits) {
    // lane-wise verdicts for t = t0 + lane, returned as warp ballots
    int gt = 0;
    if (t < wi) {
      const uint32_t hp = hi_s[t] >> level_shift;
      gt = take_all ? (hp >= prefix) : (hp > T_hi);
    }
    gt_bits = __ballot_sync(0xffffffffu, gt);
    if (!take_all && t - lane < wi) {
      const int q = (t - lane) >> 5;
      gt_bits |= gtm[q];
      eq_bits = eqm[q];
    } else {
      eq_bits = 0u;
    }
  };
  const int S = ((wi + TK_THREADS - 1) / TK_THREADS) * 32;
  const int seg0 = warp * S, seg1 = min(wi, seg0 + S);
  int n_gt = 0, n_eq = 0;
  for (int t0 = seg0; t0 < seg1; t0 += 32) {
    uint32_t gb, eb;
    classify(t0 + lane, gb, eb);
    n_gt += __popc(gb);
    n_eq += __popc(eb);
  }
  if (lane == 0) { w_gt[warp] = n_gt; w_eq[warp] = n_eq; }
  __syncthreads();
  pc.mark(3);
  if (warp == 0) {
    int eq_excl = w_eq[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, eq_excl, o);
      if (lane >= o) eq_excl += y;
    }
    eq_excl -= w_eq[lane];  // exclusive prefix of tied keys
    const int eq_take = max(0, min(need - eq_excl, w_eq[lane]));
    const int sel = w_gt[lane] + eq_take;
    int sel_incl = sel;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, sel_incl, o);
      if (lane >= o) sel_incl += y;
    }
    w_sel_pre[lane] = sel_incl - sel;
    w_eq_pre[lane] = eq_excl;
    if (lane == 31) s_above = sel_incl;  // total selected
  }
  __syncthreads();
  const int total = s_above;
  const bool keep_pos = total <= TKS_POS;
  uint32_t* il = idx_list + static_cast<int64_t>(c) * cap;
  double* vl = val_list + static_cast<int64_t>(c) * cap;
  int32_t* rsc = em.rs ? em.rs + static_cast<int64_t>(c) * (em.nr + 1) : nullptr;
  int base_sel = w_sel_pre[warp], base_eq = w_eq_pre[warp];
  const uint32_t lt = (1u << lane) - 1u;
  for (int t0 = seg0; t0 < seg1; t0 += 32) {
    const int t = t0 + lane;
    uint32_t gb, eb;
    classify(t, gb, eb);
    const int is_eq = (eb >> lane) & 1;
    const int rank_eq = base_eq + __popc(eb & lt);
    const int sel = ((gb >> lane) & 1) | (is_eq & (rank_eq < need));
    const uint32_t sm_ = __ballot_sync(0xffffffffu, sel);
    const int pos = base_sel + __popc(sm_ & lt);
    if (rsc && t < wi && (t % FOLD_RANGE) == 0) rsc[t / FOLD_RANGE] = pos;
    if (sel) {
      il[pos] = static_cast<uint32_t>(t);
      if (keep_pos) pos_list[pos] = t;
    }
    if (lane == 0) brow[t0 >> 5] = sm_;
    base_sel += __popc(sm_);
    base_eq += __popc(eb);
  }
  pc.mark(4);
  if (tid == 0) {
    count[c] = total;
    if (rsc) rsc[em.nr] = total;
  }
  __syncthreads();
  // values and the client shift update: independent entries, all threads
  for (int e0 = 0; e0 < total; e0 += 2 * TK_THREADS) {
    const int ea = e0 + tid, eb2 = e0 + TK_THREADS + tid;
    const int64_t ta = (ea < total) ? (keep_pos ? pos_list[ea] : il[ea]) : 0;
    const int64_t tb = (eb2 < total) ? (keep_pos ? pos_list[eb2] : il[eb2]) : 0;
    const double va = (ea < total) ? __ldg(v + ta) : 0.0;
    const double vb = (eb2 < total) ? __ldg(v + tb) : 0.0;
    if (ea < total) { vl[ea] = va; emit_entry(em, c, ta, va); }
    if (eb2 < total) { vl[eb2] = vb; emit_entry(em, c, tb, vb); }
  }
  pc.mark(5);
  if (g_dbg_on && tid == 0 && blockIdx.x < 1024) {
    g_dbg_span[2 * blockIdx.x] = gt_start;
    g_dbg_span[2 * blockIdx.x + 1] = globaltimer_ns();
    g_dbg_cta[blockIdx.x] = clock64() - pc.t0;
    if (!take_all) atomicAdd(reinterpret_cast<unsigned long long*>(&g_dbg[16]), 1ull);
  }
}

// ------------------------------------------------- TopK, streaming path
// For w > TKS_MAXW (c4: w = 524,800) the keys do not fit in shared memory,
// so D is streamed from HBM, normally ONCE.  Streaming itself runs at HBM
// speed (tools/probe/stream_bw.cu: 7.3 TB/s for this one-CTA-per-client
// shape), so the pass is built to be lean in instructions per element:
//  1. pivots: a strided sample of 2 * TK_THREADS keys is sorted in shared
//     memory; ranks r -/+ delta around the expected rank of the k-th key give
//     a window (H_lo, H_hi] of key high words that holds the k-th key with
//     overwhelming probability;
//  2. one pass over D: key high word above H_hi -> gt bit (a warp ballot is
//     the bitmap word: no atomics); inside the window -> (key, position)
//     appended to a per-client candidate list in global memory (one shared
//     atomic per warp); exact zeros are tracked as a tie class when the
//     window reaches down to zero (converged differences);
//  3. radix levels on the candidate list find the k-th key (ties -> smaller
//     position via the eq bitmap);
//  4. word-per-lane selection sweeps (ascending positions), then the values
//     pass with the client shift update.
// If the window misses (G >= k, G + M (+ Z) < k, or M > TKST_CAP) the kernel
// falls back to radix levels over D itself.  Selection rule as everywhere:
// descending key, ties to the smaller position.
// dynamic shared memory: gtm[wb] u32 | eqm[wb] u32 | hist[2048] u32 |
//                        sample[2 * TK_THREADS] u64
constexpr int TKST_CAP = 65536;  // candidates per client
constexpr int TKST_SAMPLE = 2 * TK_THREADS;
__host__ __device__ constexpr size_t tkst_smem_bytes(int64_t w) {
  return 2 * static_cast<size_t>((w + 31) / 32) * 4 + 2048 * 4 + TKST_SAMPLE * 8;
}
constexpr int64_t TKST_MAXW = 700000;  // bitmaps + histogram + sample within 227 KB
constexpr int64_t TKST_MINW = 32768;   // below: the shared-memory radix (k_topk_smem)

__device__ __forceinline__ uint32_t key_hi(double x, int64_t t, int weighted) {
  return static_cast<uint32_t>(rank_key(x, t, weighted) >> 32);
}

// Radix levels over the candidate keys whose bits above `top` (exclusive)
// all equal `prefix >> ...`: 11-bit digits from bit `top` down.  Returns the
// threshold prefix / shift; need is reduced by the count above it.
__device__ void tkst_resolve(const uint64_t* __restrict__ ck, int ncand, int top, int& need,
                             uint32_t* hist, int* ws, int* s_digit, int* s_above,
                             uint64_t* prefix_io, int* sh_out, bool* all) {
  const int tid = threadIdx.x, lane = tid & 31;
  uint64_t pf = *prefix_io;  // key >> (top + 1) of every candidate
  int hi_excl = top + 1;     // bits >= hi_excl are fixed by pf
  bool al = false;
  int sh = 0;
  while (true) {
    const int bits = min(11, hi_excl);
    sh = hi_excl - bits;
    for (int i = tid; i < 2048; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const uint32_t dmask = (1u << bits) - 1u;
    for (int base = 0; base < ncand; base += 4 * blockDim.x) {
      uint64_t kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = base + u * blockDim.x + tid;
        kk[u] = e < ncand ? __ldcg(ck + e) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = base + u * blockDim.x + tid;
        uint32_t dig = 0xFFFFFFFFu;
        if (e < ncand && (hi_excl >= 64 ? 0ull : (kk[u] >> hi_excl)) == pf)
          dig = static_cast<uint32_t>(kk[u] >> sh) & dmask;
        tks_add(hist, dig, lane);
      }
    }
    __syncthreads();
    tks_find_digit(hist, 1 << bits, need, ws, s_digit, s_above);
    const int dg = *s_digit;
    need -= *s_above;
    pf = (pf << bits) | static_cast<uint64_t>(dg);
    const int nbin = static_cast<int>(hist[dg]);
    __syncthreads();
    hi_excl = sh;
    if (nbin == need) { al = true; break; }
    if (sh == 0) break;
  }
  *prefix_io = pf;
  *sh_out = sh;
  *all = al;
}

__global__ void __launch_bounds__(TK_THREADS, 1) k_topk_stream(
    const DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int wb, int k,
    int weighted, const int32_t* __restrict__ clients, const int32_t* __restrict__ flags,
    uint32_t* __restrict__ bitmap, int32_t* __restrict__ count, uint32_t* __restrict__ idx_list,
    double* __restrict__ val_list, int cap, int32_t* __restrict__ draws,
    uint64_t* __restrict__ cand_key, int32_t* __restrict__ cand_pos, Emit em) {
  if (ctl && ctl->halt) return;
  if (threadIdx.x == 0) tl_mark(4, false);
  PhaseClock pc;
  extern __shared__ __align__(16) uint32_t tkst_dyn[];
  const int wi = static_cast<int>(w);
  uint32_t* gtm = tkst_dyn;        // [wb] selected (greater than the threshold)
  uint32_t* eqm = gtm + wb;        // [wb] tied with the threshold key
  uint32_t* hist = eqm + wb;       // [2048]
  uint64_t* skey = reinterpret_cast<uint64_t*>(hist + 2048);  // [TKST_SAMPLE]
  __shared__ int ws[64];
  __shared__ int s_digit, s_above, s_ncand, s_G, s_Z, s_fail;
  __shared__ int s_hhi, s_hlo, s_zero;
  __shared__ int w_sel[TK_NW], w_eqc[TK_NW];
  const int c = client_of(clients, blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* v = D + static_cast<int64_t>(c) * w;
  uint32_t* brow = bitmap + static_cast<int64_t>(c) * wb;
  uint64_t* ck = cand_key + static_cast<int64_t>(c) * TKST_CAP;
  int32_t* cp = cand_pos + static_cast<int64_t>(c) * TKST_CAP;
  if (tid == 0 && draws) draws[c] = 0;
  if (!(flags[c] & 2)) {
    clear_row(brow, wb);
    emit_empty(em, c);
    if (tid == 0) count[c] = 0;
    return;
  }
  // ---- 1. window from a strided sample: the sample's key high words at the
  //      two ranks ri -/+ delta, to 22 bits by two 11-bit radix levels
  //      (rounded outwards: a slightly wider window, never a narrower one)
  {
    uint32_t sk[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = u * TK_THREADS + tid;
      const int64_t ts = (static_cast<int64_t>(i) * w) / TKST_SAMPLE;
      sk[u] = key_hi(__ldg(v + ts), ts, weighted);
    }
    uint32_t* hist2 = reinterpret_cast<uint32_t*>(skey);  // [2048] second histogram
    for (int i = tid; i < wb; i += TK_THREADS) eqm[i] = 0u;
    for (int i = tid; i < 2048; i += TK_THREADS) { hist[i] = 0u; hist2[i] = 0u; }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) tks_add(hist, sk[u] >> 21, lane);
    __syncthreads();
    const double r = static_cast<double>(k) * TKST_SAMPLE / static_cast<double>(w);
    const int delta = static_cast<int>(4.0 * sqrt(r) + 16.0);
    const int ri = static_cast<int>(r);
    const int r_hi = ri - delta, r_lo = ri + delta;  // ranks in descending order
    const bool has_hi = r_hi >= 0, has_lo = r_lo < TKST_SAMPLE;
    int d1_hi = 0, d1_lo = 0, need_hi = r_hi + 1, need_lo = r_lo + 1;
    if (has_hi) {
      tks_find_digit(hist, 2048, need_hi, ws, &s_digit, &s_above);
      d1_hi = s_digit;
      need_hi -= s_above;
      __syncthreads();
    }
    if (has_lo) {
      tks_find_digit(hist, 2048, need_lo, ws, &s_digit, &s_above);
      d1_lo = s_digit;
      need_lo -= s_above;
      __syncthreads();
    }
    // level 2: bits 20..10 of the keys in the two level-1 bins
    for (int i = tid; i < 2048; i += TK_THREADS) hist[i] = 0u;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t top = sk[u] >> 21, dg = (sk[u] >> 10) & 2047u;
      tks_add(hist, (has_hi && top == static_cast<uint32_t>(d1_hi)) ? dg : 0xFFFFFFFFu, lane);
      tks_add(hist2, (has_lo && top == static_cast<uint32_t>(d1_lo)) ? dg : 0xFFFFFFFFu, lane);
    }
    __syncthreads();
    int hhi = 0x7FFFFFFF, hlo = -1;
    if (has_hi) {
      tks_find_digit(hist, 2048, need_hi, ws, &s_digit, &s_above);
      hhi = static_cast<int>((static_cast<uint32_t>(d1_hi) << 21) | (static_cast<uint32_t>(s_digit) << 10) | 1023u);
      __syncthreads();
    }
    if (has_lo) {
      tks_find_digit(hist2, 2048, need_lo, ws, &s_digit, &s_above);
      hlo = static_cast<int>((static_cast<uint32_t>(d1_lo) << 21) | (static_cast<uint32_t>(s_digit) << 10)) - 1;
      __syncthreads();
    }
    if (tid == 0) {
      // high words: gt iff hk > hhi; candidate iff hlo < hk <= hhi (signed)
      if (hlo >= hhi) hlo = hhi - 1;
      // exact zeros become a tie class when the window reaches them
      s_zero = hlo < 0;
      if (hlo < 0) hlo = -1;
      s_hhi = hhi;
      s_hlo = hlo;
      s_ncand = 0;
      s_G = 0;
      s_Z = 0;
      s_fail = 0;
    }
    __syncthreads();
  }
  pc.mark(0);
  const int hhi = s_hhi, hlo = s_hlo;
  const bool track_zero = s_zero;
  // ---- 2. one classification pass over D
  constexpr int UNR = 8;
  {
    int z_acc = 0;
    for (int base = 0; base < wi; base += UNR * TK_THREADS) {
      double x[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int t = base + u * TK_THREADS + tid;
        x[u] = (t < wi) ? __ldcs(v + t) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int t = base + u * TK_THREADS + tid;
        const uint64_t key = rank_key(x[u], t, weighted);
        const int hk = (t < wi) ? static_cast<int>(key >> 32) : -2;
        const bool gt = hk > hhi;
        bool mid = hk > hlo && hk <= hhi;
        if (track_zero) {
          const bool z = t < wi && key == 0ull;
          mid = mid && !z;
          const uint32_t zb = __ballot_sync(0xffffffffu, z);
          if (lane == 0 && t - lane < wi) { eqm[t >> 5] = zb; z_acc += __popc(zb); }
        }
        const uint32_t gb = __ballot_sync(0xffffffffu, gt);
        const uint32_t mb = __ballot_sync(0xffffffffu, mid);
        if (lane == 0 && t - lane < wi) gtm[t >> 5] = gb;  // the word is owned by this warp
        if (mb) {
          int wbase = 0;
          if (lane == 0) wbase = atomicAdd(&s_ncand, __popc(mb));
          wbase = __shfl_sync(0xffffffffu, wbase, 0);
          if (mid) {
            const int slot = wbase + __popc(mb & ((1u << lane) - 1u));
            if (slot < TKST_CAP) {
              ck[slot] = key;
              cp[slot] = t;
            }
          }
        }
      }
    }
    if (track_zero && lane == 0) atomicAdd(&s_Z, z_acc);
    __syncthreads();
    // G = number of gt bits (a cheap sweep over the bitmap)
    int g = 0;
    for (int q = tid; q < wb; q += TK_THREADS) g += __popc(gtm[q]);
    g = warp_sum_int(g);
    if (lane == 0) atomicAdd(&s_G, g);
    __syncthreads();
  }
  pc.mark(1);
  // ---- 3. decide where the k-th key is
  int need = k;  // after this block: number of eq-class keys to take by position
  {
    const int G = s_G, M = s_ncand, Z = track_zero ? s_Z : 0;
    const bool ok = G < k && G + M + Z >= k && M <= TKST_CAP;
    if (ok && G + M >= k) {
      // the k-th key is a candidate; zeros (if tracked) are not needed
      if (track_zero)
        for (int i = tid; i < wb; i += TK_THREADS) eqm[i] = 0u;
      need = k - G;
      __syncthreads();
      const int top = 32 + (31 - __clz(static_cast<unsigned>((hlo + 1) ^ hhi) | 1u));
      uint64_t pf = static_cast<uint64_t>(static_cast<uint32_t>(hhi)) >> (top - 31);
      int sh;
      bool all;
      tkst_resolve(ck, M, top, need, hist, ws, &s_digit, &s_above, &pf, &sh, &all);
      for (int e = tid; e < M; e += TK_THREADS) {
        const uint64_t hp = __ldcg(ck + e) >> sh;
        const int t = __ldcg(cp + e);
        if (hp > pf || (all && hp == pf)) atomicOr(&gtm[t >> 5], 1u << (t & 31));
        else if (hp == pf) atomicOr(&eqm[t >> 5], 1u << (t & 31));
      }
      if (all) need = 0;
      __syncthreads();
    } else if (ok) {
      // every candidate is taken; the first k - G - M zeros complete the set
      for (int e = tid; e < M; e += TK_THREADS) {
        const int t = __ldcg(cp + e);
        atomicOr(&gtm[t >> 5], 1u << (t & 31));
      }
      need = k - G - M;
      __syncthreads();
    } else {
      // the window missed: radix levels over D itself
      if (tid == 0) s_fail = 1;
      constexpr int NL = 6;
      constexpr int SH[NL] = {52, 41, 30, 19, 8, 0};
      constexpr int BI[NL] = {11, 11, 11, 11, 11, 8};
      uint64_t prefix = 0;
      int L = 0;
      bool take_all = false;
      for (; L < NL; ++L) {
        for (int i = tid; i < 2048; i += TK_THREADS) hist[i] = 0u;
        __syncthreads();
        const int sh = SH[L], up = (L == 0) ? 63 : SH[L - 1];
        const uint32_t dmask = (1u << BI[L]) - 1u;
        for (int base = 0; base < wi; base += TK_THREADS) {  // warp-uniform trip count (ballots)
          const int t = base + tid;
          uint32_t dig = 0xFFFFFFFFu;
          if (t < wi) {
            const uint64_t key = rank_key(__ldcs(v + t), t, weighted);
            if ((up >= 63 ? 0ull : (key >> up)) == prefix) dig = static_cast<uint32_t>(key >> sh) & dmask;
          }
          tks_add(hist, dig, lane);
        }
        __syncthreads();
        tks_find_digit(hist, 1 << BI[L], need, ws, &s_digit, &s_above);
        const int dg = s_digit;
        need -= s_above;
        prefix = (prefix << BI[L]) | static_cast<uint64_t>(dg);
        const int nbin = static_cast<int>(hist[dg]);
        __syncthreads();
        if (nbin == need) { take_all = true; break; }
      }
      if (L == NL) L = NL - 1;
      const int sh = SH[L];
      for (int base = 0; base < wi; base += TK_THREADS) {
        const int t = base + tid;
        bool gt = false, eq = false;
        if (t < wi) {
          const uint64_t hp = rank_key(__ldcs(v + t), t, weighted) >> sh;
          gt = take_all ? hp >= prefix : hp > prefix;
          eq = !take_all && hp == prefix;
        }
        const uint32_t gb = __ballot_sync(0xffffffffu, gt), eb = __ballot_sync(0xffffffffu, eq);
        if (lane == 0 && t - lane < wi) { gtm[t >> 5] = gb; eqm[t >> 5] = eb; }
      }
      if (take_all) need = 0;
      __syncthreads();
    }
  }
  pc.mark(2);
  // ---- 4. selection: lane = one bitmap word; a warp covers 32 words per step
  //         and owns the contiguous word range [warp * SW, (warp + 1) * SW)
  const int SW = (wb + TK_NW - 1) / TK_NW;
  const int q0 = warp * SW, q1 = min(wb, q0 + SW);
  {
    int ns = 0, ne = 0;
    for (int q = q0 + lane; q < q1; q += 32) {
      ns += __popc(gtm[q]);
      ne += __popc(eqm[q]);
    }
    ns = warp_sum_int(ns);
    ne = warp_sum_int(ne);
    if (lane == 0) { w_sel[warp] = ns; w_eqc[warp] = ne; }
  }
  __syncthreads();
  if (warp == 0) {
    const int g = w_sel[lane], e = w_eqc[lane];
    int e_incl = e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, e_incl, o);
      if (lane >= o) e_incl += y;
    }
    const int e_excl = e_incl - e;
    const int e_take = max(0, min(need - e_excl, e));
    const int sel = g + e_take;
    int s_incl = sel;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s_incl, o);
      if (lane >= o) s_incl += y;
    }
    w_sel[lane] = s_incl - sel;  // exclusive selected prefix
    w_eqc[lane] = e_excl;        // exclusive tied prefix
    if (lane == 31) s_above = s_incl;
  }
  __syncthreads();
  const int total = s_above;
  uint32_t* il = idx_list + static_cast<int64_t>(c) * cap;
  double* vl = val_list + static_cast<int64_t>(c) * cap;
  int32_t* rsc = em.rs ? em.rs + static_cast<int64_t>(c) * (em.nr + 1) : nullptr;
  {
    int base_sel = w_sel[warp], base_eq = w_eqc[warp];
    for (int qb = q0; qb < q1; qb += 32) {
      const int q = qb + lane;
      uint32_t gb = 0u, eb = 0u;
      if (q < q1) { gb = gtm[q]; eb = eqm[q]; }
      const int ne = __popc(eb);
      int e_pre = ne;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, e_pre, o);
        if (lane >= o) e_pre += y;
      }
      const int e_tot = __shfl_sync(0xffffffffu, e_pre, 31);
      e_pre -= ne;
      int take = max(0, min(need - (base_eq + e_pre), ne));
      uint32_t sel = gb;
      for (uint32_t m = eb; take > 0; --take) {
        const uint32_t low = m & (0u - m);
        sel |= low;
        m ^= low;
      }
      const int ns = __popc(sel);
      int s_pre = ns;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, s_pre, o);
        if (lane >= o) s_pre += y;
      }
      const int s_tot = __shfl_sync(0xffffffffu, s_pre, 31);
      s_pre -= ns;
      int pos = base_sel + s_pre;
      if (q < q1) {
        if (rsc && (q % (FOLD_RANGE / 32)) == 0) rsc[q / (FOLD_RANGE / 32)] = pos;
        brow[q] = sel;
        for (uint32_t m = sel; m; m &= m - 1) il[pos++] = static_cast<uint32_t>(q * 32 + __ffs(m) - 1);
      }
      base_sel += s_tot;
      base_eq += e_tot;
    }
  }
  if (tid == 0) {
    count[c] = total;
    if (rsc) rsc[em.nr] = total;
  }
  __syncthreads();
  pc.mark(3);
  // ---- values and the client shift update: 8 independent entries per thread
  for (int e0 = 0; e0 < total; e0 += 8 * TK_THREADS) {
    int64_t tt[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * TK_THREADS + tid;
      tt[u] = e < total ? static_cast<int64_t>(__ldcg(il + e)) : -1;
    }
    double vv[8], hv[8];
    double* hrow = em.hest ? em.hest + static_cast<int64_t>(c) * em.hest_stride : nullptr;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      vv[u] = tt[u] >= 0 ? __ldg(v + tt[u]) : 0.0;
      hv[u] = (hrow && tt[u] >= 0) ? hrow[tt[u]] : 0.0;  // positions are distinct
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * TK_THREADS + tid;
      if (tt[u] >= 0) {
        vl[e] = vv[u];
        if (hrow) hrow[tt[u]] = __dadd_rn(hv[u], __dmul_rn(em.alpha, vv[u]));  // emit_entry
      }
    }
  }
  pc.mark(4);
  if (g_dbg_on && tid == 0 && s_fail) atomicAdd(reinterpret_cast<unsigned long long*>(&g_dbg[17]), 1ull);
  if (tid == 0) tl_mark(4, true);
}

// ------------------------------------------- TopK, split streaming path
// The same selection rule as k_topk_stream (descending key, ties to the
// smaller position), as three kernels so the one pass over D is spread over
// many CTAs that each keep a TMA ring of D in flight:
//  1. k_tks_window (CTA per client): a sample of `ns` keys (ns/8 runs of 8
//     consecutive positions spread over the row) gives the key
//     high-word window (hlo, hhi] around the k-th key;
//  2. k_tks_pass (grid segments x clients): one producer thread streams the
//     segment of D into a shared-memory ring with 1-D bulk copies
//     (cp.async.bulk, mbarrier transaction counts); 16 consumer warps
//     classify each key: above the window -> gt bit (warp ballot = bitmap
//     word), inside -> the segment's candidate slots, exact zeros -> zero bit
//     (only when the window reaches zero); per-segment counts (G, M, Z).  The
//     gt and zero/tie rows are scratch that is all-zero between rounds, so
//     only nonzero words are stored;
//  3. k_tks_select (CTA per client): the gt row into shared memory (and the
//     global row cleared), the k-th key by radix levels over the candidates
//     (the first level over the candidate list in L2, the threshold digit's
//     survivors compacted into shared memory for the rest), marks by shared
//     atomics, then one sweep (contiguous words per thread, block scans) that
//     takes the first `need` tied positions and writes the list, range
//     starts, values and the client shift update.
// A window miss (G >= k, G + M (+ Z) < k) or a segment overflowing its
// candidate slots falls back to radix levels over D inside k_tks_select.
constexpr int TKP_CONS = 512;                  // consumer threads
constexpr int TKP_THREADS = TKP_CONS + 32;     // + the producer warp
constexpr int TKP_CW = TKP_CONS / 32;          // consumer warps (list regions per segment)
constexpr int TKP_CH = 2048;                   // positions per ring stage (16 KB)
constexpr int TKP_NST = 6;                     // ring stages
constexpr int TKP_STRIDE = TKP_CH + 2;         // stage stride (16-byte aligned, +1 lead)
constexpr int TKP_CH2 = 4096;                  // merged-list layout: positions per stage (32 KB)
constexpr int TKP_NST2 = 3;                    //   ring stages
constexpr size_t TKP_SMEM1 = static_cast<size_t>(TKP_NST) * TKP_STRIDE * 8;
constexpr size_t TKP_SMEM2 = static_cast<size_t>(TKP_NST2) * TKP_CH2 * 8;
constexpr size_t TKP_SMEM = TKP_SMEM1 > TKP_SMEM2 ? TKP_SMEM1 : TKP_SMEM2;
static_assert(TKP_NST2 <= TKP_NST, "the merged layout reuses the ring's barriers");
constexpr int TKP_SEGCAP = 16384;              // candidate slots per segment (max)
constexpr int TKP_MAXSEG = 16;                 // segments per client (max)
constexpr int TKP_MAXSUB = TKP_MAXSEG * TKP_CONS / 32;  // list regions per client (max)
constexpr int TKSEL_THREADS = 512;
constexpr int TKSEL_LCAP = 2048;               // threshold-digit survivors kept in smem
constexpr int TKW_THREADS = 512;
constexpr int TKW_MAXSAMPLE = 16 * TKW_THREADS;
__host__ __device__ constexpr int tks_wbp(int64_t w) {  // bitmap row stride (16-byte rows)
  return static_cast<int>(((w + 31) / 32 + 3) / 4 * 4);
}
__host__ __device__ constexpr size_t tksel_smem_bytes(int64_t w) {
  return static_cast<size_t>(tks_wbp(w)) * 4 +
         ((static_cast<size_t>(tks_wbp(w)) / 8 + 1) * 4 > TKSEL_LCAP * 12
              ? (static_cast<size_t>(tks_wbp(w)) / 8 + 1) * 4
              : TKSEL_LCAP * 12);
}

__host__ __device__ constexpr size_t tkp_smem_bytes(int64_t w) {  // ring, then the selection
  return TKP_SMEM > tksel_smem_bytes(w) ? TKP_SMEM : tksel_smem_bytes(w);
}

struct TkWin {
  int hhi, hlo, zero, active;
};
struct TkSeg {
  int g, m, z, pad;
};

// the digit holding the need-th largest element of hist[0, nbins) (counting
// from the top bin), any blockDim multiple of 32 with nbins <= 4 * blockDim
__device__ __forceinline__ void tk_find_digit_n(const uint32_t* hist, int nbins, int need, int* ws,
                                                int* s_digit, int* s_above) {
  const int per = (nbins + static_cast<int>(blockDim.x) - 1) / static_cast<int>(blockDim.x);
  const int b0 = nbins - 1 - per * static_cast<int>(threadIdx.x);
  int cnt[4], sum = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int b = b0 - i;
    cnt[i] = (i < per && b >= 0) ? static_cast<int>(hist[b]) : 0;
    sum += cnt[i];
  }
  int total;
  int above = block_excl_scan(sum, ws, &total);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (cnt[i] > 0 && above < need && need <= above + cnt[i]) {
      *s_digit = b0 - i;
      *s_above = above;
    }
    above += cnt[i];
  }
  __syncthreads();
}

// sample position i of ns: run j = i / 8 of ns / 8 runs of 8 consecutive
// positions (two full sectors) spread evenly over the row
__host__ __device__ __forceinline__ int64_t tks_sample_pos(int i, int ns, int64_t w) {
  const int64_t runs = ns / 8;
  return (static_cast<int64_t>(i >> 3) * (w - 8)) / runs + (i & 7);
}

__global__ void __launch_bounds__(TKW_THREADS, 2) k_tks_window(
    const DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int k, int ns,
    int weighted, const int32_t* __restrict__ clients, const int32_t* __restrict__ flags,
    int32_t* __restrict__ draws, TkWin* __restrict__ win, int32_t* __restrict__ ticket,
    int32_t* __restrict__ count, Emit em) {
  const int c = client_of(clients, blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) ticket[c] = 0;  // the pass CTAs of this round count in from zero
  if (ctl && ctl->halt) return;
  __shared__ uint32_t hist[2048], hist2[2048];
  __shared__ int ws[64];
  __shared__ int s_digit, s_above;
  if (tid == 0 && draws) draws[c] = 0;
  if (!(flags[c] & 2)) {  // all-zero difference: empty delta, no draws
    if (tid == 0) {
      win[c] = TkWin{0, 0, 0, 0};
      count[c] = 0;
    }
    emit_empty(em, c);
    return;
  }
  const double* v = D + static_cast<int64_t>(c) * w;
  constexpr int SPT = TKW_MAXSAMPLE / TKW_THREADS;
  uint32_t sk[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) {
    const int i = u * TKW_THREADS + tid;
    const int64_t ts = tks_sample_pos(i, ns, w);
    sk[u] = i < ns ? static_cast<uint32_t>(rank_key(__ldg(v + ts), ts, weighted) >> 32) : 0u;
  }
  for (int i = tid; i < 2048; i += TKW_THREADS) { hist[i] = 0u; hist2[i] = 0u; }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < SPT; ++u)
    tks_add(hist, (u * TKW_THREADS + tid < ns) ? (sk[u] >> 21) : 0xFFFFFFFFu, lane);
  __syncthreads();
  const double r = static_cast<double>(k) * ns / static_cast<double>(w);
  const int delta = static_cast<int>(4.0 * sqrt(r) + 16.0);
  const int ri = static_cast<int>(r);
  const int r_hi = ri - delta, r_lo = ri + delta;  // ranks in descending order
  const bool has_hi = r_hi >= 0, has_lo = r_lo < ns;
  int d1_hi = 0, d1_lo = 0, need_hi = r_hi + 1, need_lo = r_lo + 1;
  if (has_hi) {
    tk_find_digit_n(hist, 2048, need_hi, ws, &s_digit, &s_above);
    d1_hi = s_digit;
    need_hi -= s_above;
    __syncthreads();
  }
  if (has_lo) {
    tk_find_digit_n(hist, 2048, need_lo, ws, &s_digit, &s_above);
    d1_lo = s_digit;
    need_lo -= s_above;
    __syncthreads();
  }
  for (int i = tid; i < 2048; i += TKW_THREADS) hist[i] = 0u;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < SPT; ++u) {
    const bool in = u * TKW_THREADS + tid < ns;
    const uint32_t top = sk[u] >> 21, dg = (sk[u] >> 10) & 2047u;
    tks_add(hist, (in && has_hi && top == static_cast<uint32_t>(d1_hi)) ? dg : 0xFFFFFFFFu, lane);
    tks_add(hist2, (in && has_lo && top == static_cast<uint32_t>(d1_lo)) ? dg : 0xFFFFFFFFu, lane);
  }
  __syncthreads();
  int hhi = 0x7FFFFFFF, hlo = -1;
  if (has_hi) {
    tk_find_digit_n(hist, 2048, need_hi, ws, &s_digit, &s_above);
    hhi = static_cast<int>((static_cast<uint32_t>(d1_hi) << 21) | (static_cast<uint32_t>(s_digit) << 10) | 1023u);
    __syncthreads();
  }
  if (has_lo) {
    tk_find_digit_n(hist2, 2048, need_lo, ws, &s_digit, &s_above);
    hlo = static_cast<int>((static_cast<uint32_t>(d1_lo) << 21) | (static_cast<uint32_t>(s_digit) << 10)) - 1;
    __syncthreads();
  }
  if (tid == 0) {
    if (hlo >= hhi) hlo = hhi - 1;
    const int zero = hlo < 0;  // exact zeros become a tie class when the window reaches them
    win[c] = TkWin{hhi, zero ? -1 : hlo, zero, 1};
  }
}

__device__ __forceinline__ void mbar_wait_short(uint64_t* bar, uint32_t parity) {
  for (uint32_t spin = 0; !mbar_try_wait(bar, parity); ++spin) {
    if (spin > (1u << 20)) asm volatile("trap;");
  }
}

__device__ __forceinline__ void bar_sync_named(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One ring stage (TKP_CH positions) of one consumer warp's share: keys from
// shared memory, gt / zero bitmap words, and (position, raw value) appends
// to the warp's own list regions (warp-uniform running counts: no atomics).
template <bool W, bool Z, bool CHECK>
__device__ __forceinline__ void tkp_stage(const double* __restrict__ rb, int base, int t1, int hhi,
                                          int hlo, int tid, int lane, uint32_t* __restrict__ zrow, uint64_t* __restrict__ ck,
                                          int32_t* __restrict__ cp, uint64_t* __restrict__ gk,
                                          int32_t* __restrict__ gq, int capw, int& m_cnt,
                                          int& g_cnt, int& z_cnt) {
  constexpr int EPT = TKP_CH / TKP_CONS;
  uint64_t bits[EPT];
  uint32_t gb[EPT], mb[EPT];
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int tl = u * TKP_CONS + tid;
    const int t = base + tl;
    const double x = rb[tl];
    bits[u] = static_cast<uint64_t>(__double_as_longlong(x));
    const uint64_t key = W ? rank_key(x, t, 1) : (bits[u] & 0x7FFFFFFFFFFFFFFFull);
    int hk = static_cast<int>(key >> 32);
    if (CHECK && t >= t1) hk = -2;
    const bool gt = hk > hhi;
    bool mid = hk > hlo && hk <= hhi;
    if (Z) {
      const bool z = (!CHECK || t < t1) && key == 0ull;
      mid = mid && !z;
      const uint32_t zb = __ballot_sync(0xffffffffu, z);
      if (lane == 0 && zb) zrow[t >> 5] = zb;
      z_cnt += __popc(zb);
    }
    gb[u] = __ballot_sync(0xffffffffu, gt);
    mb[u] = __ballot_sync(0xffffffffu, mid);
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int t = base + u * TKP_CONS + tid;
    if (gb[u]) {
      if ((gb[u] >> lane) & 1u) {
        const int slot = g_cnt + __popc(gb[u] & lt);
        if (slot < capw) { gk[slot] = bits[u]; gq[slot] = t; }
      }
      g_cnt += __popc(gb[u]);
    }
    if (mb[u]) {
      if ((mb[u] >> lane) & 1u) {
        const int slot = m_cnt + __popc(mb[u] & lt);
        if (slot < capw) { ck[slot] = bits[u]; cp[slot] = t; }
      }
      m_cnt += __popc(mb[u]);
    }
  }
}

template <bool W, bool Z>
__device__ __forceinline__ void tkp_consume(const double* ring, uint64_t* full, uint64_t* empty,
                                            int nch, int lead, int t0, int t1, int hhi, int hlo,
                                            int tid, int lane, uint32_t* zrow,
                                            uint64_t* ck, int32_t* cp, uint64_t* gk, int32_t* gq,
                                            int capw, int& m_cnt, int& g_cnt, int& z_cnt) {
  for (int i = 0; i < nch; ++i) {
    const int st = i % TKP_NST;
    mbar_wait_short(&full[st], (i / TKP_NST) & 1);
    const double* rb = ring + st * TKP_STRIDE + lead;
    const int base = t0 + i * TKP_CH;
    if (base + TKP_CH <= t1)
      tkp_stage<W, Z, false>(rb, base, t1, hhi, hlo, tid, lane, zrow, ck, cp, gk, gq, capw, m_cnt,
                             g_cnt, z_cnt);
    else
      tkp_stage<W, Z, true>(rb, base, t1, hhi, hlo, tid, lane, zrow, ck, cp, gk, gq, capw, m_cnt,
                            g_cnt, z_cnt);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}


// Merged-list layout (no zero tie class): ring stages of TKP_CH2 positions
// starting at the segment's 16-byte aligned position `a0`; a consumer warp
// owns a contiguous 1/TKP_CW slice of every stage.  Each lane reads its
// elements as 16-byte pairs (pair j * 32 + lane of the slice: conflict-free),
// keeps one bit per element whose key high word exceeds the window's lower
// end (above the window and inside it alike: the selection tells them apart),
// and the warp appends the flagged (position, raw value) entries to its list
// region once per stage in rounds: every lane that still holds a flagged
// element writes one per round (values re-read from the stage).
template <bool W, bool CHECK>
__device__ __forceinline__ void tkp_stage_m(const double* __restrict__ wb_, int pos0, int t0, int t1,
                                            int hlo, int lane, uint64_t* __restrict__ ck,
                                            int32_t* __restrict__ cp, int capw, int& m_cnt) {
  constexpr int PPL = TKP_CH2 / TKP_CW / 64;  // pairs per lane per stage
  static_assert(PPL * 2 <= 32, "one mask bit per element");
  const double2* pr = reinterpret_cast<const double2*>(wb_);
  double2 x[PPL];
#pragma unroll
  for (int j = 0; j < PPL; ++j) x[j] = pr[j * 32 + lane];
  uint32_t mask = 0u;
#pragma unroll
  for (int j = 0; j < PPL; ++j) {
    const int t = pos0 + 2 * (j * 32 + lane);
    int h0, h1;
    if (W) {
      h0 = static_cast<int>(rank_key(x[j].x, t, 1) >> 32);
      h1 = static_cast<int>(rank_key(x[j].y, t + 1, 1) >> 32);
    } else {
      h0 = __double2hiint(x[j].x) & 0x7FFFFFFF;
      h1 = __double2hiint(x[j].y) & 0x7FFFFFFF;
    }
    bool c0 = h0 > hlo, c1 = h1 > hlo;
    if (CHECK) {
      c0 = c0 && t >= t0 && t < t1;
      c1 = c1 && t + 1 >= t0 && t + 1 < t1;
    }
    if (c0) mask |= 1u << (2 * j);
    if (c1) mask |= 2u << (2 * j);
  }
  // append rounds: in round r every lane that still has a flagged element
  // emits one (slot = running count + the rank of the lane among them)
  const uint32_t lt = (1u << lane) - 1u;
  for (;;) {
    const uint32_t hb = __ballot_sync(0xffffffffu, mask != 0u);
    if (!hb) break;
    if (mask) {
      const int b = __ffs(mask) - 1;
      mask &= mask - 1u;
      const int e = 2 * ((b >> 1) * 32 + lane) + (b & 1);
      const int slot = m_cnt + __popc(hb & lt);
      if (slot < capw) {
        ck[slot] = static_cast<uint64_t>(__double_as_longlong(wb_[e]));
        cp[slot] = pos0 + e;
      }
    }
    m_cnt += __popc(hb);
  }
}

template <bool W>
__device__ __forceinline__ void tkp_consume_m(const double* ring, uint64_t* full, uint64_t* empty,
                                              int nch, int a0, int t0, int t1, int hlo, int warp,
                                              int lane, uint64_t* ck, int32_t* cp, int capw,
                                              int& m_cnt) {
  constexpr int SL = TKP_CH2 / TKP_CW;  // the warp's slice of a stage
  int st = 0;
  uint32_t par = 0;
  const double* wb_ = ring + warp * SL;
  int pos0 = a0 + warp * SL;
  for (int i = 0; i < nch; ++i) {
    mbar_wait_short(&full[st], par);
    const int cb = pos0 - warp * SL;
    if (cb >= t0 && cb + TKP_CH2 <= t1)
      tkp_stage_m<W, false>(wb_ + st * TKP_CH2, pos0, t0, t1, hlo, lane, ck, cp, capw, m_cnt);
    else
      tkp_stage_m<W, true>(wb_ + st * TKP_CH2, pos0, t0, t1, hlo, lane, ck, cp, capw, m_cnt);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    pos0 += TKP_CH2;
    if (++st == TKP_NST2) { st = 0; par ^= 1u; }
  }
}

__device__ __noinline__ void tks_select_client(
    int c, uint32_t* sg, const double* __restrict__ D, int64_t w, int wbp, int k, int weighted,
    int S_seg, int capw, const int32_t* __restrict__ clients, const TkWin* __restrict__ win,
    const TkSeg* __restrict__ seg, uint32_t* __restrict__ eqz, const uint64_t* __restrict__ cand_key,
    const int32_t* __restrict__ cand_pos, const uint64_t* __restrict__ gt_val,
    const int32_t* __restrict__ gt_pos, int32_t* __restrict__ count, uint32_t* __restrict__ idx_list,
    double* __restrict__ val_list, int cap, Emit em);
static_assert(FOLD_RANGE == 8 * 32, "the selection's 8-word rank groups are the fold's ranges");

// seg[(c * S + s) * TKP_CW + warp] = (G, M, Z) of one consumer warp's share;
// its list region is slots [((c * S + s) * TKP_CW + warp) * capw, + capw)
template <bool W>
__global__ void __launch_bounds__(TKP_THREADS) k_tks_pass(
    const DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int wbp, int lseg,
    int capw, const int32_t* __restrict__ clients, const TkWin* __restrict__ win,
    uint32_t* __restrict__ eqz, uint64_t* __restrict__ cand_key, int32_t* __restrict__ cand_pos,
    uint64_t* __restrict__ gt_val, int32_t* __restrict__ gt_pos, TkSeg* __restrict__ seg,
    int32_t* __restrict__ ticket, int k, int32_t* __restrict__ count, uint32_t* __restrict__ idx_list,
    double* __restrict__ val_list, int cap, Emit em) {
  if (ctl && ctl->halt) return;
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[TKP_NST], empty[TKP_NST];
  __shared__ int s_last;
  const int c = client_of(clients, blockIdx.y);
  const TkWin wn = win[c];
  if (!wn.active) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int S = gridDim.x, s = blockIdx.x;
  const int wi = static_cast<int>(w);
  const int t0 = s * lseg, t1 = min(wi, t0 + lseg);
  const double* v = D + static_cast<int64_t>(c) * w;
  // bulk copies need 16-byte aligned sources: start one position early on odd rows
  const int lead = static_cast<int>((reinterpret_cast<uintptr_t>(v + t0) & 15u) >> 3);
  // no zero tie class: the merged-list layout (aligned stages of TKP_CH2)
  const bool merged = !wn.zero;
  const int a0 = t0 - lead;
  const int nch = merged ? (t1 - a0 + TKP_CH2 - 1) / TKP_CH2 : (t1 - t0 + TKP_CH - 1) / TKP_CH;
  if (tid == 0) {
    for (int i = 0; i < TKP_NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], TKP_CW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == TKP_CW) {  // producer
    if (lane == 0 && merged) {
      for (int i = 0; i < nch; ++i) {
        const int st = i % TKP_NST2;
        if (i >= TKP_NST2) mbar_wait_short(&empty[st], ((i / TKP_NST2) - 1) & 1);
        const int nel = min(TKP_CH2, t1 - a0 - i * TKP_CH2);
        const uint32_t bytes = static_cast<uint32_t>((nel + 1) & ~1) * 8u;
        mbar_arrive_expect_tx(&full[st], bytes);
        bulk_load(ring + st * TKP_CH2, v + a0 + i * TKP_CH2, bytes, &full[st]);
      }
    } else if (lane == 0) {
      for (int i = 0; i < nch; ++i) {
        const int st = i % TKP_NST;
        if (i >= TKP_NST) mbar_wait_short(&empty[st], ((i / TKP_NST) - 1) & 1);
        const int nel = min(TKP_CH, t1 - t0 - i * TKP_CH) + lead;
        const uint32_t bytes = static_cast<uint32_t>((nel + 1) & ~1) * 8u;
        mbar_arrive_expect_tx(&full[st], bytes);
        bulk_load(ring + st * TKP_STRIDE, v + t0 + i * TKP_CH - lead, bytes, &full[st]);
      }
    }
  } else {
  uint32_t* zrow = eqz + static_cast<int64_t>(c) * wbp;
  const int64_t sub = (static_cast<int64_t>(c) * S + s) * TKP_CW + warp;
  const int64_t lbase = sub * capw;
  int m_cnt = 0, g_cnt = 0, z_cnt = 0;
  if (wn.zero)
    tkp_consume<W, true>(ring, full, empty, nch, lead, t0, t1, wn.hhi, wn.hlo, tid, lane, zrow,
                         cand_key + lbase, cand_pos + lbase, gt_val + lbase, gt_pos + lbase, capw,
                         m_cnt, g_cnt, z_cnt);
  else
    tkp_consume_m<W>(ring, full, empty, nch, a0, t0, t1, wn.hlo, warp, lane, cand_key + lbase,
                     cand_pos + lbase, capw, m_cnt);
  if (lane == 0) seg[sub] = TkSeg{g_cnt, m_cnt, z_cnt, 0};
  }
  // the last of the client's segment CTAs to finish runs its selection (the
  // ring is free again: its shared memory becomes the selection row)
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&ticket[c], 1) == S - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  tks_select_client(c, reinterpret_cast<uint32_t*>(ring), D, w, wbp, k, W ? 1 : 0, S, capw, clients,
                    win, seg, eqz, cand_key, cand_pos, gt_val, gt_pos, count, idx_list, val_list,
                    cap, em);
}

// radix levels over candidate keys (source `get(e)` for e < cnt) whose bits
// >= hi_excl equal pf: 11-bit digits downwards, at most `max_levels`.
// Returns with pf extended by the chosen digits, sh = the bit position of the
// last digit, need reduced by the counts above, all = the last bin is taken
// whole.
template <class Get>
__device__ void tksel_levels(Get get, int cnt, int& hi_excl, uint64_t& pf, int& need, int& sh,
                             bool& all, int max_levels, uint32_t* hist, int* ws, int* s_digit,
                             int* s_above) {
  const int tid = threadIdx.x, lane = tid & 31;
  all = false;
  for (int lv = 0; lv < max_levels && hi_excl > 0; ++lv) {
    const int bits = min(11, hi_excl);
    sh = hi_excl - bits;
    for (int i = tid; i < 2048; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const uint32_t dmask = (1u << bits) - 1u;
    for (int base = 0; base < cnt; base += 4 * blockDim.x) {
      uint64_t kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = base + u * blockDim.x + tid;
        kk[u] = e < cnt ? get(e) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = base + u * blockDim.x + tid;
        uint32_t dig = 0xFFFFFFFFu;
        if (e < cnt && (hi_excl >= 64 ? 0ull : (kk[u] >> hi_excl)) == pf)
          dig = static_cast<uint32_t>(kk[u] >> sh) & dmask;
        tks_add(hist, dig, lane);
      }
    }
    __syncthreads();
    tk_find_digit_n(hist, 1 << bits, need, ws, s_digit, s_above);
    const int dg = *s_digit;
    need -= *s_above;
    pf = (pf << bits) | static_cast<uint64_t>(dg);
    const int nbin = static_cast<int>(hist[dg]);
    __syncthreads();
    hi_excl = sh;
    if (nbin == need) { all = true; break; }
  }
}

// Warp-per-region iteration over the per-(segment, warp) list regions of one
// client: region j holds cnt[j] entries at slots [j * capw, + cnt[j]).
// f(slot, valid) is called warp-uniformly, U slots per lane in flight.
template <int U, class F>
__device__ __forceinline__ void tksel_regions(const int* cnt, int nreg, int capw, F f) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < nreg; j += nw) {
    const int n = cnt[j];
    for (int i0 = 0; i0 < n; i0 += 32 * U) {
      int sl[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * 32 + lane;
        ok[u] = i < n;
        sl[u] = j * capw + (ok[u] ? i : 0);
      }
      f(sl, ok);
    }
  }
}

// The selection of one client, run by the last of its pass CTAs to finish
// (any blockDim multiple of 32, <= 1024; `sg` = the CTA's dynamic shared
// memory, tksel_smem_bytes(w) bytes).  Clients with an all-zero difference
// are emitted by k_tks_window.
__device__ __noinline__ void tks_select_client(
    int c, uint32_t* sg, const double* __restrict__ D, int64_t w, int wbp, int k, int weighted, int S_seg, int capw,
    const int32_t* __restrict__ clients, const TkWin* __restrict__ win, const TkSeg* __restrict__ seg,
    uint32_t* __restrict__ eqz, const uint64_t* __restrict__ cand_key,
    const int32_t* __restrict__ cand_pos, const uint64_t* __restrict__ gt_val,
    const int32_t* __restrict__ gt_pos, int32_t* __restrict__ count, uint32_t* __restrict__ idx_list,
    double* __restrict__ val_list, int cap, Emit em) {
  // dynamic: sg[wbp] u32 (the selection row) | union { lkey[LCAP] u64,
  //          lpos[LCAP] i32 (resolve) ; grp[wbp / 8 + 1] i32 (the rank of the
  //          first entry of every 8-word group, = the fold's range starts) }
  uint64_t* lkey = reinterpret_cast<uint64_t*>(sg + wbp);
  int32_t* lpos = reinterpret_cast<int32_t*>(lkey + TKSEL_LCAP);
  int32_t* grp = reinterpret_cast<int32_t*>(sg + wbp);
  __shared__ uint32_t hist[2048];
  __shared__ int mcnt[TKP_MAXSUB], gcnt[TKP_MAXSUB];
  const int TKSEL_THREADS = blockDim.x;
  __shared__ int ws[64];
  __shared__ int s_digit, s_above, s_nl, s_G, s_M, s_Z, s_over, s_need, s_eqd, s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NR = S_seg * TKP_CW;  // list regions (segment x consumer warp)
  const int wi = static_cast<int>(w);
  const int wb = static_cast<int>((w + 31) / 32);
  const double* v = D + static_cast<int64_t>(c) * w;
  uint32_t* zrow = eqz + static_cast<int64_t>(c) * wbp;
  const TkWin wn = win[c];
  {
    uint4* s4 = reinterpret_cast<uint4*>(sg);
    for (int i = tid; i < wbp / 4; i += TKSEL_THREADS) s4[i] = make_uint4(0, 0, 0, 0);
  }
  const int64_t cbase = static_cast<int64_t>(c) * NR * capw;
  const uint64_t* ck = cand_key + cbase;
  const int32_t* cp = cand_pos + cbase;
  const uint64_t* gk = gt_val + cbase;
  const int32_t* gq = gt_pos + cbase;
  // ---- region counts and totals (warp 0)
  if (warp == 0) {
    int g = 0, m = 0, z = 0, over = 0;
    for (int j = lane; j < NR; j += 32) {
      // written by the other segment CTAs of this kernel: L2, not the read-only path
      const int4 r4 = __ldcg(reinterpret_cast<const int4*>(seg) + static_cast<int64_t>(c) * NR + j);
      const TkSeg sr{r4.x, r4.y, r4.z, r4.w};
      over |= (sr.m > capw) | (sr.g > capw);
      mcnt[j] = min(sr.m, capw);
      gcnt[j] = min(sr.g, capw);
      g += sr.g;
      m += min(sr.m, capw);
      z += sr.z;
    }
    g = warp_sum_int(g);
    m = warp_sum_int(m);
    z = warp_sum_int(z);
    over = __any_sync(0xffffffffu, over);
    if (lane == 0) {
      s_G = g;
      s_M = m;
      s_Z = z;
      s_over = over;
      s_nl = 0;
      s_eqd = 0;
      s_fail = 0;
    }
  }
  __syncthreads();
  constexpr int UB = 4;  // list entries per lane in flight
  const uint64_t KMASK = 0x7FFFFFFFFFFFFFFFull;
  // merged lists (no zero tie class, see tkp_stage_m): the candidate regions
  // also hold the entries above the window.  Their rank key reads as all
  // ones here (above every prefix: outside the histograms, marked by the
  // final pass) and they are counted first (G).
  const bool merged = !wn.zero;
  auto ckey = [&](int sl) {  // candidate slot -> rank key (raw value bits stored)
    const uint64_t b = __ldcg(ck + sl);
    const uint64_t key =
        weighted ? rank_key(__longlong_as_double(static_cast<long long>(b)), __ldcg(cp + sl), 1)
                 : (b & KMASK);
    return (merged && static_cast<int>(key >> 32) > wn.hhi) ? ~0ull : key;
  };
  // merged: G is counted by the first radix level's pass (s_M = G + M until then)
  int G = s_G, M = s_M;
  const int Z = wn.zero ? s_Z : 0;
  const bool ok = !s_over && (merged ? M >= k : (G < k && G + M + Z >= k));
  bool miss = false;  // merged: the window's upper end is at or below the k-th key
  auto mark = [&](int t) { atomicOr(&sg[t >> 5], 1u << (t & 31)); };
  auto mark_eq = [&](int t) { atomicOr(&zrow[t >> 5], 1u << (t & 31)); };
  int need = k;
  if (ok) {
    // the selection row from the entries above the window
    tksel_regions<UB>(gcnt, NR, capw, [&](const int* sl, const bool* vl_) {
      int tt[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) tt[u] = vl_[u] ? __ldcg(gq + sl[u]) : -1;
#pragma unroll
      for (int u = 0; u < UB; ++u)
        if (tt[u] >= 0) mark(tt[u]);
    });
  }
  if (ok && (merged || G + M >= k)) {
    // the k-th key is a candidate; zeros (if tracked) are not needed
    if (wn.zero) {
      for (int q = tid; q < wbp; q += TKSEL_THREADS) zrow[q] = 0u;
      __syncthreads();
    }
    need = k - G;
    const int top = 32 + (31 - __clz(static_cast<unsigned>((wn.hlo + 1) ^ wn.hhi) | 1u));
    const uint64_t pf0 = static_cast<uint64_t>(static_cast<uint32_t>(wn.hhi)) >> (top - 31);
    // radix levels over the candidate regions (11 bits below `top` first)
    // until the threshold digit's bin fits the shared-memory list
    int hi_excl = top + 1, sh = hi_excl, nbin = M;
    uint64_t pf = pf0;
    bool all = false;
    for (int lv = 0; lv < 6 && hi_excl > 0; ++lv) {
      const int bits = min(11, hi_excl);
      sh = hi_excl - bits;
      const uint32_t dmask = (1u << bits) - 1u;
      for (int i = tid; i < 2048; i += TKSEL_THREADS) hist[i] = 0u;
      __syncthreads();
      int g = 0;
      tksel_regions<UB>(mcnt, NR, capw, [&](const int* sl, const bool* vl_) {
        uint64_t kk[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) kk[u] = vl_[u] ? ckey(sl[u]) : 0ull;
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          uint32_t dig = 0xFFFFFFFFu;
          if (vl_[u] && (kk[u] >> hi_excl) == pf) dig = static_cast<uint32_t>(kk[u] >> sh) & dmask;
          g += kk[u] == ~0ull;
          tks_add(hist, dig, lane);
        }
      });
      if (merged && lv == 0) {
        g = warp_sum_int(g);
        if (lane == 0 && g) atomicAdd(&s_G, g);
      }
      __syncthreads();
      if (merged && lv == 0) {
        G = s_G;
        M -= G;
        need = k - G;
        if (G >= k) { miss = true; break; }
      }
      tk_find_digit_n(hist, 1 << bits, need, ws, &s_digit, &s_above);
      need -= s_above;
      pf = (pf << bits) | static_cast<uint64_t>(s_digit);
      nbin = static_cast<int>(hist[s_digit]);
      __syncthreads();
      hi_excl = sh;
      if (nbin == need) { all = true; break; }
      if (nbin <= TKSEL_LCAP) break;
    }
    // above the threshold prefix -> selected; in it -> the shared-memory list
    // (or, when the whole bin is taken, selected as well; or, when the final
    // bin is a tie class larger than the list, tie-marked directly)
    const bool direct = !all && nbin > TKSEL_LCAP;
    if (!miss) tksel_regions<UB>(mcnt, NR, capw, [&](const int* sl, const bool* vl_) {
      uint64_t kk[UB];
      int tt[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        kk[u] = vl_[u] ? ckey(sl[u]) : 0ull;
        tt[u] = vl_[u] ? __ldcg(cp + sl[u]) : -1;
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (tt[u] < 0) continue;
        const uint64_t hp = kk[u] >> sh;
        if (hp > pf || (all && hp == pf)) {
          mark(tt[u]);
        } else if (hp == pf) {
          if (direct) {
            mark_eq(tt[u]);
            s_eqd = 1;
          } else {
            const int i = atomicAdd(&s_nl, 1);
            if (i < TKSEL_LCAP) { lkey[i] = kk[u]; lpos[i] = tt[u]; }
          }
        }
      }
    });
    __syncthreads();
    if (miss) {
      if (tid == 0) s_fail = 1;
    } else if (all) {
      need = 0;
    } else if (direct) {
      // the eq take below picks the first `need` tied positions
    } else if (s_nl <= TKSEL_LCAP) {
      const int nl = s_nl;
      auto lk = [&](int e) { return lkey[e]; };
      tksel_levels(lk, nl, hi_excl, pf, need, sh, all, 64, hist, ws, &s_digit, &s_above);
      for (int e = tid; e < nl; e += TKSEL_THREADS) {
        const uint64_t hp = lkey[e] >> sh;
        if (hp > pf || (all && hp == pf)) mark(lpos[e]);
        else if (hp == pf) { mark_eq(lpos[e]); s_eqd = 1; }
      }
      if (all) need = 0;
    } else if (tid == 0) {
      s_fail = 1;  // a tie bin of more than LCAP keys (exact ties): radix over D below
    }
  } else if (ok) {
    // every candidate is taken; the first k - G - M zeros complete the set
    tksel_regions<UB>(mcnt, NR, capw, [&](const int* sl, const bool* vl_) {
      int tt[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) tt[u] = vl_[u] ? __ldcg(cp + sl[u]) : -1;
#pragma unroll
      for (int u = 0; u < UB; ++u)
        if (tt[u] >= 0) mark(tt[u]);
    });
    need = k - G - M;
    if (tid == 0) s_eqd = 1;
  } else if (tid == 0) {
    s_fail = 1;  // the window missed or a list region overflowed
  }
  __syncthreads();
  if (s_fail) {
    // radix levels over D itself (the selection and tie rows rewritten word
    // by word; values gathered from D)
    need = k;
    if (tid == 0) s_eqd = 1;
    constexpr int NL = 6;
    constexpr int SH[NL] = {52, 41, 30, 19, 8, 0};
    constexpr int BI[NL] = {11, 11, 11, 11, 11, 8};
    uint64_t prefix = 0;
    int L = 0;
    bool take_all = false;
    for (; L < NL; ++L) {
      for (int i = tid; i < 2048; i += TKSEL_THREADS) hist[i] = 0u;
      __syncthreads();
      const int sh = SH[L], up = (L == 0) ? 63 : SH[L - 1];
      const uint32_t dmask = (1u << BI[L]) - 1u;
      for (int base = 0; base < wi; base += TKSEL_THREADS) {  // warp-uniform trip count (ballots)
        const int t = base + tid;
        uint32_t dig = 0xFFFFFFFFu;
        if (t < wi) {
          const uint64_t key = rank_key(__ldcg(v + t), t, weighted);
          if ((up >= 63 ? 0ull : (key >> up)) == prefix) dig = static_cast<uint32_t>(key >> sh) & dmask;
        }
        tks_add(hist, dig, lane);
      }
      __syncthreads();
      tk_find_digit_n(hist, 1 << BI[L], need, ws, &s_digit, &s_above);
      const int dg = s_digit;
      need -= s_above;
      prefix = (prefix << BI[L]) | static_cast<uint64_t>(dg);
      const int nbin = static_cast<int>(hist[dg]);
      __syncthreads();
      if (nbin == need) { take_all = true; break; }
    }
    if (L == NL) L = NL - 1;
    const int sh = SH[L];
    for (int base = 0; base < wb * 32; base += TKSEL_THREADS) {
      const int t = base + tid;
      bool gt = false, eq = false;
      if (t < wi) {
        const uint64_t hp = rank_key(__ldcg(v + t), t, weighted) >> sh;
        gt = take_all ? hp >= prefix : hp > prefix;
        eq = !take_all && hp == prefix;
      }
      const uint32_t gb = __ballot_sync(0xffffffffu, gt), eb = __ballot_sync(0xffffffffu, eq);
      if (lane == 0 && (t >> 5) < wb) { sg[t >> 5] = gb; zrow[t >> 5] = eb; }
    }
    if (take_all) need = 0;
  }
  if (tid == 0) s_need = need;
  __syncthreads();
  need = s_need;
  const bool gather_all = s_fail;  // values from D for every entry
  // ---- sweep: thread owns words [q0, q1) (an odd count: conflict-free)
  int wpt = (wb + TKSEL_THREADS - 1) / TKSEL_THREADS;
  wpt |= 1;
  const int q0 = min(wb, tid * wpt), q1 = min(wb, q0 + wpt);
  if (s_eqd) {  // take the first `need` tied positions; the tie row keeps
                // exactly the taken bits (values gathered below, then cleared)
    int ne = 0;
    for (int q = q0; q < q1; ++q) ne += __popc(__ldcg(zrow + q));
    int tot;
    const int before = block_excl_scan(ne, ws, &tot);
    int take = max(0, min(need - before, ne));
    for (int q = q0; q < q1; ++q) {
      uint32_t e = __ldcg(zrow + q);
      if (!e) continue;
      uint32_t add = 0u;
      for (; take > 0 && e; --take) {
        const uint32_t low = e & (0u - e);
        add |= low;
        e ^= low;
      }
      zrow[q] = add;
      sg[q] |= add;
    }
  }
  int ng = 0;
  for (int q = q0; q < q1; ++q) ng += __popc(sg[q]);
  int total;
  int pos = block_excl_scan(ng, ws, &total);  // (its syncs also retire the lkey/lpos uses)
  uint32_t* il = idx_list + static_cast<int64_t>(c) * cap;
  double* vl = val_list + static_cast<int64_t>(c) * cap;
  int32_t* rsc = em.rs ? em.rs + static_cast<int64_t>(c) * (em.nr + 1) : nullptr;
  for (int q = q0; q < q1; ++q) {
    if ((q & 7) == 0) {
      grp[q >> 3] = pos;
      if (rsc) rsc[q >> 3] = pos;  // FOLD_RANGE = 8 words
    }
    for (uint32_t m = sg[q]; m; m &= m - 1) il[pos++] = static_cast<uint32_t>(q * 32 + __ffs(m) - 1);
  }
  if (tid == 0) {
    count[c] = total;
    if (rsc) rsc[em.nr] = total;
  }
  __syncthreads();
  // ---- values (and the client shift update when this kernel owns it)
  double* hrow = em.hest ? em.hest + static_cast<int64_t>(c) * em.hest_stride : nullptr;
  auto rank = [&](int t) {
    const int q = t >> 5;
    int r = grp[q >> 3];
    for (int qq = q & ~7; qq < q; ++qq) r += __popc(sg[qq]);
    return r + __popc(sg[q] & ((1u << (t & 31)) - 1u));
  };
  auto put = [&](int t, double x) {
    const int r = rank(t);
    vl[r] = x;
    if (hrow) hrow[t] = __dadd_rn(hrow[t], __dmul_rn(em.alpha, x));  // emit_entry
  };
  if (gather_all) {
    for (int e = tid; e < total; e += TKSEL_THREADS) {
      const int t = static_cast<int>(il[e]);
      const double x = __ldg(v + t);
      vl[e] = x;
      if (hrow) hrow[t] = __dadd_rn(hrow[t], __dmul_rn(em.alpha, x));
    }
    if (s_eqd)
      for (int q = q0; q < q1; ++q) zrow[q] = 0u;
  } else {
    // entries above the window: all selected
    tksel_regions<UB>(gcnt, NR, capw, [&](const int* sl, const bool* vl_) {
      int tt[UB];
      uint64_t xb[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        tt[u] = vl_[u] ? __ldcg(gq + sl[u]) : -1;
        xb[u] = vl_[u] ? __ldcg(gk + sl[u]) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < UB; ++u)
        if (tt[u] >= 0) put(tt[u], __longlong_as_double(static_cast<long long>(xb[u])));
    });
    // candidates: the selected ones that are not taken ties
    const bool eqd = s_eqd;
    tksel_regions<UB>(mcnt, NR, capw, [&](const int* sl, const bool* vl_) {
      int tt[UB];
      uint64_t xb[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        tt[u] = vl_[u] ? __ldcg(cp + sl[u]) : -1;
        xb[u] = vl_[u] ? __ldcg(ck + sl[u]) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int t = tt[u];
        if (t < 0) continue;
        const uint32_t bit = 1u << (t & 31);
        if ((sg[t >> 5] & bit) && !(eqd && (__ldcg(zrow + (t >> 5)) & bit)))
          put(t, __longlong_as_double(static_cast<long long>(xb[u])));
      }
    });
    // taken ties (zeros or tied candidates): values from D; the tie row cleared
    if (eqd) {
      __syncthreads();
      for (int q = q0; q < q1; ++q) {
        const uint32_t e = __ldcg(zrow + q);
        if (!e) continue;
        zrow[q] = 0u;
        for (uint32_t m = e; m; m &= m - 1) {
          const int t = q * 32 + __ffs(m) - 1;
          put(t, __ldg(v + t));
        }
      }
    }
  }
  if (g_dbg_on && tid == 0 && s_fail) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&g_dbg[17]), 1ull);
    // which way the window failed: region overflow / G >= k / G + M + Z < k / digit list
    const int why = s_over ? 24 : (G >= k ? 25 : (G + M + Z < k ? 26 : 27));
    atomicAdd(reinterpret_cast<unsigned long long*>(&g_dbg[why]), 1ull);
  }
}

// --------------------------------------------------------------- RandSeqK
// grid n_active, block 256.  s = randrange(w) is the first and only draw
// (compressors.py:259-264); positions (s + j) mod w, sorted.
__global__ void __launch_bounds__(256) k_randseqk(
    const DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int wb, int k,
    const int32_t* __restrict__ clients, const int32_t* __restrict__ flags, uint64_t run_seed,
    const uint64_t* __restrict__ seeds, uint32_t* __restrict__ bitmap,
    int32_t* __restrict__ count, uint32_t* __restrict__ idx_list, double* __restrict__ val_list,
    int cap, int32_t* __restrict__ draws, Emit em) {
  if (ctl && ctl->halt) return;
  __shared__ int64_t s_start;
  const int c = client_of(clients, blockIdx.x);
  uint32_t* brow = bitmap + static_cast<int64_t>(c) * wb;
  if (!(flags[c] & 2)) {
    clear_row(brow, wb);
    emit_empty(em, c);
    if (threadIdx.x == 0) { count[c] = 0; if (draws) draws[c] = 0; }
    return;
  }
  if (threadIdx.x == 0) {
    const uint64_t seed = seeds ? seeds[blockIdx.x] : round_seed(run_seed, c, ctl->round);
    Prg p(seed);
    s_start = static_cast<int64_t>(p.randrange(static_cast<uint64_t>(w)));
    if (draws) draws[c] = p.draws;
    count[c] = k;
  }
  __syncthreads();
  const int64_t s = s_start;
  const int64_t wrap = (s + k > w) ? s + k - w : 0;
  const double scale = static_cast<double>(w) / static_cast<double>(k);
  const double* v = D + static_cast<int64_t>(c) * w;
  uint32_t* il = idx_list + static_cast<int64_t>(c) * cap;
  double* vl = val_list + static_cast<int64_t>(c) * cap;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const int64_t t = (i < wrap) ? i : s + (i - wrap);
    const double x = __dmul_rn(v[t], scale);
    il[i] = static_cast<uint32_t>(t);
    vl[i] = x;
    emit_entry(em, c, t, x);
  }
  if (em.rs) {  // selected = [0, wrap) U [s, s + k - wrap)
    for (int r = threadIdx.x; r <= em.nr; r += blockDim.x) {
      const int64_t T0 = static_cast<int64_t>(r) * FOLD_RANGE;
      const int64_t T = (T0 < w) ? T0 : w;
      const int64_t hi = s + (k - wrap);
      const int64_t lim = (T < hi) ? T : hi;
      const int64_t cnt = ((T < wrap) ? T : wrap) + ((lim > s) ? lim - s : 0);
      em.rs[static_cast<int64_t>(c) * (em.nr + 1) + r] = static_cast<int32_t>(cnt);
    }
  }
  for (int q = threadIdx.x; q < wb; q += blockDim.x) {
    uint32_t word = 0u;
    for (int bit = 0; bit < 32; ++bit) {
      const int64_t t = static_cast<int64_t>(q) * 32 + bit;
      if (t >= w) break;
      const bool in = (t >= s && t < s + k) || (t < wrap);
      word |= static_cast<uint32_t>(in) << bit;
    }
    brow[q] = word;
  }
}

// ------------------------------------------------------------------ RandK
// Partial Fisher-Yates prefix (rng.py:106-118, compressors.py:261-262).
// grid n_active, block RK_THREADS.  The k draws are generated in parallel
// from the counter-based stream; a rejection anywhere (probability
// < k w / 2^64) drops to the exact sequential loop.  The swap chain then runs
// on one thread over a sparse pool (open-addressing table in shared memory)
// and marks the selected positions in a shared-memory bitmap; the bitmap is
// compacted in ascending order by the whole block and the entries are
// emitted in parallel (values scaled by w/k, client shift update, range
// starts).
// dynamic smem: pool region | draws[k] | bitmap[wb]; the pool region holds
// either the whole pool (w <= RK_DIRECT_W) or keys[RK_TABLE] | vals[RK_TABLE]
// (k <= RK_HASH_MAXK).  Past those (any k up to w, as the reference allows)
// the draws and, for w > RK_DIRECT_W, the whole pool move to global scratch
// (gjs [n][k], gpool [n][w]): the swap chain then runs over L2.
constexpr int RK_TABLE = 16384;  // entries (key, value) -> 128 KB
constexpr int RK_HASH_MAXK = 6000;  // swap chains this short fit the table (<= 2k keys, load < 0.75)
constexpr int RK_THREADS = 256;
constexpr int64_t RK_DIRECT_W = 46000;  // pools this small live directly in shared memory
constexpr size_t RK_SMEM_MAX = 227 * 1024 - 1024;  // (+ the static shared memory)
__host__ __device__ constexpr bool rk_global_pool(int k, int64_t w) { return w > RK_DIRECT_W && k > RK_HASH_MAXK; }
__host__ __device__ constexpr size_t rk_pool_words(int k, int64_t w) {
  return rk_global_pool(k, w) ? 0
         : static_cast<size_t>(w <= RK_DIRECT_W ? (w > 2 * RK_TABLE ? w : 2 * RK_TABLE) : 2 * RK_TABLE);
}
// the draws in shared memory when they fit next to the pool and the bitmap
__host__ __device__ constexpr bool rk_js_smem(int k, int wb, int64_t w) {
  return (rk_pool_words(k, w) + static_cast<size_t>(k) + static_cast<size_t>(wb)) * 4 <= RK_SMEM_MAX;
}
// the bitmap in shared memory when it fits there too (d <= 1024: always),
// else the client's global bitmap row is worked on directly
__host__ __device__ constexpr bool rk_bm_smem(int k, int wb, int64_t w) {
  return (rk_pool_words(k, w) + (rk_js_smem(k, wb, w) ? static_cast<size_t>(k) : 0) +
          static_cast<size_t>(wb)) * 4 <= RK_SMEM_MAX;
}
__host__ __device__ constexpr size_t rk_smem_bytes(int k, int wb, int64_t w) {
  return (rk_pool_words(k, w) + (rk_js_smem(k, wb, w) ? static_cast<size_t>(k) : 0) +
          (rk_bm_smem(k, wb, w) ? static_cast<size_t>(wb) : 0)) * 4;
}
__device__ __forceinline__ int rk_slot(int32_t* keys, int32_t key) {
  uint32_t h = (static_cast<uint32_t>(key) * 2654435761u) & (RK_TABLE - 1);
  while (keys[h] != -1 && keys[h] != key) h = (h + 1) & (RK_TABLE - 1);
  return static_cast<int>(h);
}
__global__ void __launch_bounds__(RK_THREADS) k_randk(
    const DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int wb, int k,
    const int32_t* __restrict__ clients, const int32_t* __restrict__ flags, uint64_t run_seed,
    const uint64_t* __restrict__ seeds, uint32_t* __restrict__ bitmap,
    int32_t* __restrict__ count, uint32_t* __restrict__ idx_list, double* __restrict__ val_list,
    int cap, int32_t* __restrict__ draws, Emit em, int32_t* __restrict__ gjs, int32_t* __restrict__ gpool) {
  if (ctl && ctl->halt) return;
  extern __shared__ int32_t tab[];
  int32_t* keys = tab;
  int32_t* vals = tab + RK_TABLE;
  const size_t pw = rk_pool_words(k, w);
  const bool js_smem = rk_js_smem(k, wb, w);
  const int c = client_of(clients, blockIdx.x);
  int32_t* js = js_smem ? tab + pw : gjs + static_cast<int64_t>(c) * k;                // [k]
  uint32_t* bm = rk_bm_smem(k, wb, w) ? reinterpret_cast<uint32_t*>(tab + pw + (js_smem ? k : 0))  // [wb]
                                       : bitmap + static_cast<int64_t>(client_of(clients, blockIdx.x)) * wb;
  const bool global_pool = rk_global_pool(k, w);
  __shared__ int ws[64];
  __shared__ int s_reject;
  const int tid = threadIdx.x;
  uint32_t* brow = bitmap + static_cast<int64_t>(c) * wb;
  if (!(flags[c] & 2)) {
    clear_row(brow, wb);
    emit_empty(em, c);
    if (tid == 0) { count[c] = 0; if (draws) draws[c] = 0; }
    return;
  }
  const uint64_t seed = seeds ? seeds[blockIdx.x] : round_seed(run_seed, c, ctl->round);
  if (tid == 0) s_reject = 0;
  if (w > RK_DIRECT_W && !global_pool)
    for (int i = tid; i < RK_TABLE; i += RK_THREADS) keys[i] = -1;
  for (int q = tid; q < wb; q += RK_THREADS) bm[q] = 0u;
  __syncthreads();
  // parallel draw i (1-based i+1) under the no-rejection hypothesis
  for (int i = tid; i < k; i += RK_THREADS) {
    const uint64_t b = static_cast<uint64_t>(w - i);
    const uint64_t u = scramble(seed + static_cast<uint64_t>(i + 1) * GOLDEN);
    if (u < (0ull - b) % b) s_reject = 1;
    js[i] = i + static_cast<int32_t>(u % b);
  }
  __syncthreads();
  if (tid == 0 && s_reject) {  // exact sequential replay of the draws
    Prg p(seed);
    for (int i = 0; i < k; ++i) js[i] = i + static_cast<int32_t>(p.randrange(w - i));
    s_reject = p.draws;  // reused: number of draws
  } else if (tid == 0) {
    s_reject = -1;
  }
  __syncthreads();
  if (w <= RK_DIRECT_W || global_pool) {
    // the pool itself: in shared memory (over the hash table) when small,
    // else this client's global scratch row
    int32_t* pool = global_pool ? gpool + static_cast<int64_t>(c) * w : tab;
    for (int t = tid; t < w; t += RK_THREADS) pool[t] = t;
    __syncthreads();
    if (tid == 0) {
      for (int i = 0; i < k; ++i) {
        const int32_t j = js[i];
        const int32_t vi = pool[i], vj = pool[j];
        pool[j] = vi;
        pool[i] = vj;
      }
    }
    __syncthreads();
    for (int i = tid; i < k; i += RK_THREADS) {
      const int32_t v = pool[i];
      atomicOr(&bm[v >> 5], 1u << (v & 31));
    }
  } else if (tid == 0) {
    for (int i = 0; i < k; ++i) {
      const int32_t j = js[i];
      const int si = rk_slot(keys, i);
      const int32_t vi = (keys[si] == i) ? vals[si] : i;
      const int sj = rk_slot(keys, j);
      const int32_t vj = (keys[sj] == j) ? vals[sj] : j;
      keys[sj] = j; vals[sj] = vi;
      const int si2 = rk_slot(keys, i);
      keys[si2] = i; vals[si2] = vj;
      bm[vj >> 5] |= 1u << (vj & 31);
    }
  }
  if (tid == 0) {
    count[c] = k;
    if (draws) draws[c] = s_reject >= 0 ? s_reject : k;
  }
  __syncthreads();
  // ascending compaction: thread = one bitmap word, block-wide scan; the
  // positions go to idx_list (global) and the bitmap row is written out
  uint32_t* il = idx_list + static_cast<int64_t>(c) * cap;
  double* vl = val_list + static_cast<int64_t>(c) * cap;
  int32_t* rsc = em.rs ? em.rs + static_cast<int64_t>(c) * (em.nr + 1) : nullptr;
  int carry = 0;
  for (int base = 0; base < wb; base += RK_THREADS) {
    const int q = base + tid;
    const uint32_t word = (q < wb) ? bm[q] : 0u;
    int total;
    int off = block_excl_scan(__popc(word), ws, &total) + carry;
    if (q < wb) {
      brow[q] = word;
      if (rsc && (q % (FOLD_RANGE / 32)) == 0) rsc[q / (FOLD_RANGE / 32)] = off;
      for (uint32_t m = word; m; m &= m - 1) il[off++] = static_cast<uint32_t>(q * 32 + __ffs(m) - 1);
    }
    carry += total;
  }
  if (rsc && tid == 0) rsc[em.nr] = carry;
  __syncthreads();
  // values (scaled by w / k) and the client shift update, all entries in parallel
  const double scale = static_cast<double>(w) / static_cast<double>(k);
  const double* v = D + static_cast<int64_t>(c) * w;
  for (int e = tid; e < k; e += RK_THREADS) {
    const int64_t t = __ldcg(il + e);
    const double x = __dmul_rn(__ldg(v + t), scale);
    vl[e] = x;
    emit_entry(em, c, t, x);
  }
}

// ----------------------------------------------------------------- TopLEK
// grid n_active, block 1024, dynamic smem P * 12 bytes (P = pow2 >= w).
// Full bitonic sort of (energy desc, position asc) so that numpy's pairwise
// np.sum over the sorted energies can be replayed (compressors.py:179-233).
__device__ double np_pairwise_leaf(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}
// numpy's pairwise add.reduce order, replayed with an explicit stack (device
// recursion would risk the default per-thread stack): blocks of <= 128 are
// leaves; larger blocks split at n2 = n/2 - (n/2) % 8 and sum left + right.
__device__ double np_pairwise(const double* a, int n) {
  struct Frame {
    int off, len, phase;
    double left;
  };
  Frame st[24];
  int top = 0;
  st[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (top >= 0) {
    Frame& f = st[top];
    if (f.len <= 128) {
      ret = np_pairwise_leaf(a + f.off, f.len);
      --top;
      continue;
    }
    int n2 = f.len / 2;
    n2 -= n2 % 8;
    if (f.phase == 0) {
      f.phase = 1;
      st[top + 1] = {f.off, n2, 0, 0.0};
      ++top;
    } else if (f.phase == 1) {
      f.left = ret;
      f.phase = 2;
      st[top + 1] = {f.off + n2, f.len - n2, 0, 0.0};
      ++top;
    } else {
      ret = __dadd_rn(f.left, ret);
      --top;
    }
  }
  return ret;
}

// Block bitonic sort of (energy desc, position asc) with the data in
// registers: element i = tid + blockDim * r (r < R).  Strides >= blockDim
// pair elements of the same thread, strides < 32 lanes of the same warp
// (shuffles); only strides in [32, blockDim) go through shared memory.
// Sorted result written back to en / pos.
__device__ __forceinline__ bool tl_before(double ea, uint32_t pa, double eb, uint32_t pb) {
  return ea > eb || (ea == eb && pa < pb);
}
template <int R>
__device__ void tl_bitonic_sort(double* en, uint32_t* pos, int P) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  double e[R];
  uint32_t q[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    e[r] = en[tid + nt * r];
    q[r] = pos[tid + nt * r];
  }
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= nt) {  // partner in this thread: r ^ (stride / nt)
        const int rs = stride / nt;
#pragma unroll
        for (int RS = 1; RS < R; RS <<= 1) {  // compile-time partner offsets (registers)
          if (rs != RS) continue;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int r2 = r ^ RS;
            if (r2 > r) {
              const int i = tid + nt * r;
              const bool up = (i & size) == 0;
              const bool swap = tl_before(e[r2], q[r2], e[r], q[r]) == up;
              const double er = e[r], er2 = e[r2];
              const uint32_t qr = q[r], qr2 = q[r2];
              e[r] = swap ? er2 : er;
              e[r2] = swap ? er : er2;
              q[r] = swap ? qr2 : qr;
              q[r2] = swap ? qr : qr2;
            }
          }
        }
      } else if (stride < 32) {  // partner lane ^ stride
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid + nt * r;
          const double eo = __shfl_xor_sync(0xffffffffu, e[r], stride);
          const uint32_t qo = __shfl_xor_sync(0xffffffffu, q[r], stride);
          const bool up = (i & size) == 0;
          const bool lower = (lane & stride) == 0;  // i < partner
          // the lower index keeps the "before" element when ascending in our order
          const bool keep_before = (lower == up);
          const bool other_before = tl_before(eo, qo, e[r], q[r]);
          if (other_before == keep_before) { e[r] = eo; q[r] = qo; }
        }
      } else {  // partner in another warp of the block: through shared memory
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          en[tid + nt * r] = e[r];
          pos[tid + nt * r] = q[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid + nt * r;
          const int j = i ^ stride;
          const double eo = en[j];
          const uint32_t qo = pos[j];
          const bool up = (i & size) == 0;
          const bool keep_before = ((i < j) == up);
          const bool other_before = tl_before(eo, qo, e[r], q[r]);
          if (other_before == keep_before) { e[r] = eo; q[r] = qo; }
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    en[tid + nt * r] = e[r];
    pos[tid + nt * r] = q[r];
  }
  __syncthreads();
}

// The same sort with the data blocked per thread (element i = tid * R + r):
// strides < R stay in registers, strides in [R, 32R) are lane shuffles
// (partner lane ^ stride / R, same r), only strides >= 32R go through shared
// memory (15 stages instead of 25 at P = 4096, R = 4), staged in padded
// scratch (element i at i + i / 4: conflict-free for R = 4).
__device__ __forceinline__ int tl_pad(int i) { return i + (i >> 2); }
template <int R>
__device__ void tl_bitonic_sort_blocked(double* en, uint32_t* pos, int P, double* pe, uint32_t* pq) {
  const int tid = threadIdx.x, lane = tid & 31;
  double e[R];
  uint32_t q[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    e[r] = en[tid * R + r];
    q[r] = pos[tid * R + r];
  }
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < R) {  // partner r ^ stride in this thread
#pragma unroll
        for (int RS = 1; RS < R; RS <<= 1) {
          if (stride != RS) continue;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int r2 = r ^ RS;
            if (r2 > r) {
              const int i = tid * R + r;
              const bool up = (i & size) == 0;
              const bool swap = tl_before(e[r2], q[r2], e[r], q[r]) == up;
              const double er = e[r], er2 = e[r2];
              const uint32_t qr = q[r], qr2 = q[r2];
              e[r] = swap ? er2 : er;
              e[r2] = swap ? er : er2;
              q[r] = swap ? qr2 : qr;
              q[r2] = swap ? qr : qr2;
            }
          }
        }
      } else if (stride < 32 * R) {  // partner lane ^ (stride / R), same r
        const int ls = stride / R;
        const bool lower = (lane & ls) == 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid * R + r;
          const double eo = __shfl_xor_sync(0xffffffffu, e[r], ls);
          const uint32_t qo = __shfl_xor_sync(0xffffffffu, q[r], ls);
          const bool up = (i & size) == 0;
          const bool keep_before = (lower == up);
          const bool other_before = tl_before(eo, qo, e[r], q[r]);
          if (other_before == keep_before) { e[r] = eo; q[r] = qo; }
        }
      } else {  // partner thread in another warp: through padded shared memory
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          pe[tl_pad(tid * R + r)] = e[r];
          pq[tl_pad(tid * R + r)] = q[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = tid * R + r;
          const int j = i ^ stride;
          const double eo = pe[tl_pad(j)];
          const uint32_t qo = pq[tl_pad(j)];
          const bool up = (i & size) == 0;
          const bool keep_before = ((i < j) == up);
          const bool other_before = tl_before(eo, qo, e[r], q[r]);
          if (other_before == keep_before) { e[r] = eo; q[r] = qo; }
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    en[tid * R + r] = e[r];
    pos[tid * R + r] = q[r];
  }
  __syncthreads();
}

// numpy's pairwise sum, block-parallel: thread 0 lists the recursion's
// leaves (<= 128 elements, left to right), the leaves are summed in parallel
// (np_pairwise_leaf), then thread 0 folds them along the same recursion.
// Identical rounding to np_pairwise.  Whole block; result in thread 0.
constexpr int NPW_MAX_LEAVES = 512;
__device__ double np_pairwise_block(const double* a, int n, double* lsum, int* loff, int* llen,
                                    int* s_nleaf) {
  if (threadIdx.x == 0) {
    int st_off[24], st_len[24];
    int top = 0, nl = 0;
    st_off[0] = 0;
    st_len[0] = n;
    while (top >= 0) {  // preorder, left child first: leaves come out left to right
      const int off = st_off[top], len = st_len[top];
      --top;
      if (len <= 128) {
        loff[nl] = off;
        llen[nl] = len;
        ++nl;
        continue;
      }
      int n2 = len / 2;
      n2 -= n2 % 8;
      ++top; st_off[top] = off + n2; st_len[top] = len - n2;  // right (popped later)
      ++top; st_off[top] = off;      st_len[top] = n2;        // left (popped first)
    }
    *s_nleaf = nl;
  }
  __syncthreads();
  const int nl = *s_nleaf;
  for (int i = threadIdx.x; i < nl; i += blockDim.x) lsum[i] = np_pairwise_leaf(a + loff[i], llen[i]);
  __syncthreads();
  double ret = 0.0;
  if (threadIdx.x == 0) {
    struct Frame {
      int len, phase;
      double left;
    };
    Frame st[24];
    int top = 0, next = 0;
    st[0] = {n, 0, 0.0};
    while (top >= 0) {
      Frame& f = st[top];
      if (f.len <= 128) {
        ret = lsum[next++];
        --top;
        continue;
      }
      int n2 = f.len / 2;
      n2 -= n2 % 8;
      if (f.phase == 0) {
        f.phase = 1;
        st[top + 1] = {n2, 0, 0.0};
        ++top;
      } else if (f.phase == 1) {
        f.left = ret;
        f.phase = 2;
        st[top + 1] = {f.len - n2, 0, 0.0};
        ++top;
      } else {
        ret = __dadd_rn(f.left, ret);
        --top;
      }
    }
  }
  return ret;
}

// numpy's pairwise sum of a[0, n) with the recursion precomputed on the
// host (it depends on n only): tab = {nl, nn, off[nl], len[nl], left[nn],
// right[nn]}, leaves left to right, internal nodes in post-order with child
// c < nl a leaf and c >= nl node c - nl.  Each leaf is summed by 8 threads
// (one of numpy's 8 accumulators each, combined in numpy's order), the nodes
// by thread 0 in post-order.  Identical rounding to np_pairwise.  Whole
// block; the result is returned to every thread.  Scratch: val[nl + nn].
constexpr int NPW_TAB_LEAVES = 128;  // table path: w <= ~16k (larger w: np_pairwise_block)
constexpr int NPW_TAB_MAX = 4 * NPW_TAB_LEAVES + 2;
__device__ double np_pairwise_tab(const double* a, const int32_t* tab, double* val, double* red8) {
  const int nl = tab[0], nn = tab[1];
  const int32_t* off = tab + 2;
  const int32_t* len = off + nl;
  const int32_t* lft = len + nl;
  const int32_t* rgt = lft + nn;
  // 8 threads per leaf: accumulator j of leaf L
  for (int u = threadIdx.x; u < 8 * nl; u += blockDim.x) {
    const int L = u >> 3, j = u & 7;
    const int n = len[L];
    const double* x = a + off[L];
    double r = 0.0;
    if (n >= 8) {
      r = x[j];
      const int m8 = n - (n % 8);
      for (int i = 8; i < m8; i += 8) r = __dadd_rn(r, x[i + j]);
    }
    red8[u] = r;
  }
  __syncthreads();
  for (int L = threadIdx.x; L < nl; L += blockDim.x) {
    const int n = len[L];
    const double* x = a + off[L];
    double res;
    int i;
    if (n < 8) {
      res = 0.0;
      i = 0;
    } else {
      const double* r = red8 + 8 * L;
      res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      i = n - (n % 8);
    }
    for (; i < n; ++i) res = __dadd_rn(res, x[i]);
    val[L] = res;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < nn; ++q) val[nl + q] = __dadd_rn(val[lft[q]], val[rgt[q]]);
  __syncthreads();
  return val[nl + nn - 1];  // the root (the single leaf when nn == 0)
}

// en[P] f64 | pos[P] u32 | padded sort scratch (f64 + u32, P + P/4 each)
__host__ __device__ constexpr size_t toplek_smem_bytes(int P) {
  return static_cast<size_t>(P) * 12 + static_cast<size_t>(P + P / 4 + 1) * 12;
}

__global__ void __launch_bounds__(TK_THREADS) k_toplek(
    DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int wb, int k,
    const int32_t* __restrict__ clients, const int32_t* __restrict__ flags, uint64_t run_seed,
    const uint64_t* __restrict__ seeds, uint32_t* __restrict__ bitmap,
    int32_t* __restrict__ count, uint32_t* __restrict__ idx_list, double* __restrict__ val_list,
    int cap, int32_t* __restrict__ draws, int P, Emit em, const int32_t* __restrict__ npw_tab) {
  if (ctl && ctl->halt) return;
  if (threadIdx.x == 0) tl_mark(4, false);
  PhaseClock pc;
  __shared__ int32_t s_tab[NPW_TAB_MAX];
  __shared__ double s_red8[8 * NPW_TAB_LEAVES];
  extern __shared__ uint8_t tl_raw[];
  double* en = reinterpret_cast<double*>(tl_raw);                    // [P]
  uint32_t* pos = reinterpret_cast<uint32_t*>(tl_raw + 8 * static_cast<size_t>(P));  // [P]
  __shared__ int ws[64];
  __shared__ int s_t, s_nleaf;
  __shared__ double lsum[2 * NPW_MAX_LEAVES];
  __shared__ int loff[NPW_MAX_LEAVES], llen[NPW_MAX_LEAVES];
  const int c = client_of(clients, blockIdx.x);
  const double* v = D + static_cast<int64_t>(c) * w;
  uint32_t* brow = bitmap + static_cast<int64_t>(c) * wb;
  clear_row(brow, wb);
  if (!(flags[c] & 2)) {
    emit_empty(em, c);
    if (threadIdx.x == 0) { count[c] = 0; if (draws) draws[c] = 0; }
    return;
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < w) { en[i] = energy_of(v[i], i); pos[i] = i; }
    else { en[i] = 0.0; pos[i] = 0xFFFFFFFFu; }
  }
  if (npw_tab) {
    const int ntab = 2 + 2 * npw_tab[0] + 2 * npw_tab[1];
    for (int i = threadIdx.x; i < ntab; i += blockDim.x) s_tab[i] = npw_tab[i];
  }
  __syncthreads();
  pc.mark(24);
  // bitonic sort: "before" = larger energy, then smaller position
  switch (P / static_cast<int>(blockDim.x)) {  // P >= blockDim (host pads P)
    case 1: tl_bitonic_sort<1>(en, pos, P); break;
    case 2: tl_bitonic_sort<2>(en, pos, P); break;
    case 4: {
      double* pe = reinterpret_cast<double*>(tl_raw + 12 * static_cast<size_t>(P));
      tl_bitonic_sort_blocked<4>(en, pos, P, pe, reinterpret_cast<uint32_t*>(pe + tl_pad(P)));
      break;
    }
    case 8: tl_bitonic_sort<8>(en, pos, P); break;
    default: tl_bitonic_sort<16>(en, pos, P); break;
  }
  pc.mark(25);
  const double total = npw_tab ? np_pairwise_tab(en, s_tab, lsum, s_red8)
                               : np_pairwise_block(en, static_cast<int>(w), lsum, loff, llen, &s_nleaf);
  if (threadIdx.x == 0) {
    const uint64_t seed = seeds ? seeds[blockIdx.x] : round_seed(run_seed, c, ctl->round);
    Prg p(seed);
    int tsel;
    if (!(total > 0.0)) {  // compressors.py:185-186
      ctl->bad_client = c;
      raise_status(ctl, ST_TOPLEK_ZERO);
      tsel = 0;
    } else {
      const double target = static_cast<double>(k) / static_cast<double>(w);
      // shares[i] = cumsum[i] / total; first i with shares[i] >= target
      double cum = 0.0, s_prev = 0.0, s_cur = 0.0;
      int hi = -1;
      for (int i = 0; i < k; ++i) {
        cum = __dadd_rn(cum, en[i]);
        const double sh = __ddiv_rn(cum, total);
        if (sh >= target) { hi = i; s_cur = sh; break; }
        s_prev = sh;
      }
      int lo_t, hi_t;
      double p_lo;
      if (hi < 0) {  // searchsorted index >= k
        lo_t = hi_t = k; p_lo = 1.0;
      } else {
        hi_t = hi + 1;
        lo_t = hi_t - 1;
        const double share_lo = (lo_t == 0) ? 0.0 : s_prev;
        const double share_hi = s_cur;
        if (share_hi <= share_lo || share_hi <= target) {
          lo_t = hi_t; p_lo = 1.0;
        } else {
          p_lo = __ddiv_rn(__dsub_rn(share_hi, target), __dsub_rn(share_hi, share_lo));
          p_lo = fmin(fmax(p_lo, 0.0), 1.0);
        }
      }
      tsel = (p.next_f64() < p_lo) ? lo_t : hi_t;
    }
    s_t = tsel;
    count[c] = tsel;
    if (draws) draws[c] = p.draws;
  }
  __syncthreads();
  pc.mark(26);
  const int tsel = s_t;
  for (int i = threadIdx.x; i < tsel; i += blockDim.x) {
    const uint32_t t = pos[i];
    atomicOr(&brow[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  pc.mark(27);
  compact_bitmap(brow, wb, v, 1.0, idx_list + static_cast<int64_t>(c) * cap,
                 val_list + static_cast<int64_t>(c) * cap, ws, em, c);
  pc.mark(28);
  if (threadIdx.x == 0) tl_mark(4, true);
}

// ------------------------------------------------------ TopLEK, large w
// TopLEK when the w energies do not fit one CTA's shared memory (w > 8192:
// e.g. the paper's W8A run, d = 301, w = 45,451).  Same rule as k_toplek
// (compressors.py:179-233): one CTA per client sorts the energies in global
// memory — a stable LSD radix sort of the 64-bit keys ~bits(energy) (energy
// >= 0, so ascending keys = descending energy, ties keep ascending position:
// lexsort((arange, -energy))) — then forms numpy's pairwise total of the
// sorted energies (recursion table from the host, any w), the cumulative
// shares over the first k, the single draw, and emits the first t positions.
// Scratch per client (global): keys / positions twice (ping-pong), the
// pairwise leaves and nodes.
constexpr int TLB_THREADS = 1024;
constexpr int TLB_MAXW_SMEM = 8192;  // above this k_toplek_big replaces k_toplek
struct TlbScratch {
  uint64_t* key[2];    // [n][w]
  uint32_t* pos[2];    // [n][w]
  double* npw;         // [n][9 * nl + nn]: red8 then leaf / node values
  int64_t npw_stride;
};
__global__ void __launch_bounds__(TLB_THREADS, 1) k_toplek_big(
    DevCtl* __restrict__ ctl, const double* __restrict__ D, int64_t w, int wb, int k,
    const int32_t* __restrict__ clients, const int32_t* __restrict__ flags, uint64_t run_seed,
    const uint64_t* __restrict__ seeds, uint32_t* __restrict__ bitmap,
    int32_t* __restrict__ count, uint32_t* __restrict__ idx_list, double* __restrict__ val_list,
    int cap, int32_t* __restrict__ draws, Emit em, const int32_t* __restrict__ npw_tab,
    TlbScratch scr) {
  if (ctl && ctl->halt) return;
  __shared__ int hist[256];
  __shared__ int base[256];
  __shared__ int cnt[TLB_THREADS / 32][256];
  __shared__ int ws[64];
  __shared__ int s_t, s_skip;
  const int c = client_of(clients, blockIdx.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(w);
  const double* v = D + static_cast<int64_t>(c) * w;
  uint32_t* brow = bitmap + static_cast<int64_t>(c) * wb;
  clear_row(brow, wb);
  if (!(flags[c] & 2)) {
    emit_empty(em, c);
    if (tid == 0) { count[c] = 0; if (draws) draws[c] = 0; }
    return;
  }
  uint64_t* key[2] = {scr.key[0] + static_cast<int64_t>(c) * w, scr.key[1] + static_cast<int64_t>(c) * w};
  uint32_t* pos[2] = {scr.pos[0] + static_cast<int64_t>(c) * w, scr.pos[1] + static_cast<int64_t>(c) * w};
  for (int i = tid; i < n; i += TLB_THREADS) {
    key[0][i] = ~static_cast<uint64_t>(__double_as_longlong(energy_of(v[i], i)));
    pos[0][i] = static_cast<uint32_t>(i);
  }
  int cur = 0;
  const uint32_t lt_mask = (1u << lane) - 1u;
  for (int pass = 0; pass < 8; ++pass) {
    const int sh = 8 * pass;
    for (int b = tid; b < 256; b += TLB_THREADS) hist[b] = 0;
    if (tid == 0) s_skip = 0;
    __syncthreads();
    for (int i = tid; i < n; i += TLB_THREADS) atomicAdd(&hist[(key[cur][i] >> sh) & 255u], 1);
    __syncthreads();
    if (tid < 256) {  // exclusive scan of the digit counts; a pass with one digit is the identity
      int acc = 0;
      for (int b = 0; b < tid; ++b) acc += hist[b];
      base[tid] = acc;
      if (hist[tid] == n) s_skip = 1;
    }
    __syncthreads();
    if (s_skip) continue;
    const uint64_t* ki = key[cur];
    const uint32_t* pi = pos[cur];
    uint64_t* ko = key[cur ^ 1];
    uint32_t* po = pos[cur ^ 1];
    for (int t0 = 0; t0 < n; t0 += TLB_THREADS) {
      for (int e = tid; e < (TLB_THREADS / 32) * 256; e += TLB_THREADS) (&cnt[0][0])[e] = 0;
      __syncthreads();
      const int i = t0 + tid;
      const bool ok = i < n;
      const uint64_t kv = ok ? ki[i] : 0ull;
      const uint32_t pv = ok ? pi[i] : 0u;
      const int dg = ok ? static_cast<int>((kv >> sh) & 255u) : 256;
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      const int rnk = __popc(peers & lt_mask);
      if (ok && rnk == 0) cnt[warp][dg] = __popc(peers);
      __syncthreads();
      if (tid < 256) {  // stable: warps in order inside the tile, tiles in order
        int run = base[tid];
        for (int q = 0; q < TLB_THREADS / 32; ++q) {
          const int t = cnt[q][tid];
          cnt[q][tid] = run;
          run += t;
        }
        base[tid] = run;
      }
      __syncthreads();
      if (ok) {
        const int dst = cnt[warp][dg] + rnk;
        ko[dst] = kv;
        po[dst] = pv;
      }
      __syncthreads();
    }
    cur ^= 1;
  }
  // sorted energies (descending) back as doubles, in place of the keys
  double* en = reinterpret_cast<double*>(key[cur]);
  for (int i = tid; i < n; i += TLB_THREADS) en[i] = __longlong_as_double(static_cast<long long>(~key[cur][i]));
  __syncthreads();
  const int nl = npw_tab[0];
  double* red8 = scr.npw + static_cast<int64_t>(c) * scr.npw_stride;
  const double total = np_pairwise_tab(en, npw_tab, red8 + 8 * nl, red8);
  if (tid == 0) {
    const uint64_t seed = seeds ? seeds[blockIdx.x] : round_seed(run_seed, c, ctl->round);
    Prg p(seed);
    int tsel;
    if (!(total > 0.0)) {  // compressors.py:185-186
      ctl->bad_client = c;
      raise_status(ctl, ST_TOPLEK_ZERO);
      tsel = 0;
    } else {
      const double target = static_cast<double>(k) / static_cast<double>(w);
      double cum = 0.0, s_prev = 0.0, s_cur = 0.0;
      int hi = -1;
      for (int i = 0; i < k; ++i) {
        cum = __dadd_rn(cum, en[i]);
        const double shv = __ddiv_rn(cum, total);
        if (shv >= target) { hi = i; s_cur = shv; break; }
        s_prev = shv;
      }
      int lo_t, hi_t;
      double p_lo;
      if (hi < 0) {
        lo_t = hi_t = k; p_lo = 1.0;
      } else {
        hi_t = hi + 1;
        lo_t = hi_t - 1;
        const double share_lo = (lo_t == 0) ? 0.0 : s_prev;
        const double share_hi = s_cur;
        if (share_hi <= share_lo || share_hi <= target) {
          lo_t = hi_t; p_lo = 1.0;
        } else {
          p_lo = __ddiv_rn(__dsub_rn(share_hi, target), __dsub_rn(share_hi, share_lo));
          p_lo = fmin(fmax(p_lo, 0.0), 1.0);
        }
      }
      tsel = (p.next_f64() < p_lo) ? lo_t : hi_t;
    }
    s_t = tsel;
    count[c] = tsel;
    if (draws) draws[c] = p.draws;
  }
  __syncthreads();
  const int tsel = s_t;
  const uint32_t* ps = pos[cur];
  for (int i = tid; i < tsel; i += TLB_THREADS) {
    const uint32_t t = ps[i];
    atomicOr(&brow[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  compact_bitmap(brow, wb, v, 1.0, idx_list + static_cast<int64_t>(c) * cap,
                 val_list + static_cast<int64_t>(c) * cap, ws, em, c);
}

// --------------------------------------------------------- identity / natural
// Dense kinds: count = w (or 0).  Natural rounds every coordinate to one of
// its bracketing powers of two with draw t+1 of the stream
// (compressors.py:289-336); the rounded values overwrite `out` (may alias D).
__global__ void __launch_bounds__(256) k_dense_kind(
    const DevCtl* __restrict__ ctl, const double* D, double* out,  // may alias
    int64_t w, int natural, const int32_t* __restrict__ clients,
    const int32_t* __restrict__ flags, uint64_t run_seed, const uint64_t* __restrict__ seeds,
    int32_t* __restrict__ count, int32_t* __restrict__ draws) {
  if (ctl && ctl->halt) return;
  const int c = client_of(clients, blockIdx.y);
  const bool nonzero = flags[c] & 2;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    count[c] = nonzero ? static_cast<int32_t>(w) : 0;
    if (draws) draws[c] = (nonzero && natural) ? static_cast<int32_t>(w) : 0;
  }
  if (!nonzero) return;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= w) return;
  const double x = D[static_cast<int64_t>(c) * w + t];
  if (!natural) {
    if (out != D) out[static_cast<int64_t>(c) * w + t] = x;
    return;
  }
  const uint64_t seed = seeds ? seeds[blockIdx.y] : round_seed(run_seed, c, ctl->round);
  const double u =
      static_cast<double>(scramble(seed + static_cast<uint64_t>(t + 1) * GOLDEN) >> 11) * 0x1.0p-53;
  const double tiny = 0x1.0p-1022, huge = 0x1.0p+1023;
  const double mag = fabs(x);
  double low = 0.0, high = 0.0, p_up = 0.0;
  if (mag >= tiny && mag < huge) {
    int e;
    frexp(mag, &e);
    low = ldexp(0.5, e);
    high = ldexp(1.0, e);
    p_up = __ddiv_rn(__dsub_rn(mag, low), low);
  } else if (mag > 0.0 && mag < tiny) {
    high = tiny;
    p_up = __ddiv_rn(mag, tiny);
  } else if (mag >= huge) {
    low = huge;
    high = huge;
  }
  const double r = (u < p_up) ? high : low;
  out[static_cast<int64_t>(c) * w + t] = (x < 0.0) ? -r : r;
}

}  // namespace fb
