// oracle_kernels.cuh — batched logistic oracle (reference oracle.py:64-121).
//
// HBM layout of the design matrices (built by fb_upload_shards):
//   Bt[c][a][j], c < n clients, a < d features, j < ldj samples (ldj even,
//   zero padded) — feature-major, sample-contiguous rows.  This is the
//   transpose of each shard's F-order d x n_i matrix viewed per client, so a
//   TMA box {16 samples, 64 features} lands as 64 rows of 128 B
//   (SWIZZLE_128B) for the DMMA Hessian, and the margins pass below reads
//   sample-contiguous rows coalesced.
//
// Per-sample coefficients (length ldh = round_up(n_i, 16), zero padded):
//   hcoef = sigma (1 - sigma) / n_i      (oracle.py:133)
//   gcoef = (sigma - 1) / n_i            (oracle.py:116)
#pragma once
#include "common.cuh"

namespace fb {

constexpr int MARGIN_THREADS = 128;

// The margins-type passes (margins, gradient, line-search trials) read B
// from a compact copy when every value of the uploaded shards converts to a
// narrower type and back (fb_upload_shards: binary / count features with the
// labels absorbed, {-1, 0, 1}, as int8; float-exact values as float): each
// value is widened to the same double before the same fma, so the results
// are identical and the pass moves 8x (2x) fewer bytes.  (int8 drops the
// sign of a -0.0 entry, which no sum can see: every accumulation starts at
// +0.0, and +0.0 + -0.0 = +0.0.)  The Hessian's TMA tiles stay fp64.
template <class T> struct BPair;  // two consecutive samples of one row
template <> struct BPair<double> {
  using V = double2;
  __device__ static V ld(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }
  __device__ static double x(V v) { return v.x; }
  __device__ static double y(V v) { return v.y; }
};
template <> struct BPair<float> {
  using V = float2;
  __device__ static V ld(const float* p) { return __ldcs(reinterpret_cast<const float2*>(p)); }
  __device__ static double x(V v) { return static_cast<double>(v.x); }
  __device__ static double y(V v) { return static_cast<double>(v.y); }
};
template <> struct BPair<int8_t> {
  using V = short;
  __device__ static V ld(const int8_t* p) { return __ldcs(reinterpret_cast<const short*>(p)); }
  __device__ static double x(V v) { return static_cast<double>(static_cast<int8_t>(v & 0xFF)); }
  __device__ static double y(V v) { return static_cast<double>(static_cast<int8_t>(v >> 8)); }
};
template <class T> __device__ __forceinline__ double bload(const T* p) { return static_cast<double>(__ldg(p)); }
// rows per batch of the streaming loops: the same bytes in flight per thread
template <class T> __host__ __device__ constexpr int b_rows_per_batch() { return sizeof(T) >= 8 ? 8 : sizeof(T) >= 4 ? 16 : 32; }

// stable logistic, oracle.py:64-71
__device__ __forceinline__ double stable_sigmoid(double m) {
  if (m >= 0.0) return 1.0 / (1.0 + exp(-m));
  const double e = exp(m);
  return e / (1.0 + e);
}
// log(1 + exp(-m)) without overflow, oracle.py:99-103
__device__ __forceinline__ double softplus_neg(double m) {
  if (m >= 0.0) return log1p(exp(-m));
  return -m + log1p(exp(m));
}

// Margins m_j = <B_j, x>, sigmoids, per-sample Hessian / gradient
// coefficients, and per-block partial sums of the loss (for f_value).
// One block = MB_SAMPLES consecutive samples (lane = 2 samples, one 16-byte
// load) x 8 warps that split the features (warp w sums a = w, w + 8, ...):
// every load instruction reads a contiguous 512 B row segment and each
// thread keeps 8 of them in flight.
// grid (ceil(ldh / 64), n_active), block 256, dynamic smem d doubles.
constexpr int MB_SAMPLES = 64;
constexpr int MB_THREADS = 256;
template <class T>
__global__ void __launch_bounds__(MB_THREADS) k_margins(
    const DevCtl* __restrict__ ctl, const T* __restrict__ Bt, int d,
    const int32_t* __restrict__ ni_arr, int ldj,
    int ldh, const double* __restrict__ x, const int32_t* __restrict__ clients,
    double* __restrict__ hcoef, double* __restrict__ gcoef, double* __restrict__ loss_part,
    int nblk, int32_t* __restrict__ zero_flags = nullptr) {
  // the Hessian pass may launch now (it waits for these coefficients)
  asm volatile("griddepcontrol.launch_dependents;");
  if (ctl && ctl->halt) return;
  if (threadIdx.x == 0) tl_mark(0, false);
  // the round's per-client flags start clear (the Hessian's epilogue ORs
  // into them only after this grid completes)
  if (zero_flags && blockIdx.x == 0 && threadIdx.x == 0) zero_flags[client_of(clients, blockIdx.y)] = 0;
  extern __shared__ double xs[];
  __shared__ double part[8][MB_SAMPLES + 2];
  __shared__ double red[2];
  const int c = client_of(clients, blockIdx.y);
  const int ni = ni_arr[c];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int a = threadIdx.x; a < d; a += blockDim.x) xs[a] = x[a];
  __syncthreads();
  const int j = blockIdx.x * MB_SAMPLES + 2 * lane;  // this lane's samples j, j + 1
  double m0 = 0.0, m1 = 0.0;
  if (j < ldj) {  // ldj even: j + 1 < ldj too (zero padded beyond ni)
    using P = BPair<T>;
    const T* col = Bt + static_cast<int64_t>(c) * d * ldj + j;
    double2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = make_double2(0.0, 0.0);
    int a0 = warp;
    for (; a0 + 56 < d; a0 += 64) {
      typename P::V bv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) bv[u] = P::ld(col + static_cast<int64_t>(a0 + 8 * u) * ldj);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double xa = xs[a0 + 8 * u];
        acc[u & 3].x = fma(P::x(bv[u]), xa, acc[u & 3].x);
        acc[u & 3].y = fma(P::y(bv[u]), xa, acc[u & 3].y);
      }
    }
    for (; a0 < d; a0 += 8) {
      const typename P::V bv = P::ld(col + static_cast<int64_t>(a0) * ldj);
      acc[0].x = fma(P::x(bv), xs[a0], acc[0].x);
      acc[0].y = fma(P::y(bv), xs[a0], acc[0].y);
    }
    m0 = (acc[0].x + acc[1].x) + (acc[2].x + acc[3].x);
    m1 = (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y);
  }
  part[warp][2 * lane] = m0;
  part[warp][2 * lane + 1] = m1;
  __syncthreads();
  if (warp < 2) {  // thread = one sample of the block
    const int sl = warp * 32 + lane;
    const int js = blockIdx.x * MB_SAMPLES + sl;
    double mm = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) mm += part[w2][sl];
    double loss = 0.0;
    if (js < ni) {
      const double sig = stable_sigmoid(mm);
      const double nd = static_cast<double>(ni);
      hcoef[static_cast<int64_t>(c) * ldh + js] = __ddiv_rn(__dmul_rn(sig, __dsub_rn(1.0, sig)), nd);
      gcoef[static_cast<int64_t>(c) * ldh + js] = __ddiv_rn(__dsub_rn(sig, 1.0), nd);
      loss = softplus_neg(mm);
    } else if (js < ldh) {
      hcoef[static_cast<int64_t>(c) * ldh + js] = 0.0;
      gcoef[static_cast<int64_t>(c) * ldh + js] = 0.0;
    }
    const double tot = warp_sum(loss);
    if (lane == 0) red[warp] = tot;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    loss_part[static_cast<int64_t>(c) * nblk + blockIdx.x] = red[0] + red[1];
    tl_mark(0, true);
  }
}

// The same outputs with one CTA per client (used when the clients alone
// fill the GPU): the client's B_c (d x ldj doubles, contiguous) is streamed
// once front to back.  Thread t owns the sample pair sp = t % SP (SP =
// ldj / 2) in row group g = t / SP (G groups: rows a = g, g + G, ...), so
// every row is read as one contiguous segment and each thread keeps 8 rows in
// flight; the G partial margins are summed in a fixed order.  The loss
// partials per 64-sample block are formed exactly as k_margins forms them.
// grid n_active, block MC_THREADS, dynamic smem (d + G * 2 * SPc) doubles
// where SPc = min(SP, MC_THREADS) (sample pairs per chunk).
constexpr int MC_THREADS = 1024;
// sample pairs per CTA when a client's samples are split over `nsplit` CTAs
// (each a multiple of 32 pairs = 64 samples, so the loss blocks stay whole)
__host__ __device__ constexpr int mc_split_pairs(int ldj, int nsplit) {
  return nsplit <= 1 ? ldj / 2 : ((ldj / 2 + nsplit - 1) / nsplit + 31) / 32 * 32;
}
__host__ __device__ constexpr int mc_pairs_nt(int ldj, int nsplit, int nt) {
  return mc_split_pairs(ldj, nsplit) < nt ? mc_split_pairs(ldj, nsplit) : nt;
}
__host__ __device__ constexpr int mc_groups_nt(int ldj, int nsplit, int nt) {
  return nt / mc_pairs_nt(ldj, nsplit, nt) > 32 ? 32 : nt / mc_pairs_nt(ldj, nsplit, nt);
}
__host__ __device__ constexpr int mc_pairs(int ldj) { return mc_pairs_nt(ldj, 1, MC_THREADS); }
__host__ __device__ constexpr int mc_groups(int ldj) { return mc_groups_nt(ldj, 1, MC_THREADS); }
__host__ __device__ constexpr size_t mc_smem_bytes_nt(int d, int ldj, int nsplit, int nt) {
  return (static_cast<size_t>(d) + static_cast<size_t>(mc_groups_nt(ldj, nsplit, nt)) * 2 *
                                       mc_pairs_nt(ldj, nsplit, nt)) * sizeof(double);
}
__host__ __device__ constexpr size_t mc_smem_bytes(int d, int ldj) {
  return mc_smem_bytes_nt(d, ldj, 1, MC_THREADS);
}
constexpr size_t MC_SMEM_MAX = 96 * 1024;
// NT threads per CTA, NS CTAs per client (client slot = blockIdx.x / NS,
// sample pairs [part * SPS, (part + 1) * SPS) of SPS = mc_split_pairs).
template <int NT, int NS, class T>
__global__ void __launch_bounds__(NT, NS > 1 ? 2 : 1) k_margins_cpc(
    const DevCtl* __restrict__ ctl, const T* __restrict__ Bt, int d,
    const int32_t* __restrict__ ni_arr, int ldj,
    int ldh, const double* __restrict__ x, const int32_t* __restrict__ clients,
    double* __restrict__ hcoef, double* __restrict__ gcoef, double* __restrict__ loss_part,
    int nblk, int32_t* __restrict__ zero_flags = nullptr) {
  // the Hessian pass may launch now (it waits for these coefficients)
  asm volatile("griddepcontrol.launch_dependents;");
  if (ctl && ctl->halt) return;
  extern __shared__ double mcs[];
  __shared__ double red[NT / 32];
  if (threadIdx.x == 0) tl_mark(0, false);
  const int c = client_of(clients, blockIdx.x / NS);
  if (zero_flags && blockIdx.x % NS == 0 && threadIdx.x == 0) zero_flags[c] = 0;  // (as k_margins)
  const int ni = ni_arr[c];
  const int part = blockIdx.x % NS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int SPS = mc_split_pairs(ldj, NS);
  const int SPc = mc_pairs_nt(ldj, NS, NT), G = mc_groups_nt(ldj, NS, NT);
  double* xs = mcs;
  double* part_m = mcs + d;  // [G][2 * SPc]
  for (int a = tid; a < d; a += NT) xs[a] = x[a];
  __syncthreads();
  const int SP = ldj / 2;
  const int sp_lo = part * SPS, sp_hi = min(SP, sp_lo + SPS);
  const int g = tid / SPc, sp_l = tid % SPc;
  using P = BPair<T>;
  constexpr int RB = b_rows_per_batch<T>();
  const T* base = Bt + static_cast<int64_t>(c) * d * ldj;
  for (int sp0 = sp_lo; sp0 < sp_hi; sp0 += SPc) {
    // ---- partial margins of this chunk's sample pairs over row group g
    const int sp = sp0 + sp_l;
    if (g < G && sp < sp_hi) {
      const T* col = base + 2 * sp;
      double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
      // RB rows per batch (the same bytes in flight for every element type),
      // the last batch predicated (no one-row tail loop: every batch is one
      // memory round trip); within a batch the rows are added in the fp64
      // path's order (two accumulators alternating over the rows)
      for (int a = g; a < d; a += RB * G) {
        typename P::V bv[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u)  // rows past d re-read row d-1 (weight 0): no branch
          bv[u] = P::ld(col + static_cast<int64_t>(min(a + u * G, d - 1)) * ldj);
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          const double xa = a + u * G < d ? xs[a + u * G] : 0.0;
          acc[u & 1].x = fma(P::x(bv[u]), xa, acc[u & 1].x);
          acc[u & 1].y = fma(P::y(bv[u]), xa, acc[u & 1].y);
        }
      }
      part_m[g * 2 * SPc + 2 * sp_l] = acc[0].x + acc[1].x;
      part_m[g * 2 * SPc + 2 * sp_l + 1] = acc[0].y + acc[1].y;
    }
    __syncthreads();
    // ---- coefficients and loss partials of the chunk's samples
    const int js0 = 2 * sp0;  // a multiple of 64 (chunks and parts are)
    const int nchunk = 2 * min(SPc, sp_hi - sp0);
    for (int t0 = 0; t0 < nchunk; t0 += NT) {
      const int sl = t0 + tid, js = js0 + sl;
      double loss = 0.0;
      if (sl < nchunk && js < ldh) {
        double mm = 0.0;
        for (int g2 = 0; g2 < G; ++g2) mm += part_m[g2 * 2 * SPc + sl];
        if (js < ni) {
          const double sig = stable_sigmoid(mm);
          const double nd = static_cast<double>(ni);
          hcoef[static_cast<int64_t>(c) * ldh + js] = __ddiv_rn(__dmul_rn(sig, __dsub_rn(1.0, sig)), nd);
          gcoef[static_cast<int64_t>(c) * ldh + js] = __ddiv_rn(__dsub_rn(sig, 1.0), nd);
          loss = softplus_neg(mm);
        } else {
          hcoef[static_cast<int64_t>(c) * ldh + js] = 0.0;
          gcoef[static_cast<int64_t>(c) * ldh + js] = 0.0;
        }
      }
      const double tot = warp_sum(loss);
      if (lane == 0) red[warp] = tot;
      __syncthreads();
      // block b = 64 consecutive samples: the sum of its two 32-sample warps
      const int b = (js0 + t0) / 64 + tid;
      if (tid < NT / 64 && b < nblk && 64 * tid < nchunk - t0)
        loss_part[static_cast<int64_t>(c) * nblk + b] = red[2 * tid] + red[2 * tid + 1];
      __syncthreads();
    }
  }
  // padding samples past the last pair (ldj <= js < ldh) carry no weight
  if (part == NS - 1)
    for (int js = 2 * SP + tid; js < ldh; js += NT) {
      hcoef[static_cast<int64_t>(c) * ldh + js] = 0.0;
      gcoef[static_cast<int64_t>(c) * ldh + js] = 0.0;
    }
  if (tid == 0) tl_mark(0, true);
}

// Local gradients g_c = B_c gcoef_c + lam x (oracle.py:108-121).
// grid (ceil(d / 8), n_active), block 256: one warp per feature row.
template <class T>
__global__ void __launch_bounds__(256) k_gradient(
    const DevCtl* __restrict__ ctl, const T* __restrict__ Bt, int d,
    const int32_t* __restrict__ ni_arr, int ldj, int ldh, const double* __restrict__ x,
    const double* __restrict__ lam_arr, const int32_t* __restrict__ clients,
    const double* __restrict__ gcoef, double* __restrict__ grad) {
  if (ctl && ctl->halt) return;
  const int c = client_of(clients, blockIdx.y);
  const int ni = ni_arr[c];
  const double lam = lam_arr[c];
  const int a = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (a >= d) return;
  const T* row = Bt + (static_cast<int64_t>(c) * d + a) * ldj;
  const double* gc = gcoef + static_cast<int64_t>(c) * ldh;
  double s0 = 0.0, s1 = 0.0;
  int j = lane;
  for (; j + 32 < ni; j += 64) {
    s0 = fma(bload(row + j), __ldg(gc + j), s0);
    s1 = fma(bload(row + j + 32), __ldg(gc + j + 32), s1);
  }
  if (j < ni) s0 = fma(bload(row + j), __ldg(gc + j), s0);
  const double s = warp_sum(s0 + s1);
  if (lane == 0) grad[static_cast<int64_t>(c) * d + a] = __dadd_rn(s, __dmul_rn(lam, x[a]));
}

// Line-search trials (algorithms.py:304-309, runtime.py:203-208):
// trial_s = x - step_s * p for s in [s0, s0 + S), s0 = ctl->ls_next; per
// client and trial the loss partial sums, client-major
// loss_part[c][s][block] (one contiguous block per client, so a sharded run
// all-gathers it in place).  grid (ceil(ldj / 128), n_active), block 128,
// dynamic smem S * d doubles.
constexpr int LS_BATCH = 4;
template <class T>
__global__ void __launch_bounds__(MARGIN_THREADS) k_ls_trials(
    const DevCtl* __restrict__ ctl, const T* __restrict__ Bt, int d,
    const int32_t* __restrict__ ni_arr, int ldj, const int32_t* __restrict__ clients,
    const double* __restrict__ x, const double* __restrict__ p,
    const double* __restrict__ steps_table, double* __restrict__ trial_x,
    double* __restrict__ loss_part, int nblk) {
  if (ctl->halt) return;
  if (threadIdx.x == 0) tl_mark(13, false);
  extern __shared__ double xt[];  // [LS_BATCH][d]
  const int s0 = ctl->ls_next;
  const int c = client_of(clients, blockIdx.y);
  const int ni = ni_arr[c];
  for (int e = threadIdx.x; e < LS_BATCH * d; e += blockDim.x) {
    const int s = e / d, a = e - s * d;
    const int si = s0 + s;
    const double step = steps_table[si <= 60 ? si : 60];
    xt[e] = __dsub_rn(x[a], __dmul_rn(step, p[a]));
  }
  __syncthreads();
  if (blockIdx.x == 0 && blockIdx.y == 0) {
    for (int e = threadIdx.x; e < LS_BATCH * d; e += blockDim.x) trial_x[e] = xt[e];
  }
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double m[LS_BATCH];
#pragma unroll
  for (int s = 0; s < LS_BATCH; ++s) m[s] = 0.0;
  if (j < ni) {
    // 16 independent loads in flight per batch; the last batch predicated
    // (features in increasing order as before: the same fma chain)
    const T* col = Bt + static_cast<int64_t>(c) * d * ldj + j;
    for (int a = 0; a < d; a += 16) {
      double b[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) b[u] = a + u < d ? bload(col + static_cast<int64_t>(a + u) * ldj) : 0.0;
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (a + u < d)
#pragma unroll
          for (int s = 0; s < LS_BATCH; ++s) m[s] = fma(b[u], xt[s * d + a + u], m[s]);
    }
  }
  // the LS_BATCH block sums with one barrier pair (block_sum's order per trial)
  __shared__ double red4[LS_BATCH][MARGIN_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int s = 0; s < LS_BATCH; ++s) {
    const double v = warp_sum((j < ni) ? softplus_neg(m[s]) : 0.0);
    if (lane == 0) red4[s][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < LS_BATCH) {
    const int s = threadIdx.x;
    double tot = 0.0;
    for (int i = 0; i < nw; ++i) tot += red4[s][i];
    loss_part[(static_cast<int64_t>(c) * LS_BATCH + s) * nblk + blockIdx.x] = tot;
  }
  if (threadIdx.x == 0) tl_mark(13, true);
}

}  // namespace fb
