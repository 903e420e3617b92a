// round_kernels.cuh — cross-client reductions, the fused shift + master fold,
// FedNL-PP bookkeeping and the round epilogue (reference algorithms.py,
// runtime.py).  Every reduction over clients runs in ascending client id
// with sequential adds, so results do not depend on launch shape.
#pragma once
#include "common.cuh"
#include "compress_kernels.cuh"

namespace fb {

// Cross-client reductions of one round (algorithms.py:351-359, 399-402;
// runtime.py:189-201):
//   f_cli[c]    = sum_b loss_part[c][b] / n_c + (0.5 lam_c) <x, x>
//   shift_cli[c]= sqrt(sum_p frob_part[c][p])           (if frob_part)
//   gbar        = (sum_c grad_c) / n_div
//   out: ||gbar||, (sum_c f_c) / n_div, (sum_c shift_c) / n_div
// A non-finite difference raises ST_NONFINITE (compressors.py:134-135).
// Client sums use a fixed association (not the reference's sequential
// order): the parity tolerance of these scalars is 1e-12 relative.
struct RoundScalars {
  double grad_norm;
  double f_mean;
  double shift_mean;
  double decrement;  // LS: <gbar, p>
  double xx;
};

// grid = reduce_grid(d) CTAs of 1024 threads.  CTA b owns the 32-feature
// gbar tile b (its 32 warps split the clients, then a fixed-order tree over
// the warps) and the client chunk b of the per-client scalars; every load of
// a CTA is issued in one burst (the kernel is latency-, not bandwidth-bound).
// The last CTA to finish (ticket in DevCtl) forms the round scalars.
constexpr int RED_THREADS = 1024;
__host__ __device__ __forceinline__ int reduce_grid(int d) { return (d + 31) / 32; }
__global__ void __launch_bounds__(RED_THREADS) k_reduce(
    DevCtl* __restrict__ ctl, int n_active, const int32_t* __restrict__ clients, int n_div, int d,
    const int32_t* __restrict__ ni_arr, int nblk, int n_pairs, const double* __restrict__ x,
    const double* __restrict__ lam_arr,
    const double* __restrict__ grad, const double* __restrict__ loss_part,
    const double* __restrict__ frob_part, const int32_t* __restrict__ flags,
    double* __restrict__ gbar, double* __restrict__ f_cli, double* __restrict__ shift_cli,
    RoundScalars* __restrict__ out, double* __restrict__ row_grad, double* __restrict__ row_f,
    const double* __restrict__ l2_prefetch, int64_t l2_prefetch_bytes) {
  // the next kernel (the master solve) may start its H^k setup now
  asm volatile("griddepcontrol.launch_dependents;");
  if (ctl->halt) return;
  if (threadIdx.x == 0) tl_mark(12, false);
  PhaseClock pc;
  // warm L2 with the next kernel's input (the master H^k for the solve)
  if (l2_prefetch)
    for (int64_t off = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 128;
         off < l2_prefetch_bytes; off += static_cast<int64_t>(gridDim.x) * blockDim.x * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(l2_prefetch) + off));
  // programmatic dependent launch: the Hessian pass's outputs from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ double red[32];
  __shared__ double gp[32][33];
  __shared__ double stage[2048];
  __shared__ int s_bad, s_last;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int G = gridDim.x, b = blockIdx.x;
  if (threadIdx.x == 0) s_bad = 0x7fffffff;
  // ---- burst: x, this CTA's client partials, this CTA's grad tile
  const double xv = threadIdx.x < d ? x[threadIdx.x] : 0.0;
  double xx_part = xv * xv;
  for (int a = threadIdx.x + RED_THREADS; a < d; a += RED_THREADS) xx_part = fma(x[a], x[a], xx_part);
  const int per_c = nblk + (frob_part ? n_pairs : 0);
  const int cpb = (n_active + G - 1) / G;
  const int c_lo = min(n_active, b * cpb), c_hi = min(n_active, c_lo + cpb);
  // a client's partials are staged when they fit the buffer (else read in
  // place: d > ~2800)
  const bool staged = per_c <= 2048;
  const int chunk = staged ? 2048 / per_c : 1 << 30;
  auto stage_load = [&](int i0, int nc) {
    if (!staged) return;
    for (int e = threadIdx.x; e < nc * per_c; e += RED_THREADS) {
      const int ii = e / per_c, r = e - ii * per_c;
      const int c = client_of(clients, i0 + ii);
      stage[e] = r < nblk ? __ldcg(loss_part + static_cast<int64_t>(c) * nblk + r)
                          : __ldcg(frob_part + static_cast<int64_t>(c) * n_pairs + (r - nblk));
    }
  };
  stage_load(c_lo, min(chunk, c_hi - c_lo));
  {
    const int a = b * 32 + lane;
    const int per = (n_active + 31) / 32;
    const int i_lo = min(n_active, q * per), i_hi = min(n_active, i_lo + per);
    double sacc = 0.0;
    if (a < d) {
      for (int i0 = i_lo; i0 < i_hi; i0 += 8) {
        // client ids first: a load feeding an address shares the grad loads'
        // scoreboard, so interleaving them would serialise the batch
        int cc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cc[u] = (i0 + u < i_hi) ? client_of(clients, i0 + u) : -1;
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = (cc[u] >= 0) ? __ldcg(grad + static_cast<int64_t>(cc[u]) * d + a) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (cc[u] >= 0) sacc = __dadd_rn(sacc, v[u]);
      }
    }
    gp[q][lane] = sacc;
  }
  const double xx = block_sum(xx_part, red);  // also publishes stage / gp
  pc.mark(8);
  if (q == 0) {
    const int a = b * 32 + lane;
    double t2 = 0.0;
#pragma unroll 8
    for (int w2 = 0; w2 < 32; ++w2) t2 = __dadd_rn(t2, gp[w2][lane]);
    if (a < d) gbar[a] = __ddiv_rn(t2, static_cast<double>(n_div));
  }
  // ---- per-client scalars of this CTA's chunk
  for (int i0 = c_lo; i0 < c_hi; i0 += chunk) {
    const int nc = min(chunk, c_hi - i0);
    if (i0 != c_lo) {
      __syncthreads();
      stage_load(i0, nc);
      __syncthreads();
    }
    for (int ii = threadIdx.x; ii < nc; ii += RED_THREADS) {
      const int c = client_of(clients, i0 + ii);
      const double* st = stage + ii * per_c;
      auto part = [&](int r) {
        return staged ? st[r]
                      : (r < nblk ? __ldcg(loss_part + static_cast<int64_t>(c) * nblk + r)
                                  : __ldcg(frob_part + static_cast<int64_t>(c) * n_pairs + (r - nblk)));
      };
      double ls = 0.0;
      for (int r = 0; r < nblk; ++r) ls = __dadd_rn(ls, part(r));
      const double reg = __dmul_rn(__dmul_rn(0.5, lam_arr[c]), xx);
      f_cli[c] = __dadd_rn(__ddiv_rn(ls, static_cast<double>(ni_arr[c])), reg);
      if (frob_part) {
        double fp = 0.0;
        for (int r = 0; r < n_pairs; ++r) fp = __dadd_rn(fp, part(nblk + r));
        shift_cli[c] = sqrt(fp);
        if (flags[c] & 1) atomicMin(&s_bad, c);
      }
    }
  }
  __syncthreads();
  pc.mark(9);
  // ---- ticket: the last CTA forms the round scalars
  if (threadIdx.x == 0) {
    if (s_bad != 0x7fffffff) atomicMax(&ctl->reduce_bad, 0x7fffffff - s_bad);
    __threadfence();
    s_last = atomicAdd(&ctl->reduce_ticket, 1) == G - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double gg = 0.0, fs_part = 0.0, ss_part = 0.0;
  for (int a = threadIdx.x; a < d; a += RED_THREADS) {
    const double g = __ldcg(gbar + a);
    gg = fma(g, g, gg);
  }
  for (int i = threadIdx.x; i < n_active; i += RED_THREADS) {
    const int c = client_of(clients, i);
    fs_part += __ldcg(f_cli + c);
    if (frob_part) ss_part += __ldcg(shift_cli + c);
  }
  const double gn2 = block_sum(gg, red);
  const double fs = block_sum(fs_part, red);
  const double ss = block_sum(ss_part, red);
  pc.mark(10);
  if (threadIdx.x == 0) {
    ctl->reduce_ticket = 0;
    out->grad_norm = sqrt(gn2);
    out->f_mean = __ddiv_rn(fs, static_cast<double>(n_div));
    out->shift_mean = __ddiv_rn(ss, static_cast<double>(n_div));
    out->xx = xx;
    const int slot = ctl->round - ctl->row_base;
    if (row_grad) row_grad[slot] = out->grad_norm;
    if (row_f) row_f[slot] = out->f_mean;
    const int bad = atomicExch(&ctl->reduce_bad, 0);
    if (frob_part && bad != 0) {
      ctl->bad_client = 0x7fffffff - bad;
      raise_status(ctl, ST_NONFINITE);
    }
    tl_mark(12, true);
  }
}

// Holds the compressor (stream-ordered behind this one-thread kernel) until
// the solve's fused round reduction is done: the compressor streams the
// whole D through HBM, and the reduction's dependent loads (gradients,
// partials, x) would otherwise each wait several microseconds behind it
// (c0: 21 -> 12 us).  The factorisation that follows has ~20 us of slack
// over the compressor and fold.  Returns at once on a halted round; a gate
// that never opens traps (a loud failure, not a hang).
__global__ void k_wait_reduce(const DevCtl* __restrict__ ctl) {
  if (threadIdx.x != 0) return;
  const volatile int32_t* gate = &ctl->red_gate;
  const volatile int32_t* halt = &ctl->halt;
  const int32_t want = ctl->round + 1;
  for (uint32_t spin = 0; *gate != want && !*halt; ++spin) {
    __nanosleep(256);
    if (spin > (1u << 24)) asm volatile("trap;");
  }
}

// Dense kinds (identity / natural): client shift update + master fold per
// packed position t, clients in ascending id (compressors.py:373-393,
// algorithms.py:234, 369-372):
//   Hest[c][t] = fl(Hest + fl(alpha v)),  Hout[t] = fold_c fl(. + fl((alpha/n) v))
// with v = D[c][t] (identity) or its natural rounding (written into D).
__global__ void __launch_bounds__(256) k_fold_dense(
    const DevCtl* __restrict__ ctl, int64_t w, int n_active, const int32_t* __restrict__ clients,
    double alpha, double alpha_n, const double* __restrict__ D, const int32_t* __restrict__ count,
    double* __restrict__ hest, const double* h_in, double* h_out) {
  if (ctl->halt) return;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= w) return;
  double h = h_out ? h_in[t] : 0.0;
  constexpr int G = 8;  // clients per batch: independent loads in flight
  for (int i0 = 0; i0 < n_active; i0 += G) {
    int cc[G];
    double v[G], hv[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      cc[u] = (i0 + u < n_active) ? client_of(clients, i0 + u) : -1;
      const bool sel = cc[u] >= 0 && count[cc[u]] != 0;
      v[u] = sel ? D[static_cast<int64_t>(cc[u]) * w + t] : 0.0;
      hv[u] = (sel && hest) ? hest[static_cast<int64_t>(cc[u]) * w + t] : 0.0;
      if (!sel) cc[u] = -1;
    }
#pragma unroll
    for (int u = 0; u < G; ++u) {
      if (cc[u] < 0) continue;
      if (hest) hest[static_cast<int64_t>(cc[u]) * w + t] = __dadd_rn(hv[u], __dmul_rn(alpha, v[u]));
      if (h_out) h = __dadd_rn(h, __dmul_rn(alpha_n, v[u]));
    }
  }
  if (h_out) h_out[t] = h;
}

// Master fold of the sparse kinds (algorithms.py:369-372): one CTA per range
// of FOLD_RANGE packed positions.  Every client's ascending (idx, val) list is
// sliced by the compressor's range starts rs[c][r] and applied in ascending
// client order:  Hout[t] = fl(Hin[t] + fl((alpha/n) v_c))  — the reference's
// sequential sparse fold, bit for bit.  Hin may alias Hout.
//
// Per pass over a chunk of clients (at most FOLD_PC clients / FOLD_STAGE
// entries): every thread loads its entries (FOLD_EPT, all loads in flight)
// and sets bit (client) of its position's client mask; thread p then owns
// position p: its entry count is the mask's popcount, a block scan gives the
// position's slot range, each entry's rank inside it is the popcount of the
// mask below its client (so the slots hold the position's entries in client
// order), and thread p adds them in that order.  No step is sequential over
// clients.
constexpr int FOLD_THREADS = 256;
constexpr int FOLD_EPT = 12;                           // entries per thread and pass
constexpr int FOLD_STAGE = FOLD_EPT * FOLD_THREADS;    // entries per pass
constexpr int FOLD_PC = 512;                           // clients per pass
constexpr int FOLD_MW = FOLD_PC / 32;                  // mask words per position
static_assert(FOLD_RANGE == FOLD_THREADS, "thread p owns position p of the range");
__global__ void __launch_bounds__(FOLD_THREADS) k_master_fold(
    const DevCtl* __restrict__ ctl, int64_t w, int n_active, const int32_t* __restrict__ clients,
    int cap, int nr, const int32_t* __restrict__ rs, const uint32_t* __restrict__ idx_list,
    const double* __restrict__ val_list, double alpha_n, const double* h_in, double* h_out,
    double* __restrict__ hest = nullptr, int64_t hest_stride = 0, double alpha = 0.0) {
  if (ctl->halt) return;
  if (threadIdx.x == 0) tl_mark(5, false);
  extern __shared__ int32_t fold_sm[];  // beg[n], cnt[n], off[n+1]
  __shared__ uint32_t mask[FOLD_RANGE][FOLD_MW + 1];  // +1: conflict-free rows
  __shared__ double sv[FOLD_STAGE];
  __shared__ int pstart[FOLD_RANGE + 1];
  __shared__ int ws[64];
  int32_t* beg = fold_sm;
  int32_t* cnt = fold_sm + n_active;
  int32_t* off = fold_sm + 2 * n_active;
  const int tid = threadIdx.x;
  const int r = blockIdx.x;
  const int64_t t0 = static_cast<int64_t>(r) * FOLD_RANGE;
  const int len = static_cast<int>((w - t0 < FOLD_RANGE) ? (w - t0) : FOLD_RANGE);
  double h = tid < len ? h_in[t0 + tid] : 0.0;  // thread p owns position p
  for (int i = tid; i < n_active; i += FOLD_THREADS) {
    const int c = client_of(clients, i);
    const int32_t* rc = rs + static_cast<int64_t>(c) * (nr + 1);
    const int b = rc[r];
    beg[i] = b;
    cnt[i] = rc[r + 1] - b;
  }
  __syncthreads();
  // exclusive scan of cnt in client order (chunks of FOLD_THREADS)
  {
    int carry = 0;
    for (int base = 0; base < n_active; base += FOLD_THREADS) {
      const int i = base + tid;
      const int v = (i < n_active) ? cnt[i] : 0;
      int total;
      const int o = block_excl_scan(v, ws, &total) + carry;
      if (i < n_active) off[i] = o;
      carry += total;
    }
    if (tid == 0) off[n_active] = carry;
  }
  __syncthreads();
  int ca = 0;
  while (ca < n_active) {
    // largest cb with off[cb] - off[ca] <= FOLD_STAGE, cb - ca <= FOLD_PC (at least one client)
    int lo = ca + 1, hi = min(n_active, ca + FOLD_PC);
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] - off[ca] <= FOLD_STAGE) lo = mid; else hi = mid - 1;
    }
    const int cb = lo;
    const int e0 = off[ca], e1 = off[cb];  // a client's slice is <= FOLD_RANGE < FOLD_STAGE
    const int mwp = (cb - ca + 31) >> 5;
    for (int q = tid; q < FOLD_RANGE * mwp; q += FOLD_THREADS) mask[q / mwp][q % mwp] = 0u;
    // this thread's entries: client (binary search in the staged offsets),
    // then every load in flight
    int ci[FOLD_EPT], pp[FOLD_EPT];
    int64_t src[FOLD_EPT];
#pragma unroll
    for (int u = 0; u < FOLD_EPT; ++u) {
      const int e = e0 + u * FOLD_THREADS + tid;
      ci[u] = -1;
      src[u] = 0;
      if (e < e1) {
        int a = ca, b = cb - 1;
        while (a < b) {
          const int mid = (a + b + 1) >> 1;
          if (off[mid] <= e) a = mid; else b = mid - 1;
        }
        ci[u] = a;
        src[u] = static_cast<int64_t>(client_of(clients, a)) * cap + beg[a] + (e - off[a]);
      }
    }
    uint32_t ti[FOLD_EPT];
    double tv[FOLD_EPT];
#pragma unroll
    for (int u = 0; u < FOLD_EPT; ++u) {
      ti[u] = ci[u] >= 0 ? idx_list[src[u]] : 0u;
      tv[u] = ci[u] >= 0 ? val_list[src[u]] : 0.0;
    }
    __syncthreads();  // masks cleared
#pragma unroll
    for (int u = 0; u < FOLD_EPT; ++u) {
      if (ci[u] < 0) continue;
      if (hest) {  // the client shift update (compressors.py:373-393), distinct (c, t)
        double* hp = hest + static_cast<int64_t>(client_of(clients, ci[u])) * hest_stride + ti[u];
        *hp = __dadd_rn(*hp, __dmul_rn(alpha, tv[u]));
      }
      pp[u] = static_cast<int>(ti[u] - t0);
      const int k = ci[u] - ca;
      atomicOr(&mask[pp[u]][k >> 5], 1u << (k & 31));
    }
    __syncthreads();
    // position p's slot range: its mask's popcount, scanned over the range
    {
      int np = 0;
      for (int q = 0; q < mwp; ++q) np += __popc(mask[tid][q]);
      int total;
      pstart[tid] = block_excl_scan(np, ws, &total);
      if (tid == 0) pstart[FOLD_RANGE] = total;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < FOLD_EPT; ++u) {
      if (ci[u] < 0) continue;
      const int k = ci[u] - ca, p = pp[u];
      int rank = __popc(mask[p][k >> 5] & ((1u << (k & 31)) - 1u));
      for (int q = 0; q < (k >> 5); ++q) rank += __popc(mask[p][q]);
      sv[pstart[p] + rank] = tv[u];
    }
    __syncthreads();
    for (int j = pstart[tid]; j < pstart[tid + 1]; ++j) h = __dadd_rn(h, __dmul_rn(alpha_n, sv[j]));
    __syncthreads();  // sv / pstart / mask are rewritten by the next pass
    ca = cb;
  }
  if (tid < len) h_out[t0 + tid] = h;
  if (threadIdx.x == 0) tl_mark(5, true);
}

// Round epilogue (algorithms.py:385-387): x <- x_new, round += 1,
// DivergenceError on a non-finite iterate; per-client entry counts into the
// row buffers (-1 for clients that did not participate).  With
// ctl->stop_gn >= 0 a FedNL round whose row grad_norm <= stop_gn ends the run
// after its step (runtime.py:270-272): ST_STOPPED halts the later rounds of
// the chunk.
__global__ void __launch_bounds__(256) k_finish(
    DevCtl* __restrict__ ctl, int d, int n, int n_active, const int32_t* __restrict__ clients,
    double* __restrict__ x, const double* __restrict__ x_new, int copy_x,
    const int32_t* __restrict__ count, int32_t* __restrict__ row_counts,
    int32_t* __restrict__ row_ls, const double* __restrict__ row_grad,
    const double* __restrict__ hcopy_src = nullptr, double* __restrict__ hcopy_dst = nullptr,
    int64_t hcopy_n = 0) {
  // H^{k+1} (the fold's second buffer) back into H^k, over every block of the
  // grid (unconditionally, as the copy it replaces), then the epilogue on block 0
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < hcopy_n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    hcopy_dst[t] = hcopy_src[t];
  if (threadIdx.x == 0) tl_mark(6, false);
  if (blockIdx.x != 0) return;
  if (ctl->halt) return;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    const double v = copy_x ? x_new[a] : x[a];
    if (copy_x) x[a] = v;
    if (!isfinite(v)) bad = 1;
  }
  const int slot = ctl->round - ctl->row_base;
  if (row_counts) {
    int32_t* rc = row_counts + static_cast<int64_t>(slot) * n;
    if (clients) {
      for (int c = threadIdx.x; c < n; c += blockDim.x) rc[c] = -1;
      __syncthreads();
      for (int i = threadIdx.x; i < n_active; i += blockDim.x) rc[clients[i]] = count[clients[i]];
    } else {
      for (int c = threadIdx.x; c < n; c += blockDim.x) rc[c] = count[c];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (row_ls) row_ls[slot] = ctl->ls_steps;
    ctl->round += 1;
    if (bad) raise_status(ctl, ST_DIVERGED);
    else if (row_grad && ctl->stop_gn >= 0.0 && row_grad[slot] <= ctl->stop_gn)
      raise_status(ctl, ST_STOPPED);
    tl_mark(6, true);
  }
}

// FedNL-PP between the master's new point and the participants' round
// (runtime.py:235-243, algorithms.py:422-433): the row of round k describes
// x^k (the metric probes); when its grad_norm <= stop_gn the run ends BEFORE
// the step (the row counts, the round does not advance x).  Otherwise
// x <- x_new, DivergenceError on a non-finite new point.  One CTA.
__global__ void __launch_bounds__(256) k_pp_advance(DevCtl* __restrict__ ctl, int d, int n,
                                                     double* __restrict__ x,
                                                     const double* __restrict__ x_new,
                                                     const double* __restrict__ row_grad,
                                                     int32_t* __restrict__ row_counts,
                                                     int32_t* __restrict__ row_ls) {
  if (ctl->halt) return;
  __shared__ int s_stop, bad;
  const int slot = ctl->round - ctl->row_base;
  if (threadIdx.x == 0) {
    s_stop = ctl->stop_gn >= 0.0 && row_grad[slot] <= ctl->stop_gn;
    bad = 0;
  }
  __syncthreads();
  if (s_stop) {  // no participant this round
    for (int c = threadIdx.x; c < n; c += blockDim.x) row_counts[static_cast<int64_t>(slot) * n + c] = -1;
    __syncthreads();
    if (threadIdx.x == 0) {
      row_ls[slot] = 0;
      ctl->round += 1;
      raise_status(ctl, ST_STOPPED);
    }
    return;
  }
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    const double v = x_new[a];
    x[a] = v;
    if (!isfinite(v)) bad = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0 && bad) raise_status(ctl, ST_DIVERGED);
}

// ------------------------------------------------------------------ FedNL-PP

// Participant subset of the round: the persistent TAG_MASTER stream's
// partial Fisher-Yates prefix of range(n) of length tau, sorted ascending
// (algorithms.py:422-425).  One thread.
__global__ void k_pp_select(DevCtl* __restrict__ ctl, int n, int tau, int32_t* __restrict__ subset,
                            int32_t* __restrict__ pool) {
  // the swap chain in shared memory when the pool fits (one thread draws)
  constexpr int SMAX = 4096;
  __shared__ int32_t pool_s[SMAX];
  int32_t* pl = n <= SMAX ? pool_s : pool;
  for (int i = threadIdx.x; i < n; i += blockDim.x) pl[i] = i;
  __syncthreads();
  if (threadIdx.x != 0 || ctl->halt) return;
  Prg p(ctl->master_state);
  for (int i = 0; i < tau; ++i) {
    const int j = i + static_cast<int>(p.randrange(static_cast<uint64_t>(n - i)));
    const int32_t tmp = pl[i];
    pl[i] = pl[j];
    pl[j] = tmp;
  }
  ctl->master_state = p.state;
  for (int i = 0; i < tau; ++i) subset[i] = pl[i];
  for (int i = 1; i < tau; ++i) {  // insertion sort (tau is small)
    const int32_t v = subset[i];
    int j = i - 1;
    while (j >= 0 && subset[j] > v) { subset[j + 1] = subset[j]; --j; }
    subset[j + 1] = v;
  }
}

// Per participant after its shift update (algorithms.py:250-256):
//   shift_new = ||Hest_c - hess||_F,  gvec_new = Hest_c x + shift_new x - grad_c
// and the increments against the stored client state.
// k_pp_shift_part: grid (PP_SB, tau), block 256 — Frobenius partials.
// k_pp_client:     grid (ceil(d / 8), tau), block 256 — one warp per row a of
//   Hest_c x (b <= a: packed column a, contiguous; b > a: packed columns b);
//   the CTAs of a client each fold the PP_SB partials in the same order.
constexpr int PP_SB = 16;
__global__ void __launch_bounds__(256) k_pp_shift_part(
    const DevCtl* __restrict__ ctl, int d, const int32_t* __restrict__ subset,
    const double* __restrict__ hest, const double* __restrict__ hess_part,
    double* __restrict__ shift_part) {
  if (ctl->halt) return;
  __shared__ double red[8];
  const int slot = blockIdx.y;
  const int c = subset[slot];
  const int64_t w = packed_len(d);
  const double* hc = hest + static_cast<int64_t>(c) * w;
  const double* hp = hess_part + static_cast<int64_t>(slot) * w;
  double part = 0.0;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < w;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double dv = __dsub_rn(hc[t], hp[t]);
    const double wt = packed_is_diag_fast(t) ? 1.0 : 2.0;
    part = fma(__dmul_rn(wt, dv), dv, part);
  }
  const double tot = block_sum(part, red);
  if (threadIdx.x == 0) shift_part[slot * PP_SB + blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256) k_pp_client(
    const DevCtl* __restrict__ ctl, int d, const int32_t* __restrict__ subset,
    const double* __restrict__ hest, const double* __restrict__ shift_part,
    const double* __restrict__ x, const double* __restrict__ grad,
    double* __restrict__ cli_shift, double* __restrict__ cli_gvec,
    double* __restrict__ dshift, double* __restrict__ dgvec) {
  if (ctl->halt) return;
  const int slot = blockIdx.y;
  const int c = subset[slot];
  const int64_t w = packed_len(d);
  const double* hc = hest + static_cast<int64_t>(c) * w;
  double tot = 0.0;
  for (int q = 0; q < PP_SB; ++q) tot += shift_part[slot * PP_SB + q];
  const double sh = sqrt(tot);
  const int lane = threadIdx.x & 31;
  const int a = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (a < d) {
    double s = 0.0;
    const int64_t ca = packed_at(0, a);
    for (int b = lane; b <= a; b += 32) s = fma(__ldg(hc + ca + b), __ldg(x + b), s);
    for (int b = a + 1 + lane; b < d; b += 32) s = fma(__ldg(hc + packed_at(a, b)), __ldg(x + b), s);
    s = warp_sum(s);
    if (lane == 0) {
      const double gnew = __dsub_rn(__dadd_rn(s, __dmul_rn(sh, x[a])), grad[static_cast<int64_t>(c) * d + a]);
      const double gold = cli_gvec[static_cast<int64_t>(c) * d + a];
      dgvec[static_cast<int64_t>(slot) * d + a] = __dsub_rn(gnew, gold);
      cli_gvec[static_cast<int64_t>(c) * d + a] = gnew;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    dshift[slot] = __dsub_rn(sh, cli_shift[c]);
    cli_shift[c] = sh;
  }
}

// Master running averages (algorithms.py:435-441): ascending participants,
// gvec = gvec + dg / n, shift += ds / n.  Single CTA.
__global__ void __launch_bounds__(256) k_pp_master(
    const DevCtl* __restrict__ ctl, int d, int n, int tau, const double* __restrict__ dshift,
    const double* __restrict__ dgvec, double* __restrict__ gvec, double* __restrict__ shift) {
  if (ctl->halt) return;
  const double nn = static_cast<double>(n);
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    double g = gvec[a];
    for (int i0 = 0; i0 < tau; i0 += 8) {  // 8 loads in flight, added in client order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = i0 + u < tau ? dgvec[static_cast<int64_t>(i0 + u) * d + a] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i0 + u < tau) g = __dadd_rn(g, __ddiv_rn(v[u], nn));
    }
    gvec[a] = g;
  }
  if (threadIdx.x == 0) {
    double s = *shift;
    for (int i = 0; i < tau; ++i) s = __dadd_rn(s, __ddiv_rn(dshift[i], nn));
    *shift = s;
  }
}

// k_check_flags_pp: non-finite participant difference -> ST_NONFINITE
__global__ void k_check_flags_pp(DevCtl* ctl, int tau, const int32_t* subset,
                                 const int32_t* flags) {
  if (ctl->halt) return;
  // one warp, 32 participants per step; the first bad one in subset order
  for (int i0 = 0; i0 < tau; i0 += 32) {
    const int i = i0 + static_cast<int>(threadIdx.x);
    const int c = i < tau ? (subset ? subset[i] : i) : -1;
    const uint32_t bad = __ballot_sync(0xffffffffu, c >= 0 && (flags[c] & 1));
    if (bad) {
      if (threadIdx.x == __ffs(bad) - 1) {
        ctl->bad_client = c;
        raise_status(ctl, ST_NONFINITE);
      }
      return;
    }
  }
}

// ----------------------------------------------- FedNL-PP across GPUs
// Sharded FedNL-PP (fb_set_shard): every rank draws the same participant
// subset (replicated master stream) and rank r computes the participant
// slots [r * spr, (r + 1) * spr) of it (B and every H_i^k are held by every
// rank).  The owner's per-slot results go through a slot-major exchange
// buffer (all-gathered in blocks of spr slots): the compressed delta, the
// client's new shift / shifted gradient and their increments, the flags.
// Every rank then holds every participant's outputs and applies the client
// shift update of the slots it did not compute itself (the same
// fl(h + fl(alpha v)) the owner applied), so all ranks keep identical state.
struct PpX {
  uint32_t* idx;    // [tau_pad][cap]
  double* val;      // [tau_pad][cap]
  int32_t* cnt;     // [tau_pad]
  int32_t* rs;      // [tau_pad][nr + 1]
  int32_t* flags;   // [tau_pad]
  double* gvec;     // [tau_pad][d]  client's new shifted gradient
  double* shift;    // [tau_pad]     client's new shift
  double* dg;       // [tau_pad][d]  its increment (master running average)
  double* ds;       // [tau_pad]
  double* dense;    // [tau_pad][w]  dense kinds: the (rounded) update, else null
  int32_t* code;    // [world]       each rank's status code after its slots
};
// this rank's participants: sub_loc[i] = subset[s_lo + i], i < m
__global__ void k_pp_subloc(const int32_t* __restrict__ subset, int s_lo, int m,
                            int32_t* __restrict__ sub_loc) {
  for (int i = threadIdx.x; i < m; i += blockDim.x) sub_loc[i] = subset[s_lo + i];
}
// grid m (this rank's slots), block 256
__global__ void __launch_bounds__(256) k_pp_pack(const DevCtl* __restrict__ ctl, int d, int64_t w,
                                                 int cap, int nr, int s_lo, int rank,
                                                 const int32_t* __restrict__ sub_loc,
                                                 const uint32_t* __restrict__ idx_list,
                                                 const double* __restrict__ val_list,
                                                 const int32_t* __restrict__ count,
                                                 const int32_t* __restrict__ rs,
                                                 const int32_t* __restrict__ flags,
                                                 const double* __restrict__ cli_gvec,
                                                 const double* __restrict__ cli_shift,
                                                 const double* __restrict__ dgvec,
                                                 const double* __restrict__ dshift,
                                                 const double* __restrict__ D, PpX x) {
  const int i = blockIdx.x, j = s_lo + i;
  const int c = sub_loc[i];
  const int cn = count[c];
  for (int e = threadIdx.x; e < cap; e += blockDim.x)
    if (e < cn) {
      x.idx[static_cast<int64_t>(j) * cap + e] = idx_list[static_cast<int64_t>(c) * cap + e];
      x.val[static_cast<int64_t>(j) * cap + e] = val_list[static_cast<int64_t>(c) * cap + e];
    }
  for (int r = threadIdx.x; r <= nr; r += blockDim.x)
    x.rs[static_cast<int64_t>(j) * (nr + 1) + r] = rs[static_cast<int64_t>(c) * (nr + 1) + r];
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    x.gvec[static_cast<int64_t>(j) * d + a] = cli_gvec[static_cast<int64_t>(c) * d + a];
    x.dg[static_cast<int64_t>(j) * d + a] = dgvec[static_cast<int64_t>(i) * d + a];
  }
  if (x.dense)
    for (int64_t t = threadIdx.x; t < w; t += blockDim.x)
      x.dense[static_cast<int64_t>(j) * w + t] = D[static_cast<int64_t>(c) * w + t];
  if (threadIdx.x == 0) {
    x.cnt[j] = cn;
    x.flags[j] = flags[c];
    x.shift[j] = cli_shift[c];
    x.ds[j] = dshift[i];
  }
}
// grid tau (every slot), block 256: the per-client rows / state of every
// participant, the slot-major increments, and the client shift update of the
// slots owned by other ranks
__global__ void __launch_bounds__(256) k_pp_unpack(DevCtl* __restrict__ ctl, int d, int64_t w,
                                                   int cap, int nr, int s_lo, int s_hi, int world,
                                                   double alpha, const int32_t* __restrict__ subset,
                                                   PpX x, uint32_t* __restrict__ idx_list,
                                                   double* __restrict__ val_list,
                                                   int32_t* __restrict__ count, int32_t* __restrict__ rs,
                                                   int32_t* __restrict__ flags,
                                                   double* __restrict__ cli_gvec,
                                                   double* __restrict__ cli_shift,
                                                   double* __restrict__ dgvec_all,
                                                   double* __restrict__ dshift_all,
                                                   double* __restrict__ D, double* __restrict__ hest) {
  const int j = blockIdx.x;
  const int c = subset[j];
  const bool mine = j >= s_lo && j < s_hi;
  if (j == 0 && threadIdx.x == 0 && ctl->code == 0) {  // a rank-local failure halts every rank
    for (int r = 0; r < world; ++r)
      if (x.code[r] != 0) {
        raise_status(ctl, x.code[r]);
        break;
      }
  }
  const int cn = x.cnt[j];
  double* hc = hest + static_cast<int64_t>(c) * w;
  for (int e = threadIdx.x; e < cn; e += blockDim.x) {
    const uint32_t t = x.idx[static_cast<int64_t>(j) * cap + e];
    const double v = x.val[static_cast<int64_t>(j) * cap + e];
    idx_list[static_cast<int64_t>(c) * cap + e] = t;
    val_list[static_cast<int64_t>(c) * cap + e] = v;
    if (!mine && !x.dense) hc[t] = __dadd_rn(hc[t], __dmul_rn(alpha, v));  // distinct t
  }
  if (x.dense && cn != 0)
    for (int64_t t = threadIdx.x; t < w; t += blockDim.x) {
      const double v = x.dense[static_cast<int64_t>(j) * w + t];
      D[static_cast<int64_t>(c) * w + t] = v;
      if (!mine) hc[t] = __dadd_rn(hc[t], __dmul_rn(alpha, v));
    }
  for (int r = threadIdx.x; r <= nr; r += blockDim.x)
    rs[static_cast<int64_t>(c) * (nr + 1) + r] = x.rs[static_cast<int64_t>(j) * (nr + 1) + r];
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    cli_gvec[static_cast<int64_t>(c) * d + a] = x.gvec[static_cast<int64_t>(j) * d + a];
    dgvec_all[static_cast<int64_t>(j) * d + a] = x.dg[static_cast<int64_t>(j) * d + a];
  }
  if (threadIdx.x == 0) {
    count[c] = cn;
    flags[c] = x.flags[j];
    cli_shift[c] = x.shift[j];
    dshift_all[j] = x.ds[j];
  }
}

// Sharded FedNL: every rank's status code after its own clients' work
// (compressor failures are rank-local), all-gathered; the first raised code
// halts every rank (otherwise the others would go on calling collectives)
__global__ void k_code_post(const DevCtl* __restrict__ ctl, int rank, int32_t* __restrict__ code) {
  if (threadIdx.x == 0) code[rank] = ctl->code;
}
__global__ void k_code_sync(DevCtl* __restrict__ ctl, int world, const int32_t* __restrict__ code) {
  if (threadIdx.x != 0 || ctl->code != 0) return;
  for (int r = 0; r < world; ++r)
    if (code[r] != 0) {
      raise_status(ctl, code[r]);
      return;
    }
}

// ------------------------------------------------------------ initialisation

// Hest[c] = lam_c I (cli_diag set: the shard's lambda) or 0 for every
// client, Hmas = master_diag I (algorithms.py:202-206: ClientShard.lam;
// 334-335: RunConfig.lam).  grid (ceil(w/256), n + 1).
__global__ void k_init_diag(int64_t w, int n, const double* __restrict__ cli_diag,
                            double master_diag, double* __restrict__ hest,
                            double* __restrict__ hmas) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= w) return;
  const bool dg = packed_is_diag_fast(t);
  if (blockIdx.y < static_cast<unsigned>(n))
    hest[static_cast<int64_t>(blockIdx.y) * w + t] = (dg && cli_diag) ? cli_diag[blockIdx.y] : 0.0;
  else if (hmas)
    hmas[t] = dg ? master_diag : 0.0;
}

// exact init (algorithms.py:336-341): Hmas = (sum_c Hest_c) / n, ascending c.
__global__ void k_mean_packed(int64_t w, int n, const double* __restrict__ hest,
                              double* __restrict__ hmas) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= w) return;
  double s = 0.0;
  for (int c = 0; c < n; ++c) s = __dadd_rn(s, hest[static_cast<int64_t>(c) * w + t]);
  hmas[t] = __ddiv_rn(s, static_cast<double>(n));
}

// PP init (algorithms.py:211-222, 342-349) for all clients at x0:
// cli_shift[c] = ||Hest_c - hess_c|| (= sqrt of the Hessian kernel's
// Frobenius partials), cli_gvec[c] = Hest_c x0 + shift x0 - grad_c.
__global__ void __launch_bounds__(256) k_pp_init_client(
    int d, int n_pairs, const double* __restrict__ hest, const double* __restrict__ x,
    const double* __restrict__ grad, const double* __restrict__ frob_part,
    double* __restrict__ cli_shift, double* __restrict__ cli_gvec) {
  const int c = blockIdx.x;
  const int64_t w = packed_len(d);
  const double* hc = hest + static_cast<int64_t>(c) * w;
  double fp = 0.0;
  for (int p = 0; p < n_pairs; ++p) fp = __dadd_rn(fp, frob_part[static_cast<int64_t>(c) * n_pairs + p]);
  const double sh = sqrt(fp);
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < d; ++b) {
      const int64_t tt = (a <= b) ? packed_at(a, b) : packed_at(b, a);
      s = fma(hc[tt], x[b], s);
    }
    cli_gvec[static_cast<int64_t>(c) * d + a] =
        __dsub_rn(__dadd_rn(s, __dmul_rn(sh, x[a])), grad[static_cast<int64_t>(c) * d + a]);
  }
  if (threadIdx.x == 0) cli_shift[c] = sh;
}

__global__ void k_pp_init_master(int d, int n, const double* __restrict__ cli_shift,
                                 const double* __restrict__ cli_gvec, double* __restrict__ gvec,
                                 double* __restrict__ shift) {
  for (int a = threadIdx.x; a < d; a += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < n; ++c) s = __dadd_rn(s, cli_gvec[static_cast<int64_t>(c) * d + a]);
    gvec[a] = __ddiv_rn(s, static_cast<double>(n));
  }
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int c = 0; c < n; ++c) s = __dadd_rn(s, cli_shift[c]);
    *shift = __ddiv_rn(s, static_cast<double>(n));
  }
}

// ------------------------------------------------------------- line search

// After a trial batch: f_trial[s] = mean_c (loss_sum / n_i + reg(trial_s));
// accept the first s with f_trial <= f_x - c * step * decrement
// (algorithms.py:302-311).  The trial/decide pair is the body of a
// while-conditional graph node (`loop`): the body runs again (next batch of
// LS_BATCH trials) until a trial is accepted, or past s = 60 ST_LINE_SEARCH
// is raised.  Every exit path clears the loop condition, including a round
// that is already halted.  Single CTA of 256 threads.
constexpr int LS_DECIDE_MAXN = 4096;
__global__ void __launch_bounds__(256) k_ls_decide(
    DevCtl* __restrict__ ctl, int d, int n, const int32_t* __restrict__ ni_arr,
    const double* __restrict__ lam_arr, int nblk, double ls_c,
    const double* __restrict__ steps_table, const double* __restrict__ trial_x,
    const double* __restrict__ loss_part, RoundScalars* __restrict__ sc,
    double* __restrict__ x_new, int batch, const double* __restrict__ gbar,
    const double* __restrict__ p, cudaGraphConditionalHandle loop) {
  const int s0 = ctl->ls_next;
  if (threadIdx.x == 0) tl_mark(14, true);
  if (ctl->halt || s0 > 60) {  // nothing to decide: leave the loop
    if (threadIdx.x == 0) {
      ctl->ls_next = 0;
      cudaGraphSetConditional(loop, 0);
    }
    return;
  }
  __shared__ double red[8];
  __shared__ int s_acc;
  __shared__ double s_fbest;
  __shared__ double s_lsum[LS_DECIDE_MAXN];  // per-client f of one trial
  if (s0 == 0) {  // decrement = <gbar, p> (algorithms.py:302), as k_dot forms it
    double part = 0.0;
    for (int i = threadIdx.x; i < d; i += blockDim.x) part = fma(gbar[i], p[i], part);
    const double dec = block_sum(part, red);
    if (threadIdx.x == 0) sc->decrement = dec;
    __syncthreads();
  }
  if (threadIdx.x == 0) { s_acc = -1; s_fbest = (s0 == 0) ? INFINITY : ctl->f_best; }
  __syncthreads();
  auto client_f = [&](int s, int c, double xx) {  // oracle.py:95-105
    const double* lp = loss_part + (static_cast<int64_t>(c) * LS_BATCH + s) * nblk;
    double ls = 0.0;
    for (int b = 0; b < nblk; ++b) ls = __dadd_rn(ls, __ldcg(lp + b));
    const double reg = __dmul_rn(__dmul_rn(0.5, lam_arr[c]), xx);
    return __dadd_rn(__ddiv_rn(ls, static_cast<double>(ni_arr[c])), reg);
  };
  for (int s = 0; s < batch; ++s) {
    const int si = s0 + s;
    const double* xt = trial_x + static_cast<int64_t>(s) * d;
    double part = 0.0;
    for (int a = threadIdx.x; a < d; a += blockDim.x) part = fma(xt[a], xt[a], part);
    const double xx = block_sum(part, red);
    // per-client f in parallel (client order is restored by the sequential
    // fold below)
    for (int c = threadIdx.x; c < n && c < LS_DECIDE_MAXN; c += blockDim.x) s_lsum[c] = client_f(s, c, xx);
    __syncthreads();
    if (threadIdx.x == 0 && s_acc < 0 && si <= 60) {
      double tot = 0.0;
      for (int c = 0; c < n; ++c) tot = __dadd_rn(tot, c < LS_DECIDE_MAXN ? s_lsum[c] : client_f(s, c, xx));
      const double ft = __ddiv_rn(tot, static_cast<double>(n));
      const double step = steps_table[si];
      const double rhs = __dsub_rn(sc->f_mean, __dmul_rn(__dmul_rn(ls_c, step), sc->decrement));
      if (ft <= rhs) s_acc = si;
      else s_fbest = fmin(s_fbest, ft);
    }
    __syncthreads();
    if (s_acc >= 0) break;  // accepted: the batch's later trials are not needed (block-uniform)
  }
  const int acc = s_acc;
  if (acc >= 0) {
    const double* xt = trial_x + static_cast<int64_t>(acc - s0) * d;
    for (int a = threadIdx.x; a < d; a += blockDim.x) x_new[a] = xt[a];
  }
  if (threadIdx.x == 0) {
    if (acc >= 0) {
      ctl->ls_steps = acc;
      ctl->ls_next = 0;
      cudaGraphSetConditional(loop, 0);
    } else if (s0 + batch > 60) {
      ctl->f_start = sc->f_mean;
      ctl->f_best = s_fbest;
      ctl->ls_next = 0;
      raise_status(ctl, ST_LINE_SEARCH);
      cudaGraphSetConditional(loop, 0);
    } else {  // the next batch of trials
      ctl->f_best = s_fbest;
      ctl->ls_next = s0 + batch;
      cudaGraphSetConditional(loop, 1);
    }
  }
}

// decrement = <gbar, p> (algorithms.py:302)
__global__ void __launch_bounds__(256) k_dot(const DevCtl* __restrict__ ctl, int d,
                                             const double* __restrict__ a,
                                             const double* __restrict__ b,
                                             RoundScalars* __restrict__ sc) {
  if (ctl->halt) return;
  __shared__ double red[8];
  double part = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) part = fma(a[i], b[i], part);
  const double s = block_sum(part, red);
  if (threadIdx.x == 0) sc->decrement = s;
}

}  // namespace fb
