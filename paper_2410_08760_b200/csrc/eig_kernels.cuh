// eig_kernels.cuh — FedNL option (a): the Newton system is the estimate with
// its eigenvalues lifted to the floor mu (algorithms.py:361-364,
// linalg.py:189-259 eigen_clamp_min / jacobi_eigh).
//
// The reference runs cyclic Jacobi (one rotation at a time, p < q in row
// order) until the off-diagonal Frobenius mass is <= 1e-12 ||A||_F, at most
// 30 sweeps, then forms (V max(L, mu)) V^T and symmetrizes from the upper
// triangle.  Here the same rotation (theta, t, c, s formulas, |a_pq| <= 1e-300
// skipped, a_pq := 0 afterwards) is applied in the parallel (round-robin)
// Jacobi order: each sweep is n'-1 rounds of n'/2 disjoint pairs (n' = d
// rounded up to even), every round one J^T A J of commuting rotations, so the
// same convergence test and sweep limit apply.  The eigen-decomposition is
// unique up to the order of rotations; the clamped matrix is a continuous
// function of A, so it agrees with the reference to rounding (checked at
// 1e-10 normwise against the oracle in tests/).
//
// One CTA of 1024 threads: A (d x d, row-major, both triangles) lives in
// shared memory when it fits (d <= 160) and in global memory (L2-resident)
// otherwise; V^T (row k = eigenvector k) in global memory.  Latency-bound
// (4 CTA barriers per round, (d-1) rounds per sweep): option (a) is outside
// the BASELINE configs and this is its correctness path.
#pragma once

#include "common.cuh"

namespace fb {

constexpr int EIG_THREADS = 1024;
constexpr int EIG_SMEM_MAX_D = 160;  // A in shared memory up to 160 x 160 (200 KB)
constexpr int EIG_MAX_SWEEPS = 30;   // linalg.py:190 max_sweeps
__host__ __device__ constexpr size_t eig_smem_bytes(int d) {
  return d <= EIG_SMEM_MAX_D ? static_cast<size_t>(d) * d * 8 : 0;
}

// round-robin (circle method) pair k of round r over players 0..np-1
// (np even; player np-1 fixed): every pair exactly once per np-1 rounds
__device__ __forceinline__ void eig_pair(int np, int r, int k, int& p, int& q) {
  const int m = np - 1;
  if (k == 0) {
    p = m;
    q = r;
  } else {
    p = (r + k) % m;
    q = (r - k + m) % m;
  }
  if (p > q) { const int t = p; p = q; q = t; }
}

__device__ double eig_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    s = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// out (packed upper, column-wise t = j(j+1)/2 + i) = eigen_clamp_min(H, mu)
// for H given packed the same way.  eig_out (nullable): the eigenvalues in
// the order of V's rows.  Raises ST_EIGEN when the sweeps run out.
__global__ void __launch_bounds__(EIG_THREADS, 1) k_eig_clamp(
    DevCtl* __restrict__ ctl, int d, const double* __restrict__ hpk, const double* __restrict__ mu_ptr,
    double mu_val, double* __restrict__ Ag, double* __restrict__ Vt, double* __restrict__ out,
    double* __restrict__ eig_out, int ignore_halt) {
  if (!ignore_halt && ctl->halt) return;
  extern __shared__ __align__(16) double eig_sm[];
  __shared__ double red[33];
  __shared__ double cs[EIG_THREADS / 2 + 1], sn[EIG_THREADS / 2 + 1];
  __shared__ int pp[EIG_THREADS / 2 + 1], qq[EIG_THREADS / 2 + 1];
  const int tid = threadIdx.x;
  const double mu = mu_ptr ? *mu_ptr : mu_val;
  double* A = d <= EIG_SMEM_MAX_D ? eig_sm : Ag;
  const int64_t w = packed_len(d);
  // A <- H (both triangles), V^T <- I; ||A||_F the reference's way
  // (frobenius_norm_symmetric: weights 1 on the diagonal, 2 off it)
  double fro = 0.0;
  for (int64_t t = tid; t < w; t += EIG_THREADS) {
    const int j = static_cast<int>((sqrt(8.0 * static_cast<double>(t) + 1.0) - 1.0) * 0.5);
    int jj = j;
    while (packed_len(jj + 1) <= t) ++jj;
    while (packed_len(jj) > t) --jj;
    const int i = static_cast<int>(t - packed_len(jj));
    const double v = hpk[t];
    A[static_cast<int64_t>(i) * d + jj] = v;
    A[static_cast<int64_t>(jj) * d + i] = v;
    fro += (i == jj ? 1.0 : 2.0) * v * v;
  }
  for (int64_t e = tid; e < static_cast<int64_t>(d) * d; e += EIG_THREADS)
    Vt[e] = (e / d == e % d) ? 1.0 : 0.0;
  const double norm = sqrt(eig_block_sum(fro, red));
  const double thresh = 1e-12 * norm;
  const int np = d + (d & 1);
  const int npairs = np / 2;
  bool converged = d == 1 || norm == 0.0;
  for (int sweep = 0; sweep <= EIG_MAX_SWEEPS && !converged; ++sweep) {
    // off-diagonal mass sqrt(2 sum_{i<j} a_ij^2)
    double off = 0.0;
    for (int64_t e = tid; e < static_cast<int64_t>(d) * d; e += EIG_THREADS) {
      const int i = static_cast<int>(e / d), j = static_cast<int>(e % d);
      if (i < j) off += A[e] * A[e];
    }
    off = sqrt(2.0 * eig_block_sum(off, red));
    if (off <= thresh) { converged = true; break; }
    if (sweep == EIG_MAX_SWEEPS) break;
    for (int r = 0; r < np - 1; ++r) {
      // rotation parameters of the round's pairs (linalg.py:222-229)
      for (int k = tid; k < npairs; k += EIG_THREADS) {
        int p, q;
        eig_pair(np, r, k, p, q);
        double c = 1.0, s = 0.0;
        if (q < d) {
          const double apq = A[static_cast<int64_t>(p) * d + q];
          if (fabs(apq) > 1e-300) {
            const double theta = (A[static_cast<int64_t>(q) * d + q] - A[static_cast<int64_t>(p) * d + p]) / (2.0 * apq);
            const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
          }
        } else {
          q = -1;  // the bye of an odd dimension
        }
        pp[k] = p;
        qq[k] = (s == 0.0 && c == 1.0) ? -1 : q;
        cs[k] = c;
        sn[k] = s;
      }
      __syncthreads();
      // rows p, q of A and of V^T (= columns of V)
      for (int64_t it = tid; it < static_cast<int64_t>(npairs) * d; it += EIG_THREADS) {
        const int k = static_cast<int>(it / d), j = static_cast<int>(it % d);
        const int q = qq[k];
        if (q < 0) continue;
        const int p = pp[k];
        const double c = cs[k], s = sn[k];
        double* ap = A + static_cast<int64_t>(p) * d + j;
        double* aq = A + static_cast<int64_t>(q) * d + j;
        const double rp = *ap, rq = *aq;
        *ap = c * rp - s * rq;
        *aq = s * rp + c * rq;
        double* vp = Vt + static_cast<int64_t>(p) * d + j;
        double* vq = Vt + static_cast<int64_t>(q) * d + j;
        const double xp = *vp, xq = *vq;
        *vp = c * xp - s * xq;
        *vq = s * xp + c * xq;
      }
      __syncthreads();
      // columns p, q of A
      for (int64_t it = tid; it < static_cast<int64_t>(npairs) * d; it += EIG_THREADS) {
        const int i = static_cast<int>(it / npairs), k = static_cast<int>(it % npairs);
        const int q = qq[k];
        if (q < 0) continue;
        const int p = pp[k];
        const double c = cs[k], s = sn[k];
        double* ap = A + static_cast<int64_t>(i) * d + p;
        double* aq = A + static_cast<int64_t>(i) * d + q;
        const double cp = *ap, cq = *aq;
        *ap = c * cp - s * cq;
        *aq = s * cp + c * cq;
      }
      __syncthreads();
      for (int k = tid; k < npairs; k += EIG_THREADS) {
        const int q = qq[k];
        if (q < 0) continue;
        const int p = pp[k];
        A[static_cast<int64_t>(p) * d + q] = 0.0;
        A[static_cast<int64_t>(q) * d + p] = 0.0;
      }
      __syncthreads();
    }
  }
  if (!converged) {
    if (tid == 0) raise_status(ctl, ST_EIGEN);
    return;
  }
  if (eig_out)
    for (int k = tid; k < d; k += EIG_THREADS) eig_out[k] = A[static_cast<int64_t>(k) * d + k];
  // (V max(L, mu)) V^T, upper triangle, packed (linalg.py:255-258)
  __syncthreads();
  if (d <= EIG_SMEM_MAX_D) {  // the diagonal to the front of shared memory
    double dk = 0.0;
    if (tid < d) dk = A[static_cast<int64_t>(tid) * d + tid];
    __syncthreads();
    if (tid < d) eig_sm[tid] = fmax(dk, mu);
  } else {
    for (int k = tid; k < d; k += EIG_THREADS) Ag[k] = fmax(Ag[static_cast<int64_t>(k) * d + k], mu);
  }
  __syncthreads();
  const double* lam = d <= EIG_SMEM_MAX_D ? eig_sm : Ag;
  for (int64_t t = tid; t < w; t += EIG_THREADS) {
    int j = static_cast<int>((sqrt(8.0 * static_cast<double>(t) + 1.0) - 1.0) * 0.5);
    while (packed_len(j + 1) <= t) ++j;
    while (packed_len(j) > t) --j;
    const int i = static_cast<int>(t - packed_len(j));
    double acc = 0.0;
    for (int k = 0; k < d; ++k)
      acc = fma(Vt[static_cast<int64_t>(k) * d + i] * lam[k], Vt[static_cast<int64_t>(k) * d + j], acc);
    out[t] = acc;
  }
}

}  // namespace fb
