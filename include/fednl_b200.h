/*
 * fednl_b200.h — C ABI of the B200-native FedNL round (libfednl_b200.so).
 *
 * Drop-in boundary for the reference's simulated FedNL path
 * (arxiv/paper_2410_08760, /root/reference/pkg/src/fednl).  The reference is
 * pure Python/numpy; the entry points below replace, one for one, the
 * Python-level operations its simulator drives (citations are reference
 * file:line).  The Python package paper_2410_08760_b200 binds them with
 * ctypes; INTEGRATION.md shows the stub a reference maintainer would add.
 *
 * Conventions
 *   - Plain pointers and sizes only; every pointer argument is HOST memory.
 *     Device memory, the CUDA stream and the captured round graphs are owned
 *     by the opaque context and never cross the ABI.
 *   - Packed symmetric layout: upper triangle, column-wise,
 *     t(i, j) = j (j + 1) / 2 + i for i <= j   (reference linalg.py:54-58).
 *   - Shards: n host pointers, each an F-order (column-major) d x n_i double
 *     matrix whose column j is label_j * (features_j, 1)  (oracle.py:33-46).
 *   - Return value 0 = ok, otherwise an FB_ERR_* code; fb_last_error() and
 *     fb_get_status() give the detail.  A context is not re-entrant: one host
 *     thread per context.
 */
#ifndef FEDNL_B200_H
#define FEDNL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return / status codes ------------------------------------------- */
#define FB_OK 0
#define FB_ERR_CUDA 1          /* CUDA runtime/driver failure                */
#define FB_ERR_INVALID 2       /* bad argument / config (-> ValueError)      */
#define FB_ERR_NOT_PD 3        /* linalg.py:24-33 NotPositiveDefiniteError   */
#define FB_ERR_NONFINITE 4     /* compressors.py:134 non-finite input        */
#define FB_ERR_DIVERGED 5      /* algorithms.py:52-57 DivergenceError        */
#define FB_ERR_LINE_SEARCH 6   /* algorithms.py:41-49 LineSearchError        */
#define FB_ERR_UNSUPPORTED 7   /* outside this build's envelope              */
/* (8 was an internal line-search continuation code, retired: the trial
 * batches now loop inside the round graph) */
#define FB_ERR_EIGEN 9         /* linalg.py:36 EigenConvergenceError         */

/* compressor kinds (compressors.py:41-47) */
#define FB_KIND_IDENTITY 0
#define FB_KIND_TOPK 1
#define FB_KIND_TOPLEK 2
#define FB_KIND_RANDK 3
#define FB_KIND_RANDSEQK 4
#define FB_KIND_NATURAL 5

/* algorithms (algorithms.py:35) */
#define FB_ALG_FEDNL 0
#define FB_ALG_LS 1
#define FB_ALG_PP 2

/* Newton system (algorithms.py:361-367): option b = H^k + l^k I, option a =
 * eigen_clamp_min(H^k, mu) */
#define FB_OPTION_B 0
#define FB_OPTION_A 1

/* TopK variant for w > 32,767 (a tuning knob with no effect on results:
 * every variant selects the same index set, bit for bit) */
#define FB_TOPK_PATH_AUTO 0    /* by size: split when n * w >= 2^26           */
#define FB_TOPK_PATH_STREAM 1  /* one CTA per client, one pass over D         */
#define FB_TOPK_PATH_SPLIT 2   /* window / segmented pass / select kernels    */

/* Storage of the design matrices for the margins-type passes (margins,
 * gradient, line-search trials; no effect on results): AUTO keeps a compact
 * int8 / float copy when every uploaded value converts to it exactly (e.g.
 * binary LIBSVM features with the labels absorbed), F64 never does. */
#define FB_BSTORE_AUTO 0
#define FB_BSTORE_F64 1

/* Largest dimension of this build (every dataset of the paper and every
 * BASELINE config has d <= 1024; above that the solve runs the
 * global-memory blocked Cholesky, solve_big.cuh). */
#define FB_MAX_D 4096

/* hessian_init (algorithms.py:37) */
#define FB_INIT_LAMBDA_IDENTITY 0
#define FB_INIT_ZERO 1
#define FB_INIT_EXACT 2

/* Mirror of the trajectory-defining RunConfig fields (algorithms.py:60-120)
 * plus the shard shape.  alpha is the RESOLVED step (resolve_alpha,
 * algorithms.py:138-139); ls_steps_table[s] = ls_gamma ** s as the host
 * evaluates it (algorithms.py:305), s = 0..60. */
typedef struct fb_config {
  int32_t d;              /* dimension (features + intercept)          */
  int32_t n_clients;      /* n                                          */
  int32_t n_samples;      /* n_i; the LARGEST shard's with fb_upload_shards_ex */
  int32_t algorithm;      /* FB_ALG_*                                   */
  int32_t kind;           /* FB_KIND_*                                  */
  int32_t k;              /* budget for the sparse kinds, else 0        */
  int32_t topk_weighted;  /* CompressorSpec.topk_weighted               */
  int32_t tau;            /* FedNL-PP participants per round            */
  int32_t hessian_init;   /* FB_INIT_*                                  */
  int32_t option;         /* FB_OPTION_*                                */
  double alpha;
  double lam;             /* RunConfig.lam (master lambda-identity init) */
  double ls_c;
  double ls_gamma;
  uint64_t run_seed;
  double ls_steps_table[61];
  double mu;              /* option a eigenvalue floor (effective_mu)   */
  int32_t topk_path;      /* FB_TOPK_PATH_*                             */
  int32_t b_store;        /* FB_BSTORE_*                                */
} fb_config;

/* Detail of the last failure raised by a round (mirrors the reference's
 * exception payloads). */
typedef struct fb_status {
  int32_t code;           /* FB_ERR_* or 0                               */
  int32_t round;          /* round at which it was raised                */
  int32_t pivot_index;    /* NotPositiveDefiniteError.pivot_index        */
  int32_t client;         /* client whose input was non-finite           */
  double pivot_value;     /* NotPositiveDefiniteError.pivot_value        */
  double f_start;         /* LineSearchError: f at x                      */
  double f_best;          /* LineSearchError: best trial f                */
} fb_status;

/* Per-kernel device time of the most recent fb_run_rounds(..., timed=1),
 * averaged over its rounds (CUDA events on the launching stream). */
typedef struct fb_profile {
  int32_t rounds;
  int32_t launches_per_round;   /* kernels launched per round            */
  double ms_oracle;             /* margins + gradient                    */
  double ms_hessian;            /* DMMA Hessian + shift-difference epilogue */
  double ms_reduce;             /* cross-client reductions                */
  double ms_compress;           /* compressor                             */
  double ms_solve;              /* master Cholesky solve                  */
  double ms_fold;               /* fused shift update + master fold       */
  double ms_round;              /* whole round (graph launch to end)      */
} fb_profile;

/* ---- lifecycle -------------------------------------------------------- */
/* sizeof(fb_config), sizeof(fb_status), sizeof(fb_profile) as this library
 * was compiled (a binding checks its struct mirrors against them; no GPU) */
int fb_abi_sizes(int32_t* out3);
/* Validate cfg, allocate every device buffer, build TMA descriptors.
 * Replaces runtime.simulate's setup (runtime.py:145-155). */
int fb_create(const fb_config* cfg, void** ctx);
void fb_destroy(void* ctx);
const char* fb_last_error(void* ctx);
int fb_get_status(void* ctx, fb_status* out);
int fb_device_info(char* name, int32_t name_len, int32_t* sm_count, int32_t* cc_major,
                   int32_t* cc_minor);

/* ---- multi-GPU: client sharding ------------------------------------------ */
/* Client ranges over `world` GPUs, one process per GPU: rank
 * r owns clients [r*ceil(n/world), (r+1)*ceil(n/world)) ∩ [0, n); each round
 * every rank computes its clients' oracle, Hessian and compressed deltas,
 * all-gathers the per-client gradients / loss / Frobenius partials / flags
 * and the deltas over NCCL (NVLink), and runs the same reduction, master
 * solve and ascending-client fold as one GPU would — so every rank holds the
 * bit-identical master state and trajectory.  NCCL (libnccl.so.2) is loaded
 * on first use.  The reference is single-process (runtime.simulate); this
 * replaces its per-client loop (runtime.py:255-268) across GPUs. */
#define FB_NCCL_ID_BYTES 128
/* a fresh NCCL unique id (rank 0 creates it and shares it out of band) */
int fb_nccl_unique_id(uint8_t* out);
/* before fb_upload_shards; FedNL only.  world == 1 runs the sharded path on
 * one GPU (NCCL with one rank). */
int fb_set_shard(void* ctx, int32_t world, int32_t rank, const uint8_t* nccl_id);

/* ---- data ------------------------------------------------------------- */
/* Copy n shards to HBM (feature-major, sample-contiguous rows; under
 * fb_set_shard only this rank's clients are read).  Host memory is only
 * borrowed for the call.  Replaces ClientShard residency
 * (oracle.py:33-46, data.py:186-213). */
int fb_upload_shards(void* ctx, const double* const* bmats);
/* The same for shards of different sizes and regularisers, as the reference
 * accepts them (runtime.py:145-151 checks only the dimension; each
 * ClientShard carries its own n_samples and lam, oracle.py:33-46):
 * n_samples[c] in [1, cfg.n_samples] columns of shard c (may be NULL: all
 * cfg.n_samples), lam[c] its lambda (may be NULL: all cfg.lam), used by the
 * client's oracle and its lambda-identity H_c^0. */
int fb_upload_shards_ex(void* ctx, const double* const* bmats, const int32_t* n_samples,
                        const double* lam);
/* The copy of the design matrices the margins-type passes read after the
 * last upload (fb_config.b_store): 0 = the fp64 matrices, 1 = float,
 * 2 = int8 (diagnostic; results are identical). */
int fb_bstore_kind(void* ctx);

/* ---- run -------------------------------------------------------------- */
/* Round-0 state: client/master Hessian estimates per hessian_init and, for
 * FedNL-PP, the shift / shifted-gradient state (algorithms.py:195-223,
 * 331-349).  x0 may be NULL (zeros, as runtime.py:224). */
int fb_init_state(void* ctx, const double* x0);

/* Run rounds [first_round, first_round + count) — the body of
 * runtime._simulate_loop (runtime.py:235-271).  Per round r (index
 * i = r - first_round): grad_norm[i], f_value[i], ls_steps[i] as in the
 * MetricsRow; entry_counts[i*n + c] = compressed entry count of client c
 * (-1 when c did not participate, FedNL-PP); wall_ms[i] = device time from
 * the start of the call to the end of round r.  When timed != 0 per-kernel
 * CUDA-event times are collected (fb_get_profile).  Stops early at the first
 * failure (status set, *rounds_done = rounds completed) or when
 * stop_grad_norm >= 0 and a row's grad_norm <= stop_grad_norm: the rule is
 * evaluated on the device inside each round, so no round runs past the
 * stopping row (FedNL / LS: after that round's step, runtime.py:270-272;
 * PP: before it, runtime.py:239-242). */
int fb_run_rounds(void* ctx, int32_t first_round, int32_t count, double stop_grad_norm,
                  int32_t timed, double* grad_norm, double* f_value, int32_t* ls_steps,
                  int32_t* entry_counts, double* wall_ms, int32_t* rounds_done);

/* ||mean grad(x)|| and mean f(x) at the current iterate (the final row,
 * runtime.py:273-275). */
int fb_final_eval(void* ctx, double* grad_norm, double* f_value);

int fb_get_profile(void* ctx, fb_profile* out);

/* ---- state taps (teacher forcing / debugging) ------------------------- */
int fb_get_x(void* ctx, double* x);
int fb_set_x(void* ctx, const double* x);
/* client Hessian estimates H_i^k of clients [c0, c1), packed, row-major */
int fb_get_client_hest(void* ctx, int32_t c0, int32_t c1, double* out);
int fb_set_client_hest(void* ctx, int32_t c0, int32_t c1, const double* in);
int fb_get_master_hest(void* ctx, double* out);
int fb_set_master_hest(void* ctx, const double* in);
/* FedNL-PP running state: master shift / gvec, per-client shift / gvec */
int fb_get_pp_state(void* ctx, double* shift, double* gvec, double* cli_shift, double* cli_gvec);
/* last round's packed difference D_i = H_i(x) - H_i^k of client cid */
int fb_get_round_diff(void* ctx, int32_t cid, double* out);
/* last round's compressed delta of client cid: ascending packed indices,
 * values (already scaled for the Rand kinds), count */
int fb_get_round_delta(void* ctx, int32_t cid, uint32_t* idx, double* val, int32_t* count);
/* last round's scalars {grad_norm, f_mean, shift_mean, decrement, <x,x>} and
 * per-client shifts l_i = ||D_i||_F [n] (may be NULL) */
int fb_get_round_scalars(void* ctx, double* out5, double* client_shift);
/* mean gradient of the last round and per-client gradients [n*d] */
int fb_get_round_grads(void* ctx, double* mean_grad, double* client_grads);

/* ---- leaf operations (parity entry points) ---------------------------- */
/* compress(m, spec, prg) for every client at once (compressors.py:350-370):
 * diffs = [n*w] packed inputs, seeds[c] = the fresh Prg's seed.  Outputs
 * idx/val [n*w] (first count[c] valid per client), count [n], draws [n] =
 * number of u64 draws consumed from each stream.  Returns FB_ERR_NONFINITE
 * (status.client set) on a non-finite input. */
int fb_compress(void* ctx, const double* diffs, const uint64_t* seeds, uint32_t* idx,
                double* val, int32_t* count, int32_t* draws);
/* local f / gradient / packed Hessian of every client at x
 * (oracle.py:74-139); any output may be NULL. */
int fb_oracle_eval(void* ctx, const double* x, double* f, double* grad, double* hess_packed);
/* solve (H + shift I) z = rhs from packed H (algorithms.py:361-367 option b,
 * linalg.py:151-186); FB_ERR_NOT_PD with status.pivot_* on failure. */
int fb_shifted_solve(void* ctx, const double* h_packed, double shift, const double* rhs,
                     double* z);
/* eigen_clamp_min (linalg.py:248-259) of a packed symmetric matrix:
 * out_packed = (V max(L, floor)) V^T; eigvals (d, nullable) and eigvecs
 * (d x d column-major, column k = eigenvector k, nullable) as jacobi_eigh
 * (linalg.py:189-245) returns them; FB_ERR_EIGEN when 30 sweeps do not
 * converge.  Parallel-order Jacobi on the device. */
int fb_eigen_clamp(void* ctx, const double* a_packed, double floor, double* out_packed,
                   double* eigvals, double* eigvecs);

/* diagnostic: per-phase clock64 cycles of one shifted solve on the rank-0
 * CTA.  cluster > 0: the cluster-redundant solver with that cluster size,
 * 12 slots (setup, A, syncA, pull, B, B-writeback, C, syncC, back-solve,
 * back-total, -, -).  cluster == 0: the default solver; for the
 * panel-owning solver cycles must hold 16 + 64 * 16 slots (16 phase slots,
 * then per-panel globaltimer stamps).  ms = event time of an uninstrumented
 * run of the same solve. */
int fb_solve_phase_cycles(void* ctx, const double* h_packed, double shift, const double* rhs,
                          int32_t cluster, long long* cycles, float* ms);

/* diagnostic: read (and zero) the device phase-clock counters: out[0..32)
 * accumulated from thread 0 of block 0 of instrumented kernels, out[32..1056)
 * per-CTA durations of the last instrumented compressor launch; `enable`
 * arms the next run */
int fb_debug_counters(int32_t enable, long long* out);
/* diagnostic: out[2 s], out[2 s + 1] = first-CTA start / last-CTA end
 * globaltimer ns of instrumented kernel slot s (16 slots) since the last
 * call (which re-arms them); slots: 0 margins, 1 Hessian, 2 solve, 3 solve's
 * wait for its producer, 4 TopK, 5 master fold, 6 round epilogue */
int fb_debug_timeline(unsigned long long* out);

/* ---- context-free device SplitMix64 (rng.py:37-136) -------------------- */
int fb_prg_u64(uint64_t seed, int32_t count, uint64_t* out);
/* reps draws of randrange(bounds[b]) from a fresh Prg(seed) per bound;
 * out[b*reps + r]; next[b] = the following next_u64() */
int fb_prg_randrange(uint64_t seed, const uint64_t* bounds, int32_t n_bounds, int32_t reps,
                     uint64_t* out, uint64_t* next);
int fb_prg_partial_shuffle(uint64_t seed, int64_t n, int32_t k, int64_t* out);
int fb_round_seeds(uint64_t run_seed, int32_t n_clients, int32_t rnd, uint64_t* out);

/* ---- measurement ------------------------------------------------------ */
/* fp64 peak of this device: register-resident DMMA (mma.sync f64) and DFMA
 * loops, TFLOP/s. */
int fb_fp64_peak(double* dmma_tflops, double* dfma_tflops);

#ifdef __cplusplus
}
#endif
#endif /* FEDNL_B200_H */
