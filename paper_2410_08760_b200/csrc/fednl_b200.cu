// fednl_b200.cu — libfednl_b200.so: context, round graphs and the C ABI
// declared in include/fednl_b200.h.
//
// One context = one simulated FedNL run on one GPU: all client shards, the
// per-client Hessian estimates, the master state and the per-round scratch
// live in HBM; each round is a captured CUDA graph replayed back to back
// (the round index lives in device memory), so the host issues one graph
// launch per round and reads the metrics rows once per chunk.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is dlopen'ed on first use

#include <algorithm>
#include <atomic>
#include <cmath>
#include <map>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <functional>
#include <vector>
#include <type_traits>

#include "../../include/fednl_b200.h"
#include "common.cuh"
#include "compress_kernels.cuh"
#include "eig_kernels.cuh"
#include "fp64_peak.cuh"
#include "hessian_dmma.cuh"
#include "oracle_kernels.cuh"
#include "round_kernels.cuh"
#include "solve_kernels.cuh"
#include "solve_big.cuh"

using namespace fb;

namespace {

constexpr int ROW_CHUNK = 256;  // rounds per graph-replay chunk

enum EvSlot {
  EV_START = 0,
  EV_ORACLE_END,
  EV_HESS_END,
  EV_REDUCE_END,
  EV_COMP_START,
  EV_COMP_END,
  EV_SOLVE_END,
  EV_FOLD_START,
  EV_FOLD_END,
  EV_END,
  EV_COUNT
};

struct Ctx {
  fb_config cfg{};
  int d = 0, n = 0, ni = 0, ldj = 0, ldh = 0, nblk = 0, ls_nblk = 0, nb_tiles = 0, n_pairs = 0,
      wb = 0;
  int cap = 0, tau = 0, n_active_max = 0;
  int64_t w = 0;
  double alpha_n = 0.0, rand_scale = 1.0;
  int solve_cs = 1, solve_nb = 32;
  bool solve_panels = false;  // k_chol_panels (d <= CP_MAX_D) instead of k_chol_solve
  bool solve_big = false;     // d > CP_MAX_D: the global-memory blocked solve (solve_big.cuh)
  int cp_kp = 1, cp_cs = 1;
  bool topk_stream = false;  // one-pass sampled-window TopK (else the shared-memory radix)
  bool topk_split = false;   // ... as window / segmented pass / select kernels
  int tks_S = 1, tks_lseg = 0, tks_capseg = 0, tks_ns = 2048;
  bool phase_events = false;   // per-kernel event records while capturing (timed runs)
  bool gexec_phase = false;    // the flavour the cached round graph was built with
  int num_sms = 148;
  int32_t* pair_order = nullptr;  // Hessian tile pairs, costliest first
  double* Lg = nullptr;       // k_chol_panels: released L panels
  double* Lbig = nullptr;     // solve_big: the factor below the diagonal blocks ((d+1) x (d+1))
  double* Tbig = nullptr;     // solve_big: inverse diagonal blocks, [panels][32][32]
  double* pp_shift_part = nullptr;  // FedNL-PP: Frobenius partials [tau][PP_SB]
  // client sharding over `world` GPUs (fb_set_shard): this rank owns clients
  // [c_lo, c_hi) of blocks of npr; per-client exchange arrays are padded to
  // world * npr clients so an in-place ncclAllGather fills them
  int world = 1, rank = 0, npr = 0, c_lo = 0, c_hi = 0;
  int32_t* local_clients = nullptr;  // device [c_hi - c_lo] = c_lo, c_lo + 1, ...
  int32_t* xcode = nullptr;          // [world] status codes exchanged after rank-local work
  // FedNL-PP across ranks: participant slots [s_lo, s_hi) of spr per rank
  int spr = 0, s_lo = 0, s_hi = 0;
  int32_t* sub_loc = nullptr;        // this rank's participants
  PpX ppx{};
  double *dgvec_all = nullptr, *dshift_all = nullptr;  // [tau][d], [tau]
  ncclComm_t comm = nullptr;
  int prio_high = 0;
  size_t solve_smem = 0;
  int toplek_P = 0;
  int32_t* npw_tab = nullptr;  // TopLEK: numpy pairwise-sum recursion for n = w
  TlbScratch tlb{};            // TopLEK for w > TLB_MAXW_SMEM: global sort / sum scratch
  int32_t* rk_js = nullptr;    // RandK draws [n][k] when they do not fit shared memory
  int32_t* rk_pool = nullptr;  // RandK pools [n][w] when w > RK_DIRECT_W and k > RK_HASH_MAXK
  bool uploaded = false, initialised = false;
  std::string err;

  cudaStream_t st = nullptr, st2 = nullptr;
  cudaStream_t st_body = nullptr;  // captures the line search's while-loop body
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_solve_launched = nullptr;

  DevCtl* ctl = nullptr;
  int32_t* hess_sched = nullptr;  // k_hessian_ws item tickets (zero between launches)
  int32_t* ni_arr = nullptr;  // [n] samples per client (ragged shards; <= cfg.n_samples)
  double* lam_arr = nullptr;  // [n] lambda per client (ClientShard.lam)
  double *Bt = nullptr, *x = nullptr, *x_new = nullptr, *pvec = nullptr, *zbuf = nullptr;
  // compact copy of Bt for the margins-type passes (oracle_kernels.cuh BPair):
  // bkind 0 = none (fp64 Bt), 1 = float, 2 = int8; chosen after each upload
  void* Bc = nullptr;
  int bkind = 0;
  double *hcoef = nullptr, *gcoef = nullptr, *loss_part = nullptr, *grad = nullptr;
  double *gbar = nullptr, *f_cli = nullptr, *shift_cli = nullptr, *frob_part = nullptr;
  int32_t* flags = nullptr;
  double *hest = nullptr, *D = nullptr, *hmas = nullptr, *hmas2 = nullptr, *M = nullptr,
         *zeros_w = nullptr;
  double *eigA = nullptr, *eigV = nullptr, *hclamp = nullptr;  // option a
  int32_t* rs = nullptr;  // per-client range starts of the compressed lists
  int nr = 0;
  uint32_t* bitmap = nullptr;
  int32_t *count = nullptr, *draws = nullptr;
  uint32_t* idx_list = nullptr;
  double* val_list = nullptr;
  uint64_t* cand_key = nullptr;  // TopK streaming path: threshold-bin candidates
  int32_t* cand_pos = nullptr;
  TkWin* tks_win = nullptr;      // split TopK: per-client key window
  TkSeg* tks_seg = nullptr;      // split TopK: per-(client, segment) counts
  uint64_t* gt_val = nullptr;    // split TopK: entries above the window (raw values)
  int32_t* gt_pos = nullptr;
  int32_t* tks_ticket = nullptr;  // split TopK: finished segment CTAs per client
  uint32_t* tks_eqz = nullptr;   // split TopK: zero / tie bit rows (all-zero between rounds)
  uint64_t* seeds = nullptr;
  RoundScalars* sc = nullptr;
  double *steps_table = nullptr, *trial_x = nullptr, *ls_loss_part = nullptr;
  int32_t *subset = nullptr, *pool = nullptr;
  double *hess_part = nullptr, *cli_shift = nullptr, *cli_gvec = nullptr, *gvec = nullptr;
  double *pp_shift = nullptr, *dshift = nullptr, *dgvec = nullptr, *scalar = nullptr;
  double *row_grad = nullptr, *row_f = nullptr;
  int32_t *row_counts = nullptr, *row_ls = nullptr;

  CUtensorMap tmap{};

  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  // production flavour only: GRAPH_ROUNDS rounds captured back to back (no
  // graph boundary between them)
  cudaGraph_t graph_multi = nullptr;
  cudaGraphExec_t gexec_multi = nullptr;
  cudaEvent_t ev_fixed[EV_COUNT] = {};
  cudaGraphNode_t ev_node[EV_COUNT] = {};
  bool ev_used[EV_COUNT] = {};
  std::vector<cudaEvent_t> ev_pool;  // [ROW_CHUNK][EV_COUNT]
  fb_profile prof{};
  int launches_per_round = 0;

  std::vector<std::pair<void*, size_t>> allocs;
  std::vector<cudaEvent_t> ev_ends;  // per-round end events of a run chunk
};

thread_local std::string g_err;

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      char b_[2048];                                                                \
      snprintf(b_, sizeof b_, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
               __FILE__, __LINE__);                                                \
      ctx->err = b_;                                                               \
      return FB_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

#define CKL()                                                                      \
  do {                                                                             \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess) {                                                       \
      char b_[2048];                                                                \
      snprintf(b_, sizeof b_, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
               __FILE__, __LINE__);                                                \
      ctx->err = b_;                                                               \
      return FB_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

// Process-wide cache of device buffers: contexts of the same shape (one per
// simulate() call) reuse their predecessor's allocations instead of paying
// cudaMalloc / cudaFree every call (the caching-allocator pattern).
struct DevCache {
  std::mutex mu;
  std::multimap<size_t, void*> free;
  size_t bytes = 0;
};
DevCache& dev_cache() {
  static DevCache* c = new DevCache;  // process lifetime
  return *c;
}
constexpr size_t DEV_CACHE_LIMIT = size_t(32) << 30;
size_t cache_round(size_t bytes) { return (bytes + 4095) & ~size_t(4095); }
cudaError_t cache_alloc(void** p, size_t bytes) {
  DevCache& c = dev_cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.free.find(bytes);
    if (it != c.free.end()) {
      *p = it->second;
      c.free.erase(it);
      c.bytes -= bytes;
      return cudaSuccess;
    }
  }
  return cudaMalloc(p, bytes);
}
void cache_release(void* p, size_t bytes) {
  DevCache& c = dev_cache();
  std::lock_guard<std::mutex> g(c.mu);
  if (c.bytes + bytes > DEV_CACHE_LIMIT) {
    cudaFree(p);
    return;
  }
  c.free.emplace(bytes, p);
  c.bytes += bytes;
}

// zero-filled device buffer owned by ctx (zeroing is queued on ctx->st;
// fb_create synchronises before returning)
template <typename T>
int dalloc(Ctx* ctx, T** p, size_t count) {
  if (count == 0) count = 1;
  const size_t bytes = cache_round(count * sizeof(T));
  void* q = nullptr;
  CK(cache_alloc(&q, bytes));
  ctx->allocs.emplace_back(q, bytes);
  CK(cudaMemsetAsync(q, 0, bytes, ctx->st));
  *p = static_cast<T*>(q);
  return FB_OK;
}

#define TRY(expr)              \
  do {                         \
    int r_ = (expr);           \
    if (r_ != FB_OK) return r_; \
  } while (0)

int invalid(Ctx* ctx, const char* msg) {
  if (ctx) ctx->err = msg;
  else g_err = msg;
  return FB_ERR_INVALID;
}
int fail_code(Ctx* ctx, int code, const char* msg) {
  if (ctx) ctx->err = msg;
  else g_err = msg;
  return code;
}

// ---------------------------------------------------------------- TMA map
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_tmap(Ctx* ctx) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !fn) {
    ctx->err = "cuTensorMapEncodeTiled entry point not found";
    return FB_ERR_CUDA;
  }
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(ctx->ni), static_cast<cuuint64_t>(ctx->d),
                              static_cast<cuuint64_t>(ctx->n)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ctx->ldj) * 8,
                                 static_cast<cuuint64_t>(ctx->ldj) * ctx->d * 8};
  const cuuint32_t box[3] = {HKC, HT, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(
      &ctx->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ctx->Bt, dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    ctx->err = "cuTensorMapEncodeTiled failed (code " + std::to_string(static_cast<int>(r)) + ")";
    return FB_ERR_CUDA;
  }
  return FB_OK;
}

// -------------------------------------------------------------- launchers
// ------------------------------------------------------------------ NCCL
// Loaded with dlopen the first time sharding is requested, so single-GPU use
// has no NCCL dependency (and an already loaded libnccl — e.g. torch's — is
// reused: same soname).
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl_api() {
  static NcclApi api;
  if (!api.tried) {
    api.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllGather && api.CommDestroy && api.GetErrorString;
    }
  }
  return api;
}
#define NCK(call)                                                                    \
  do {                                                                               \
    ncclResult_t r_ = (call);                                                        \
    if (r_ != ncclSuccess) {                                                         \
      ctx->err = std::string(#call) + ": " + nccl_api().GetErrorString(r_);          \
      return FB_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

// in-place all-gather of a per-client array: this rank's block of npr
// clients (`per` elements each) at element offset rank * npr * per
template <typename T>
int gather_clients(Ctx* ctx, T* base, size_t per, ncclDataType_t type, cudaStream_t s) {
  const size_t cnt = static_cast<size_t>(ctx->npr) * per;
  NCK(nccl_api().AllGather(base + static_cast<size_t>(ctx->rank) * cnt, base, cnt, type, ctx->comm, s));
  return FB_OK;
}
// in-place all-gather of per-rank blocks of `cnt` elements (rank r's at r * cnt)
template <typename T>
int gather_blocks(Ctx* ctx, T* base, size_t cnt, ncclDataType_t type, cudaStream_t s) {
  NCK(nccl_api().AllGather(base + static_cast<size_t>(ctx->rank) * cnt, base, cnt, type, ctx->comm, s));
  return FB_OK;
}
bool sharded(const Ctx* ctx) { return ctx->world > 1 || ctx->comm != nullptr; }

// clients per Hessian item group.  Items run group by group, each group's
// tile pairs costliest first: the group's B rows stay in L2 for all its tiles
// (round 1, one tile per CTA at c0: one group 586 MB of DRAM traffic, groups
// of 48 clients 218 MB) and the last items of the pass are cheap diagonal /
// edge tiles.  Base size: about 2.5 rounds of the 2 * num_sms tile pipes
// (3.75 for small clients, B_c <= 4 MB: their rows are loaded evict-first);
// the groups are then made equal, so the last one — the pass's tail — has as
// many items to balance with as the others (c0, n = 142: 49 + 49 + 44 ->
// 71 + 71, Hessian 190.2 -> 187.8 us; 57 / 64 / 80 / 95 are all worse).
int hess_group(const Ctx* ctx, int n_active) {
  const bool small = static_cast<size_t>(ctx->d) * ctx->ldj * sizeof(double) <= (size_t{4} << 20);
  const int base = std::max(1, (small ? 15 : 10) * ctx->num_sms / (2 * std::max(1, ctx->n_pairs)));
  const int groups = std::max(1, (n_active + base - 1) / base);
  return std::max(1, (n_active + groups - 1) / groups);
}
// programmatic dependent launch attributes, except under a profiler's
// injection library (serialised launches there anyway)
bool under_profiler() {
  static const bool injected = getenv("CUDA_INJECTION64_PATH") != nullptr ||
                               getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr ||
                               getenv("NV_TPS_LAUNCH_TOKEN") != nullptr;
  return injected;
}
bool pdl_ok(const Ctx*) { return !under_profiler(); }
void drop_graphs(Ctx* ctx);

// bit 0: every value is an integer in [-128, 127] (int8; -0.0 maps to 0,
// see BPair); bit 1: double -> float -> double bit for bit (cleared by any
// value that does not)
__global__ void k_b_exact(const double* __restrict__ Bt, int64_t count, int32_t* __restrict__ flags) {
  int ok = 3;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = __ldcs(Bt + i);
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v));
    const bool i8 = v >= -128.0 && v <= 127.0 && v == rint(v);
    const bool f32 = static_cast<uint64_t>(__double_as_longlong(static_cast<double>(__double2float_rn(v)))) == bits;
    ok &= (i8 ? 1 : 0) | (f32 ? 2 : 0);
  }
  ok = __reduce_and_sync(0xffffffffu, ok);
  if ((threadIdx.x & 31) == 0 && ok != 3) atomicAnd(flags, ok);
}
template <class T>
__global__ void k_b_convert(const double* __restrict__ Bt, int64_t count, T* __restrict__ Bc) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    Bc[i] = static_cast<T>(__ldcs(Bt + i));  // exact (k_b_exact)
}
// picks the compact copy after an upload (fb_config.b_store = AUTO); the
// round graph is rebuilt when the choice changes
int choose_bstore(Ctx* ctx) {
  const int64_t count = static_cast<int64_t>(ctx->n) * ctx->d * ctx->ldj;
  int kind = 0;
  if (ctx->cfg.b_store == FB_BSTORE_AUTO) {
    int32_t* flags = nullptr;
    CK(cudaMalloc(&flags, sizeof(int32_t)));
    const int32_t init = 3;
    CK(cudaMemcpyAsync(flags, &init, sizeof init, cudaMemcpyHostToDevice, ctx->st));
    k_b_exact<<<4 * ctx->num_sms, 256, 0, ctx->st>>>(ctx->Bt, count, flags);
    int32_t got = 0;
    CK(cudaMemcpyAsync(&got, flags, sizeof got, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    cudaFree(flags);
    kind = (got & 1) ? 2 : (got & 2) ? 1 : 0;
  }
  if (kind != ctx->bkind) {
    if (ctx->Bc) {
      for (auto it = ctx->allocs.begin(); it != ctx->allocs.end(); ++it)
        if (it->first == ctx->Bc) {
          cache_release(it->first, it->second);
          ctx->allocs.erase(it);
          break;
        }
      ctx->Bc = nullptr;
    }
    if (kind == 1) {
      float* b = nullptr;
      TRY(dalloc(ctx, &b, static_cast<size_t>(count)));
      ctx->Bc = b;
    } else if (kind == 2) {
      int8_t* b = nullptr;
      TRY(dalloc(ctx, &b, static_cast<size_t>(count)));
      ctx->Bc = b;
    }
    ctx->bkind = kind;
    drop_graphs(ctx);
  }
  if (kind == 1)
    k_b_convert<<<4 * ctx->num_sms, 256, 0, ctx->st>>>(ctx->Bt, count, static_cast<float*>(ctx->Bc));
  else if (kind == 2)
    k_b_convert<<<4 * ctx->num_sms, 256, 0, ctx->st>>>(ctx->Bt, count, static_cast<int8_t*>(ctx->Bc));
  CKL();
  CK(cudaStreamSynchronize(ctx->st));
  return FB_OK;
}
// f(B) with B the margins-type passes' copy of Bt (typed)
template <class F>
void with_b(const Ctx* ctx, F f) {
  if (ctx->bkind == 2) f(static_cast<const int8_t*>(ctx->Bc));
  else if (ctx->bkind == 1) f(static_cast<const float*>(ctx->Bc));
  else f(static_cast<const double*>(ctx->Bt));
}

int launch_margins(Ctx* ctx, cudaStream_t s, const double* x, const int32_t* clients, int n_active,
                   bool with_ctl = true, int32_t* zero_flags = nullptr) {
  if (n_active >= ctx->num_sms * 3 / 4 && mc_smem_bytes(ctx->d, ctx->ldj) <= MC_SMEM_MAX) {
    // enough clients to fill the GPU: one CTA streams each client's rows
    // two 512-thread CTAs per client (each half of its samples, two CTAs per
    // SM) when that halves the row batches a thread streams; else one
    with_b(ctx, [&](auto B) {
      using T = std::remove_cv_t<std::remove_pointer_t<decltype(B)>>;
      if (ctx->ldj / 2 > 64) {
        k_margins_cpc<512, 2, T><<<2 * n_active, 512, mc_smem_bytes_nt(ctx->d, ctx->ldj, 2, 512), s>>>(
            with_ctl ? ctx->ctl : nullptr, B, ctx->d, ctx->ni_arr, ctx->ldj, ctx->ldh, x, clients,
            ctx->hcoef, ctx->gcoef, ctx->loss_part, ctx->nblk, zero_flags);
      } else {
        k_margins_cpc<MC_THREADS, 1, T><<<n_active, MC_THREADS, mc_smem_bytes(ctx->d, ctx->ldj), s>>>(
            with_ctl ? ctx->ctl : nullptr, B, ctx->d, ctx->ni_arr, ctx->ldj, ctx->ldh, x, clients,
            ctx->hcoef, ctx->gcoef, ctx->loss_part, ctx->nblk, zero_flags);
      }
    });
  } else {
    dim3 grid(ctx->nblk, n_active);
    with_b(ctx, [&](auto B) {
      using T = std::remove_cv_t<std::remove_pointer_t<decltype(B)>>;
      k_margins<T><<<grid, MB_THREADS, ctx->d * sizeof(double), s>>>(
          with_ctl ? ctx->ctl : nullptr, B, ctx->d, ctx->ni_arr, ctx->ldj, ctx->ldh, x, clients,
          ctx->hcoef, ctx->gcoef, ctx->loss_part, ctx->nblk, zero_flags);
    });
  }
  CKL();
  return FB_OK;
}
int launch_gradient(Ctx* ctx, cudaStream_t s, const double* x, const int32_t* clients,
                    int n_active, bool with_ctl = true) {
  dim3 grid((ctx->d + 7) / 8, n_active);
  with_b(ctx, [&](auto B) {
    using T = std::remove_cv_t<std::remove_pointer_t<decltype(B)>>;
    k_gradient<T><<<grid, 256, 0, s>>>(with_ctl ? ctx->ctl : nullptr, B, ctx->d, ctx->ni_arr,
                                       ctx->ldj, ctx->ldh, x, ctx->lam_arr, clients, ctx->gcoef,
                                       ctx->grad);
  });
  CKL();
  return FB_OK;
}
// fuse_grad: the diagonal-tile CTAs also compute the local gradients at x
// (ctx->grad), replacing k_gradient in the FedNL round
// B's TMA tiles are marked L2 evict-first when a client's rows are small
// (c0: 0.8 MB, re-read by its tile pairs within microseconds): the round's
// streamed bytes then no longer push the latency-bound solve's code and state
// out of L2.  A large client (c4: 16.8 MB) is re-read over milliseconds and
// keeps the normal policy (evict-first there tripled its DRAM traffic).
bool hess_b_evict_first(const Ctx* ctx) {
  return static_cast<size_t>(ctx->d) * ctx->ldj * sizeof(double) <= (size_t{4} << 20);
}
int launch_hessian(Ctx* ctx, cudaStream_t s, const int32_t* clients, int n_active,
                   const double* hest, int64_t hest_stride, double* D, double* hess_out,
                   bool with_ctl = true, const double* fuse_grad_x = nullptr) {
  // persistent warp-specialised DMMA pass: one CTA (two tile pipes) per SM
  // over the (client, tile pair) items; programmatic dependent launch after
  // the margins kernel (the TMA producers wait for it)
  cudaLaunchConfig_t lc{};
  const int items = n_active * ctx->n_pairs;
  lc.gridDim = dim3(std::min((items + HW_PIPES - 1) / HW_PIPES, ctx->num_sms));
  // about two tiles per pipe or fewer: no later tile to hide an epilogue
  // behind, so each pipe's five warps finish every tile together
  const int solo = items <= 2 * HW_PIPES * static_cast<int>(lc.gridDim.x) ? 1 : 0;
  lc.blockDim = dim3(HW_THREADS);
  lc.dynamicSmemBytes = HESS_WS_SMEM;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = pdl_ok(ctx) ? 1 : 0;
  CK(cudaLaunchKernelEx(&lc, solo ? k_hessian_ws<true> : k_hessian_ws<false>, ctx->tmap, static_cast<const DevCtl*>(with_ctl ? ctx->ctl : nullptr),
                        ctx->d, static_cast<const int32_t*>(ctx->ni_arr), ctx->ldh,
                        static_cast<const double*>(ctx->hcoef), static_cast<const double*>(ctx->lam_arr), clients,
                        hest, hest_stride, D, hess_out, ctx->frob_part, ctx->flags,
                        0u /* zero_mask: see mbar_arrive_dep */, static_cast<const double*>(ctx->gcoef),
                        fuse_grad_x, fuse_grad_x ? ctx->grad : nullptr,
                        static_cast<const int32_t*>(ctx->pair_order), ctx->n_pairs, n_active, hess_group(ctx, n_active),
                        ctx->hess_sched, hess_b_evict_first(ctx) ? 1 : 0));
  return FB_OK;
}
int launch_reduce(Ctx* ctx, cudaStream_t s, const double* x, const int32_t* clients, int n_active,
                  int n_div, bool with_frob, double* row_grad, double* row_f,
                  const double* l2_prefetch = nullptr) {
  // programmatic dependent launch after the Hessian pass (k_reduce waits for
  // it after warming L2 with the solve's input)
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(reduce_grid(ctx->d));
  lc.blockDim = dim3(RED_THREADS);
  lc.dynamicSmemBytes = 0;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = pdl_ok(ctx) ? 1 : 0;
  CK(cudaLaunchKernelEx(&lc, k_reduce, ctx->ctl, n_active, clients, n_div, ctx->d,
                        static_cast<const int32_t*>(ctx->ni_arr), ctx->nblk, ctx->n_pairs, x,
                        static_cast<const double*>(ctx->lam_arr), static_cast<const double*>(ctx->grad),
                        static_cast<const double*>(ctx->loss_part),
                        static_cast<const double*>(with_frob ? ctx->frob_part : nullptr),
                        static_cast<const int32_t*>(ctx->flags), ctx->gbar, ctx->f_cli, ctx->shift_cli, ctx->sc,
                        row_grad, row_f, l2_prefetch, static_cast<int64_t>(ctx->w) * 8));
  return FB_OK;
}
// compressor of the configured kind over `n_active` clients; seeds null =
// per-(client, round) streams from the device round counter.
int launch_compress(Ctx* ctx, cudaStream_t s, const int32_t* clients, int n_active,
                    const uint64_t* seeds, double* dense_out, bool with_ctl = true,
                    bool emit = true, bool client_update_in_fold = false) {
  const fb_config& c = ctx->cfg;
  DevCtl* ctl = with_ctl ? ctx->ctl : nullptr;
  Emit em{};
  if (emit) {
    em.hest = ctx->hest;
    em.hest_stride = ctx->w;
    em.alpha = c.alpha;
    em.rs = ctx->rs;
    em.nr = ctx->nr;
  }
  switch (c.kind) {
    case FB_KIND_TOPK:
      if (ctx->w <= TKS_MAXW && !ctx->topk_stream)
        k_topk_smem<<<n_active, TK_THREADS, tks_smem_bytes(ctx->w), s>>>(
            ctl, ctx->D, ctx->w, ctx->wb, c.k, c.topk_weighted, clients, ctx->flags, ctx->bitmap,
            ctx->count, ctx->idx_list, ctx->val_list, ctx->cap, ctx->draws, em);
      else if (ctx->topk_split) {
        Emit es = em;
        if (client_update_in_fold) es.hest = nullptr;
        k_tks_window<<<n_active, TKW_THREADS, 0, s>>>(ctl, ctx->D, ctx->w, c.k, ctx->tks_ns,
                                                      c.topk_weighted, clients, ctx->flags,
                                                      ctx->draws, ctx->tks_win, ctx->tks_ticket,
                                                      ctx->count, es);
        CKL();
        const int capw = ctx->tks_capseg / TKP_CW;
        auto pass = c.topk_weighted ? k_tks_pass<true> : k_tks_pass<false>;
        pass<<<dim3(ctx->tks_S, n_active), TKP_THREADS, tkp_smem_bytes(ctx->w), s>>>(
            ctl, ctx->D, ctx->w, tks_wbp(ctx->w), ctx->tks_lseg, capw, clients, ctx->tks_win,
            ctx->tks_eqz, ctx->cand_key, ctx->cand_pos, ctx->gt_val, ctx->gt_pos, ctx->tks_seg,
            ctx->tks_ticket, c.k, ctx->count, ctx->idx_list, ctx->val_list, ctx->cap, es);
      } else if (ctx->w <= TKST_MAXW)
        k_topk_stream<<<n_active, TK_THREADS, tkst_smem_bytes(ctx->w), s>>>(
            ctl, ctx->D, ctx->w, ctx->wb, c.k, c.topk_weighted, clients, ctx->flags, ctx->bitmap,
            ctx->count, ctx->idx_list, ctx->val_list, ctx->cap, ctx->draws, ctx->cand_key,
            ctx->cand_pos, em);
      else
        k_topk<<<n_active, TK_THREADS, 0, s>>>(ctl, ctx->D, ctx->w, ctx->wb, c.k, c.topk_weighted,
                                               clients, ctx->flags, ctx->bitmap, ctx->count,
                                               ctx->idx_list, ctx->val_list, ctx->cap, ctx->draws,
                                               em);
      break;
    case FB_KIND_RANDSEQK:
      k_randseqk<<<n_active, 256, 0, s>>>(ctl, ctx->D, ctx->w, ctx->wb, c.k, clients, ctx->flags,
                                          c.run_seed, seeds, ctx->bitmap, ctx->count,
                                          ctx->idx_list, ctx->val_list, ctx->cap, ctx->draws, em);
      break;
    case FB_KIND_RANDK:
      k_randk<<<n_active, RK_THREADS, rk_smem_bytes(c.k, ctx->wb, ctx->w), s>>>(
          ctl, ctx->D, ctx->w, ctx->wb, c.k, clients, ctx->flags, c.run_seed, seeds, ctx->bitmap,
          ctx->count, ctx->idx_list, ctx->val_list, ctx->cap, ctx->draws, em, ctx->rk_js, ctx->rk_pool);
      break;
    case FB_KIND_TOPLEK:
      if (ctx->w > TLB_MAXW_SMEM) {
        k_toplek_big<<<n_active, TLB_THREADS, 0, s>>>(
            ctl ? ctl : ctx->ctl, ctx->D, ctx->w, ctx->wb, c.k, clients, ctx->flags, c.run_seed,
            seeds, ctx->bitmap, ctx->count, ctx->idx_list, ctx->val_list, ctx->cap, ctx->draws, em,
            ctx->npw_tab, ctx->tlb);
        break;
      }
      k_toplek<<<n_active, TK_THREADS, toplek_smem_bytes(ctx->toplek_P), s>>>(
          ctl ? ctl : ctx->ctl, ctx->D, ctx->w, ctx->wb, c.k, clients, ctx->flags, c.run_seed,
          seeds, ctx->bitmap, ctx->count, ctx->idx_list, ctx->val_list, ctx->cap, ctx->draws,
          ctx->toplek_P, em, ctx->npw_tab);
      break;
    case FB_KIND_IDENTITY:
    case FB_KIND_NATURAL: {
      dim3 grid(static_cast<unsigned>((ctx->w + 255) / 256), n_active);
      k_dense_kind<<<grid, 256, 0, s>>>(ctl, ctx->D, dense_out ? dense_out : ctx->D, ctx->w,
                                        c.kind == FB_KIND_NATURAL, clients, ctx->flags,
                                        c.run_seed, seeds, ctx->count, ctx->draws);
      break;
    }
    default:
      return invalid(ctx, "unknown compressor kind");
  }
  CKL();
  return FB_OK;
}
int launch_solve(Ctx* ctx, cudaStream_t s, const double* hpk, const double* shift_ptr,
                 const double* rhs, const double* x, double* z, double* x_out, int mode,
                 int ignore_halt, long long* dbg = nullptr, cudaEvent_t launched = nullptr,
                 bool force_old = false, bool after_reduce = false, const CpRed* red = nullptr) {
  if (ctx->solve_big && !(force_old && ctx->d <= CH_MAX_D)) {
    // d > CP_MAX_D: setup, then one kernel per 32-column panel (block factor,
    // panel rows and the trailing update of one tile per CTA), then the back
    // substitution (solve_big.cuh)
    const int d = ctx->d;
    // high priority, as the cluster solvers: the panel kernels' CTAs take
    // the SM slots the concurrent compressor's CTAs free, ahead of its own
    // pending ones (at default priority the solve only ran after the c4
    // TopK pass had dispatched its last CTA)
    cudaLaunchAttribute pattr[2];
    pattr[0].id = cudaLaunchAttributePriority;
    pattr[0].val.priority = ctx->prio_high;
    // the panel kernels and the back substitution chain with programmatic
    // dependent launch (each waits for its predecessor after its prologue)
    pattr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pattr[1].val.programmaticStreamSerializationAllowed = 1;
    const bool pdl = pdl_ok(ctx);
    auto cfg = [&](int grid, int block, size_t smem, bool dep = false) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(grid);
      lc.blockDim = dim3(block);
      lc.dynamicSmemBytes = smem;
      lc.stream = s;
      lc.attrs = pattr;
      lc.numAttrs = (dep && pdl) ? 2 : 1;
      return lc;
    };
    {
      cudaLaunchConfig_t lc = cfg(std::min(d + 1, 4 * ctx->num_sms), BIG_THREADS, 0);
      CK(cudaLaunchKernelEx(&lc, k_big_setup, static_cast<const DevCtl*>(ctx->ctl), d, hpk, shift_ptr, rhs,
                            ctx->M));
    }
    if (launched) CK(cudaEventRecord(launched, s));
    for (int p0 = 0; p0 < d; p0 += BIG_NB) {
      const int p1 = std::min(d, p0 + BIG_NB);
      const int T = (d + 1 - p1 + BIG_TILE - 1) / BIG_TILE;  // tiles of rows p1..d (the rhs row included)
      cudaLaunchConfig_t lc = cfg(T * (T + 1) / 2, BIG_THREADS, sizeof(BigSmem), p0 > 0);
      CK(cudaLaunchKernelEx(&lc, k_big_panel, ctx->ctl, d, p0, ctx->M, ctx->Lbig, ctx->Tbig));
    }
    {
      cudaLaunchConfig_t lc = cfg(1, BIG_BACK_THREADS, big_back_smem(d), true);
      CK(cudaLaunchKernelEx(&lc, k_big_back, ctx->ctl, d, static_cast<const double*>(ctx->Lbig),
                            static_cast<const double*>(ctx->Tbig), x, z, x_out, mode, ignore_halt));
    }
    return FB_OK;
  }
  const bool panels = ctx->solve_panels && !force_old;
  const int cs = panels ? ctx->cp_cs : ctx->solve_cs;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(cs);
  lc.blockDim = dim3(CH_THREADS);
  lc.dynamicSmemBytes = panels ? static_cast<size_t>(ctx->cp_kp) * cp_panel_bytes(ctx->d) + CP_STAMP_BYTES
                               : ctx->solve_smem;
  lc.stream = s;
  cudaLaunchAttribute attr[4];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // the solve is the round's critical path and needs cs SMs at once:
  // schedule its cluster ahead of the concurrent compressor's CTAs
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = ctx->prio_high;
  lc.attrs = attr;
  lc.numAttrs = 2;
  if (launched) {
    // fires once every CTA of the cluster is resident: the concurrent
    // compressor is held back until then, so the solve never waits for SMs
    attr[lc.numAttrs].id = cudaLaunchAttributeLaunchCompletionEvent;
    attr[lc.numAttrs].val.launchCompletionEvent.event = launched;
    attr[lc.numAttrs].val.launchCompletionEvent.flags = 0;
    ++lc.numAttrs;
  }
  CpRed rd{};
  if (red && panels) rd = *red;
  if (after_reduce && panels) {
    // programmatic dependent launch: the panel setup overlaps k_reduce
    attr[lc.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[lc.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++lc.numAttrs;
  }
  if (panels) {
    if (ctx->cp_kp == 1)
      CK(cudaLaunchKernelEx(&lc, k_chol_panels<1>, ctx->ctl, ctx->d, hpk, shift_ptr, rhs, x, ctx->Lg,
                            z, x_out, mode, ignore_halt, dbg, rd));
    else
      CK(cudaLaunchKernelEx(&lc, k_chol_panels<2>, ctx->ctl, ctx->d, hpk, shift_ptr, rhs, x, ctx->Lg,
                            z, x_out, mode, ignore_halt, dbg, rd));
  } else if (ctx->solve_nb == 32) {
    CK(cudaLaunchKernelEx(&lc, k_chol_solve<32>, ctx->ctl, ctx->d, hpk, shift_ptr, rhs, x, ctx->M,
                          z, x_out, mode, ignore_halt, dbg));
  } else {
    CK(cudaLaunchKernelEx(&lc, k_chol_solve<16>, ctx->ctl, ctx->d, hpk, shift_ptr, rhs, x, ctx->M,
                          z, x_out, mode, ignore_halt, dbg));
  }
  return FB_OK;
}
bool dense_kind(const Ctx* ctx) {
  return ctx->cfg.kind == FB_KIND_IDENTITY || ctx->cfg.kind == FB_KIND_NATURAL;
}
// master fold Hout = Hin + (alpha/n) sum_c delta_c (ascending c); for the
// dense kinds the client shift update rides along when `hest` is non-null
// k_finish grid when it also copies H^{k+1} -> H^k: about 8 doubles per thread
int finish_grid(const Ctx* ctx) {
  return static_cast<int>(std::min<int64_t>(2 * ctx->num_sms, (ctx->w + 2047) / 2048));
}

int launch_master_fold(Ctx* ctx, cudaStream_t s, const int32_t* clients, int n_active,
                       double* hest, const double* h_in, double* h_out, bool client_update = false) {
  if (dense_kind(ctx)) {
    k_fold_dense<<<static_cast<unsigned>((ctx->w + 255) / 256), 256, 0, s>>>(
        ctx->ctl, ctx->w, n_active, clients, ctx->cfg.alpha, ctx->alpha_n, ctx->D, ctx->count,
        hest, h_in, h_out);
  } else {
    const size_t smem = sizeof(int32_t) * (3 * static_cast<size_t>(n_active) + 1);
    k_master_fold<<<ctx->nr, FOLD_THREADS, smem, s>>>(
        ctx->ctl, ctx->w, n_active, clients, ctx->cap, ctx->nr, ctx->rs, ctx->idx_list,
        ctx->val_list, ctx->alpha_n, h_in, h_out, client_update ? ctx->hest : nullptr, ctx->w,
        ctx->cfg.alpha);
  }
  CKL();
  return FB_OK;
}

int record(Ctx* ctx, EvSlot slot, cudaStream_t s) {
  // event-record nodes only in the instrumented graph: a node between two
  // kernels costs the overlap of their launches (measured 24 us per c0 round
  // for the seven per-kernel ones; the production graph has none, its rows'
  // wall times come from the host's per-launch events)
  if (!ctx->phase_events) return FB_OK;
  ctx->ev_used[slot] = true;
  CK(cudaEventRecordWithFlags(ctx->ev_fixed[slot], s, cudaEventRecordExternal));
  return FB_OK;
}

// ---------------------------------------------------------- round bodies
int enqueue_fednl_round(Ctx* ctx) {
  cudaStream_t s = ctx->st;
  const int n = ctx->n;
  const bool ls = ctx->cfg.algorithm == FB_ALG_LS;
  TRY(record(ctx, EV_START, s));
  const bool shd = sharded(ctx);
  const int32_t* loc = shd ? ctx->local_clients : nullptr;  // this rank's clients
  const int n_loc = shd ? ctx->c_hi - ctx->c_lo : n;
  // the margins clear the round's client flags (no memset node before them)
  TRY(launch_margins(ctx, s, ctx->x, loc, n_loc, true, ctx->flags));
  TRY(record(ctx, EV_ORACLE_END, s));
  // Hessian + D + Frobenius partials, with the local gradients fused in
  TRY(launch_hessian(ctx, s, loc, n_loc, ctx->hest, ctx->w, ctx->D, nullptr, true, ctx->x));
  if (shd) {  // every rank gets every client's oracle outputs (same reduction order)
    TRY(gather_clients(ctx, ctx->grad, ctx->d, ncclFloat64, s));
    TRY(gather_clients(ctx, ctx->loss_part, ctx->nblk, ncclFloat64, s));
    TRY(gather_clients(ctx, ctx->frob_part, ctx->n_pairs, ncclFloat64, s));
    TRY(gather_clients(ctx, ctx->flags, 1, ncclInt32, s));
  }
  TRY(record(ctx, EV_HESS_END, s));
  // the round reduction: folded into the panel solve's prologue when that
  // kernel runs (its cluster forms the scalars it needs first), else k_reduce
  const bool opt_a = ctx->cfg.option == FB_OPTION_A;
  const bool fuse_red = ctx->solve_panels && !opt_a;
  CpRed red{};
  if (fuse_red) {
    red.n_active = n;
    red.n_div = n;
    red.ni = ctx->ni_arr;
    red.lam = ctx->lam_arr;
    red.nblk = ctx->nblk;
    red.n_pairs = ctx->n_pairs;
    red.grad = ctx->grad;
    red.loss_part = ctx->loss_part;
    red.frob_part = ctx->frob_part;
    red.flags = ctx->flags;
    red.gbar = ctx->gbar;
    red.f_cli = ctx->f_cli;
    red.shift_cli = ctx->shift_cli;
    red.out = ctx->sc;
    red.row_grad = ctx->row_grad;
    red.row_f = ctx->row_f;
  } else {
    TRY(launch_reduce(ctx, s, ctx->x, nullptr, n, n, true, ctx->row_grad, ctx->row_f, ctx->hmas));
  }
  TRY(record(ctx, EV_REDUCE_END, s));
  // fork: the master solve on st, the compressor and master fold on st2.  The
  // solve's cluster is launched first and the compressor waits for its
  // launch-completion event (the solve is the critical path and needs
  // CH_MAX_CLUSTER SMs at once; the compressor would otherwise fill them).
  // Under a profiler's injection library (ncu serialises every launch anyway)
  // the launch-completion attribute is not supported: order the compressor
  // after the solve instead.
#ifdef FB_SERIAL_EXP
  const bool serial = true;
#else
  const bool serial = under_profiler();
#endif
  CK(cudaEventRecord(ctx->ev_fork, s));
  CK(cudaStreamWaitEvent(ctx->st2, ctx->ev_fork, 0));
  if (opt_a) {  // eigen_clamp_min(H^k, mu) of the pre-fold estimate, then its Cholesky solve
    k_eig_clamp<<<1, EIG_THREADS, eig_smem_bytes(ctx->d), s>>>(
        ctx->ctl, ctx->d, ctx->hmas, nullptr, ctx->cfg.mu, ctx->eigA, ctx->eigV, ctx->hclamp, nullptr, 0);
    CKL();
  }
  TRY(launch_solve(ctx, s, opt_a ? ctx->hclamp : ctx->hmas,
                   opt_a ? ctx->zeros_w : &ctx->sc->shift_mean, ctx->gbar, ctx->x, ctx->pvec,
                   ctx->x_new, ls ? 2 : 0, 0, nullptr, serial ? nullptr : ctx->ev_solve_launched,
                   false, !serial && !opt_a, fuse_red ? &red : nullptr));
  if (serial) {
    CK(cudaEventRecord(ctx->ev_solve_launched, s));
  }
  CK(cudaStreamWaitEvent(ctx->st2, ctx->ev_solve_launched, 0));
  if (fuse_red && !serial) {  // the compressor waits for the solve's reduction (k_wait_reduce)
    k_wait_reduce<<<1, 32, 0, ctx->st2>>>(ctx->ctl);
    CKL();
  }
  TRY(record(ctx, EV_COMP_START, ctx->st2));
  // split TopK: the client shift update runs in the fold (K7), which stages
  // every client's entries per position range anyway
  const bool cu_fold = ctx->topk_split && !shd;
  TRY(launch_compress(ctx, ctx->st2, loc, n_loc, nullptr, nullptr, true, true, cu_fold));
  if (shd) {  // every rank folds every client's delta (ascending client id)
    if (dense_kind(ctx)) {  // the dense update itself (natural: the rounded values)
      TRY(gather_clients(ctx, ctx->D, static_cast<size_t>(ctx->w), ncclFloat64, ctx->st2));
    } else {
      TRY(gather_clients(ctx, ctx->idx_list, ctx->cap, ncclUint32, ctx->st2));
      TRY(gather_clients(ctx, ctx->val_list, ctx->cap, ncclFloat64, ctx->st2));
      TRY(gather_clients(ctx, ctx->rs, ctx->nr + 1, ncclInt32, ctx->st2));
    }
    TRY(gather_clients(ctx, ctx->count, 1, ncclInt32, ctx->st2));
    // a compressor failure is rank-local: every rank halts on the first one
    k_code_post<<<1, 32, 0, ctx->st2>>>(ctx->ctl, ctx->rank, ctx->xcode);
    CKL();
    TRY(gather_blocks(ctx, ctx->xcode, 1, ncclInt32, ctx->st2));
    k_code_sync<<<1, 32, 0, ctx->st2>>>(ctx->ctl, ctx->world, ctx->xcode);
    CKL();
  }
  TRY(record(ctx, EV_COMP_END, ctx->st2));
  TRY(record(ctx, EV_FOLD_START, ctx->st2));
  // dense kinds: the client shift update rides in the fold over this rank's
  // clients' rows (every rank folds all clients into H^{k+1})
  TRY(launch_master_fold(ctx, ctx->st2, nullptr, n, dense_kind(ctx) ? ctx->hest : nullptr,
                         ctx->hmas, ctx->hmas2, cu_fold));
  TRY(record(ctx, EV_FOLD_END, ctx->st2));
  CK(cudaEventRecord(ctx->ev_join, ctx->st2));
  TRY(record(ctx, EV_SOLVE_END, s));
  int launches = ctx->topk_split ? 9 : 8;
  if (ls) {
    // FedNL-LS: the first batch of LS_BATCH Armijo trials in line, later
    // batches (rare) as the body of a while-conditional node that the first
    // k_ls_decide arms; k_ls_decide keeps the loop going until a trial
    // passes, or raises ST_LINE_SEARCH past s = 60 (algorithms.py:284-311)
    cudaStreamCaptureStatus cst;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CK(cudaStreamGetCaptureInfo(s, &cst, nullptr, &cg, &deps, &ndeps));
    cudaGraphConditionalHandle loop;
    CK(cudaGraphConditionalHandleCreate(&loop, cg, 0, cudaGraphCondAssignDefault));
    auto ls_batch = [&](cudaStream_t q) -> int {
      dim3 grid(ctx->ls_nblk, n_loc);
      with_b(ctx, [&](auto B) {
        using T = std::remove_cv_t<std::remove_pointer_t<decltype(B)>>;
        k_ls_trials<T><<<grid, MARGIN_THREADS, LS_BATCH * ctx->d * sizeof(double), q>>>(
            ctx->ctl, B, ctx->d, ctx->ni_arr, ctx->ldj, loc, ctx->x, ctx->pvec, ctx->steps_table,
            ctx->trial_x, ctx->ls_loss_part, ctx->ls_nblk);
      });
      CKL();
      if (shd)  // the trials' per-client loss partials of every rank
        TRY(gather_clients(ctx, ctx->ls_loss_part, static_cast<size_t>(LS_BATCH) * ctx->ls_nblk,
                           ncclFloat64, q));
      k_ls_decide<<<1, 256, 0, q>>>(ctx->ctl, ctx->d, n, ctx->ni_arr, ctx->lam_arr, ctx->ls_nblk,
                                    ctx->cfg.ls_c, ctx->steps_table, ctx->trial_x, ctx->ls_loss_part,
                                    ctx->sc, ctx->x_new, LS_BATCH, ctx->gbar, ctx->pvec, loop);
      CKL();
      return FB_OK;
    };
    TRY(ls_batch(s));
    CK(cudaStreamGetCaptureInfo(s, &cst, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = loop;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, cg, deps, ndeps, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(ctx->st_body, body, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    const int r1 = ls_batch(ctx->st_body);
    cudaGraph_t body_out = body;
    const cudaError_t e2 = cudaStreamEndCapture(ctx->st_body, &body_out);
    if (r1 != FB_OK) return r1;
    CK(e2);
    CK(cudaStreamUpdateCaptureDependencies(s, &wnode, 1, cudaStreamSetCaptureDependencies));
    launches += 2;
  }
  CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
  k_finish<<<finish_grid(ctx), 256, 0, s>>>(ctx->ctl, ctx->d, n, n, nullptr, ctx->x, ctx->x_new, 1,
                                            ctx->count, ctx->row_counts, ctx->row_ls, ctx->row_grad,
                                            ctx->hmas2, ctx->hmas, ctx->w);
  CKL();
  TRY(record(ctx, EV_END, s));
  ctx->launches_per_round = launches;
  return FB_OK;
}

// FedNL-PP participants across ranks (fb_set_shard): this rank's slots
// [s_lo, s_hi) of the replicated subset, then the slot exchange (k_pp_pack /
// all-gathers / k_pp_unpack) and the replicated master update and fold.
int enqueue_pp_participants_sharded(Ctx* ctx) {
  cudaStream_t s = ctx->st;
  const int n = ctx->n, tau = ctx->tau, d = ctx->d, m = ctx->s_hi - ctx->s_lo;
  CK(cudaMemsetAsync(ctx->flags, 0, sizeof(int32_t) * n, s));
  if (m > 0) {
    k_pp_subloc<<<1, 32, 0, s>>>(ctx->subset, ctx->s_lo, m, ctx->sub_loc);
    CKL();
    TRY(launch_margins(ctx, s, ctx->x, ctx->sub_loc, m));
    TRY(launch_gradient(ctx, s, ctx->x, ctx->sub_loc, m));
    TRY(launch_hessian(ctx, s, ctx->sub_loc, m, ctx->hest, ctx->w, ctx->D, ctx->hess_part));
    k_check_flags_pp<<<1, 32, 0, s>>>(ctx->ctl, m, ctx->sub_loc, ctx->flags);  // (exchanged below)
    CKL();
    TRY(launch_compress(ctx, s, ctx->sub_loc, m, nullptr, nullptr));
    if (dense_kind(ctx)) TRY(launch_master_fold(ctx, s, ctx->sub_loc, m, ctx->hest, nullptr, nullptr));
    k_pp_shift_part<<<dim3(PP_SB, m), 256, 0, s>>>(ctx->ctl, d, ctx->sub_loc, ctx->hest, ctx->hess_part,
                                                   ctx->pp_shift_part);
    CKL();
    k_pp_client<<<dim3((d + 7) / 8, m), 256, 0, s>>>(ctx->ctl, d, ctx->sub_loc, ctx->hest, ctx->pp_shift_part,
                                                     ctx->x, ctx->grad, ctx->cli_shift, ctx->cli_gvec,
                                                     ctx->dshift, ctx->dgvec);
    CKL();
    k_pp_pack<<<m, 256, 0, s>>>(ctx->ctl, d, ctx->w, ctx->cap, ctx->nr, ctx->s_lo, ctx->rank, ctx->sub_loc,
                                ctx->idx_list, ctx->val_list, ctx->count, ctx->rs, ctx->flags, ctx->cli_gvec,
                                ctx->cli_shift, ctx->dgvec, ctx->dshift, ctx->D, ctx->ppx);
    CKL();
  }
  k_code_post<<<1, 32, 0, s>>>(ctx->ctl, ctx->rank, ctx->ppx.code);
  CKL();
  const size_t sp = static_cast<size_t>(ctx->spr);
  PpX& x = ctx->ppx;
  TRY(gather_blocks(ctx, x.idx, sp * ctx->cap, ncclUint32, s));
  TRY(gather_blocks(ctx, x.val, sp * ctx->cap, ncclFloat64, s));
  TRY(gather_blocks(ctx, x.cnt, sp, ncclInt32, s));
  TRY(gather_blocks(ctx, x.rs, sp * (ctx->nr + 1), ncclInt32, s));
  TRY(gather_blocks(ctx, x.flags, sp, ncclInt32, s));
  TRY(gather_blocks(ctx, x.gvec, sp * d, ncclFloat64, s));
  TRY(gather_blocks(ctx, x.shift, sp, ncclFloat64, s));
  TRY(gather_blocks(ctx, x.dg, sp * d, ncclFloat64, s));
  TRY(gather_blocks(ctx, x.ds, sp, ncclFloat64, s));
  if (x.dense) TRY(gather_blocks(ctx, x.dense, sp * static_cast<size_t>(ctx->w), ncclFloat64, s));
  TRY(gather_blocks(ctx, x.code, 1, ncclInt32, s));
  k_pp_unpack<<<tau, 256, 0, s>>>(ctx->ctl, d, ctx->w, ctx->cap, ctx->nr, ctx->s_lo, ctx->s_hi, ctx->world,
                                  ctx->cfg.alpha, ctx->subset, x, ctx->idx_list, ctx->val_list, ctx->count,
                                  ctx->rs, ctx->flags, ctx->cli_gvec, ctx->cli_shift, ctx->dgvec_all,
                                  ctx->dshift_all, ctx->D, ctx->hest);
  CKL();
  k_check_flags_pp<<<1, 32, 0, s>>>(ctx->ctl, tau, ctx->subset, ctx->flags);
  CKL();
  k_pp_master<<<1, 256, 0, s>>>(ctx->ctl, d, n, tau, ctx->dshift_all, ctx->dgvec_all, ctx->gvec, ctx->pp_shift);
  CKL();
  TRY(launch_master_fold(ctx, s, ctx->subset, tau, nullptr, ctx->hmas, ctx->hmas));
  k_finish<<<1, 256, 0, s>>>(ctx->ctl, d, n, tau, ctx->subset, ctx->x, nullptr, 0, ctx->count,
                             ctx->row_counts, ctx->row_ls, nullptr);
  CKL();
  TRY(record(ctx, EV_END, s));
  ctx->launches_per_round = 16;
  return FB_OK;
}

int enqueue_pp_round(Ctx* ctx) {
  cudaStream_t s = ctx->st;
  const int n = ctx->n, tau = ctx->tau;
  TRY(record(ctx, EV_START, s));
  // the metric probes over all clients at the current iterate
  // (runtime.py:237-238) only feed the row: they run on the second stream
  // while the master forms the new point from the running averages
  // (algorithms.py:422-433) into x_new (x <- x_new after the join).  The
  // solve's cluster is launched first; the probes wait for its launch
  // completion (as the FedNL round's compressor does).
  const bool pp_serial = under_profiler();
  TRY(launch_solve(ctx, s, ctx->hmas, ctx->pp_shift, ctx->gvec, nullptr, ctx->pvec, ctx->x_new, 1, 0,
                   nullptr, pp_serial ? nullptr : ctx->ev_solve_launched));
  cudaStream_t sp = pp_serial ? s : ctx->st2;
  if (!pp_serial) CK(cudaStreamWaitEvent(sp, ctx->ev_solve_launched, 0));
  // this round's participants (master subset stream) off the critical path too
  k_pp_select<<<1, 128, 0, sp>>>(ctx->ctl, n, tau, ctx->subset, ctx->pool);
  CKL();
  const bool shd = sharded(ctx);
  if (shd) {  // the probes of this rank's client range, all-gathered
    TRY(launch_margins(ctx, sp, ctx->x, ctx->local_clients, ctx->c_hi - ctx->c_lo));
    TRY(launch_gradient(ctx, sp, ctx->x, ctx->local_clients, ctx->c_hi - ctx->c_lo));
    TRY(gather_clients(ctx, ctx->grad, ctx->d, ncclFloat64, sp));
    TRY(gather_clients(ctx, ctx->loss_part, ctx->nblk, ncclFloat64, sp));
  } else {
    TRY(launch_margins(ctx, sp, ctx->x, nullptr, n));
    TRY(launch_gradient(ctx, sp, ctx->x, nullptr, n));
  }
  TRY(launch_reduce(ctx, sp, ctx->x, nullptr, n, n, false, ctx->row_grad, ctx->row_f));
  if (!pp_serial) {
    CK(cudaEventRecord(ctx->ev_join, sp));
    CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
  }
  // the stop rule on the probe row, then x <- x_new (or DivergenceError)
  k_pp_advance<<<1, 256, 0, s>>>(ctx->ctl, ctx->d, n, ctx->x, ctx->x_new, ctx->row_grad,
                                 ctx->row_counts, ctx->row_ls);
  CKL();
  TRY(record(ctx, EV_SOLVE_END, s));
  if (shd) return enqueue_pp_participants_sharded(ctx);
  // participants' oracle at x_new (algorithms.py:240-249)
  CK(cudaMemsetAsync(ctx->flags, 0, sizeof(int32_t) * n, s));
  TRY(launch_margins(ctx, s, ctx->x, ctx->subset, tau));
  TRY(launch_gradient(ctx, s, ctx->x, ctx->subset, tau));
  TRY(record(ctx, EV_ORACLE_END, s));
  TRY(launch_hessian(ctx, s, ctx->subset, tau, ctx->hest, ctx->w, ctx->D, ctx->hess_part));
  TRY(record(ctx, EV_HESS_END, s));
  k_check_flags_pp<<<1, 32, 0, s>>>(ctx->ctl, tau, ctx->subset, ctx->flags);
  CKL();
  TRY(record(ctx, EV_REDUCE_END, s));
  TRY(record(ctx, EV_COMP_START, s));
  TRY(launch_compress(ctx, s, ctx->subset, tau, nullptr, nullptr));
  TRY(record(ctx, EV_COMP_END, s));
  TRY(record(ctx, EV_FOLD_START, s));
  if (dense_kind(ctx))  // the sparse compressors already applied the client update
    TRY(launch_master_fold(ctx, s, ctx->subset, tau, ctx->hest, nullptr, nullptr));
  k_pp_shift_part<<<dim3(PP_SB, tau), 256, 0, s>>>(ctx->ctl, ctx->d, ctx->subset, ctx->hest,
                                                   ctx->hess_part, ctx->pp_shift_part);
  CKL();
  k_pp_client<<<dim3((ctx->d + 7) / 8, tau), 256, 0, s>>>(
      ctx->ctl, ctx->d, ctx->subset, ctx->hest, ctx->pp_shift_part, ctx->x, ctx->grad,
      ctx->cli_shift, ctx->cli_gvec, ctx->dshift, ctx->dgvec);
  CKL();
  k_pp_master<<<1, 256, 0, s>>>(ctx->ctl, ctx->d, n, tau, ctx->dshift, ctx->dgvec, ctx->gvec,
                                ctx->pp_shift);
  CKL();
  TRY(launch_master_fold(ctx, s, ctx->subset, tau, nullptr, ctx->hmas, ctx->hmas));
  TRY(record(ctx, EV_FOLD_END, s));
  k_finish<<<1, 256, 0, s>>>(ctx->ctl, ctx->d, n, tau, ctx->subset, ctx->x, nullptr, 0, ctx->count,
                             ctx->row_counts, ctx->row_ls, nullptr);
  CKL();
  TRY(record(ctx, EV_END, s));
  ctx->launches_per_round = ctx->topk_split ? 17 : 16;
  return FB_OK;
}

// rounds per launch of the plain FedNL production graph (the run loop falls
// back to the one-round graph for a chunk's remainder): c0 +1%, c1 +3%.  The
// FedNL-LS (while node) and FedNL-PP (concurrent probe branch) rounds lose
// 11-14% when several are captured into one graph and keep one per launch.
constexpr int GRAPH_ROUNDS = 4;

void drop_graphs(Ctx* ctx) {
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->graph) cudaGraphDestroy(ctx->graph);
  if (ctx->gexec_multi) cudaGraphExecDestroy(ctx->gexec_multi);
  if (ctx->graph_multi) cudaGraphDestroy(ctx->graph_multi);
  ctx->gexec = nullptr;
  ctx->graph = nullptr;
  ctx->gexec_multi = nullptr;
  ctx->graph_multi = nullptr;
}

int build_graph(Ctx* ctx, bool phase_events) {
  if (ctx->gexec && ctx->gexec_phase == phase_events) return FB_OK;
  drop_graphs(ctx);  // the other flavour: rebuilt (the first call of a timed run)
  ctx->phase_events = phase_events;
  ctx->gexec_phase = phase_events;
  for (int i = 0; i < EV_COUNT; ++i) {
    ctx->ev_used[i] = false;
    ctx->ev_node[i] = nullptr;
  }
  CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
  int r = (ctx->cfg.algorithm == FB_ALG_PP) ? enqueue_pp_round(ctx) : enqueue_fednl_round(ctx);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(ctx->st, &g);
  if (r != FB_OK) {
    if (g) cudaGraphDestroy(g);
    return r;
  }
  CK(e);
  ctx->graph = g;
  // locate the event-record nodes so timed runs can retarget them
  size_t nn = 0;
  CK(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CK(cudaGraphGetNodes(g, nodes.data(), &nn));
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess) {  // (the LS loop's conditional node)
      cudaGetLastError();
      continue;
    }
    if (ty != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t ev;
    CK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
    for (int i = 0; i < EV_COUNT; ++i)
      if (ev == ctx->ev_fixed[i]) ctx->ev_node[i] = nd;
  }
  // the blocked solve's many launches need their per-node priority honoured
  // (without the flag a graph runs every node at the launch stream's
  // priority: each panel kernel queued behind the c4 TopK pass and the fold;
  // c4 solve 1.16 -> 0.63 ms in the round).  The cluster solvers launch once
  // and hold the compressor back until resident: no flag there (c1 -3% with it)
  const unsigned gflags = ctx->solve_big ? cudaGraphInstantiateFlagUseNodePriority : 0;
  CK(cudaGraphInstantiateWithFlags(&ctx->gexec, g, gflags));
  if (!phase_events && ctx->cfg.algorithm == FB_ALG_FEDNL) {
    CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    int rr = FB_OK;
    for (int k = 0; k < GRAPH_ROUNDS && rr == FB_OK; ++k)
      rr = (ctx->cfg.algorithm == FB_ALG_PP) ? enqueue_pp_round(ctx) : enqueue_fednl_round(ctx);
    cudaGraph_t gm = nullptr;
    cudaError_t em = cudaStreamEndCapture(ctx->st, &gm);
    if (rr != FB_OK) {
      if (gm) cudaGraphDestroy(gm);
      return rr;
    }
    CK(em);
    ctx->graph_multi = gm;
    CK(cudaGraphInstantiateWithFlags(&ctx->gexec_multi, gm, gflags));
  }
  return FB_OK;
}

int read_status(Ctx* ctx, DevCtl* host_ctl) {
  CK(cudaMemcpyAsync(host_ctl, ctx->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return FB_OK;
}

int status_to_code(int32_t code) {
  switch (code) {
    case ST_OK: return FB_OK;
    case ST_NOT_PD: return FB_ERR_NOT_PD;
    case ST_NONFINITE: return FB_ERR_NONFINITE;
    case ST_TOPLEK_ZERO: return FB_ERR_INVALID;
    case ST_DIVERGED: return FB_ERR_DIVERGED;
    case ST_LINE_SEARCH: return FB_ERR_LINE_SEARCH;
    case ST_STOPPED: return FB_OK;
    case ST_EIGEN: return FB_ERR_EIGEN;
    default: return FB_ERR_CUDA;
  }
}

int clear_status(Ctx* ctx) {
  DevCtl h;
  TRY(read_status(ctx, &h));
  h.halt = 0;
  h.code = 0;
  h.code_round = 0;
  h.ls_next = 0;
  CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof(DevCtl), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return FB_OK;
}

}  // namespace

// ======================================================================
// C ABI
// ======================================================================
extern "C" {

int fb_abi_sizes(int32_t* out3) {
  if (!out3) return invalid(nullptr, "null argument");
  out3[0] = static_cast<int32_t>(sizeof(fb_config));
  out3[1] = static_cast<int32_t>(sizeof(fb_status));
  out3[2] = static_cast<int32_t>(sizeof(fb_profile));
  return FB_OK;
}

const char* fb_last_error(void* handle) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  return ctx ? ctx->err.c_str() : g_err.c_str();
}

int fb_device_info(char* name, int32_t name_len, int32_t* sm_count, int32_t* cc_major,
                   int32_t* cc_minor) {
  int dev = 0;
  cudaDeviceProp p;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
    g_err = "no CUDA device";
    return FB_ERR_CUDA;
  }
  if (name && name_len > 0) {
    strncpy(name, p.name, name_len - 1);
    name[name_len - 1] = 0;
  }
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return FB_OK;
}

int fb_create(const fb_config* cfg_in, void** out) {
  if (!cfg_in || !out) return invalid(nullptr, "null argument");
  *out = nullptr;
  const fb_config& c = *cfg_in;
  if (c.d < 1 || c.n_clients < 1 || c.n_samples < 1) return invalid(nullptr, "bad shape");
  if (c.d > FB_MAX_D) return invalid(nullptr, "d > 4096 is outside this build's envelope");
  if (c.n_clients >= (1 << 24)) return invalid(nullptr, "too many clients");
  const int64_t w = packed_len(c.d);
  if (c.kind < FB_KIND_IDENTITY || c.kind > FB_KIND_NATURAL) return invalid(nullptr, "bad kind");
  const bool sparse = c.kind == FB_KIND_TOPK || c.kind == FB_KIND_TOPLEK ||
                      c.kind == FB_KIND_RANDK || c.kind == FB_KIND_RANDSEQK;
  if (sparse && (c.k < 1 || c.k > w)) return invalid(nullptr, "k out of range");
  if (c.algorithm == FB_ALG_PP && (c.tau < 1 || c.tau > c.n_clients))
    return invalid(nullptr, "tau out of range");
  if (c.topk_path < FB_TOPK_PATH_AUTO || c.topk_path > FB_TOPK_PATH_SPLIT)
    return invalid(nullptr, "bad topk_path");
  if (c.kind == FB_KIND_RANDK && rk_smem_bytes(c.k, static_cast<int>((w + 31) / 32), w) > RK_SMEM_MAX)
    return invalid(nullptr, "randk scratch does not fit shared memory");

  Ctx* ctx = new Ctx();
  ctx->cfg = c;
  ctx->d = c.d;
  ctx->n = c.n_clients;
  ctx->ni = c.n_samples;
  ctx->w = w;
  ctx->npr = c.n_clients;
  ctx->c_lo = 0;
  ctx->c_hi = c.n_clients;
  ctx->ldj = (c.n_samples + 1) & ~1;
  ctx->ldh = (c.n_samples + 15) & ~15;
  ctx->nblk = (ctx->ldh + MB_SAMPLES - 1) / MB_SAMPLES;
  ctx->ls_nblk = (ctx->ldh + MARGIN_THREADS - 1) / MARGIN_THREADS;
  ctx->nb_tiles = (c.d + HT - 1) / HT;
  ctx->n_pairs = ctx->nb_tiles * (ctx->nb_tiles + 1) / 2;
  ctx->wb = static_cast<int>((w + 31) / 32);
  ctx->cap = sparse ? c.k : 1;
  ctx->nr = static_cast<int>((w + FOLD_RANGE - 1) / FOLD_RANGE);
  ctx->tau = c.algorithm == FB_ALG_PP ? c.tau : c.n_clients;
  ctx->alpha_n = c.alpha / static_cast<double>(c.n_clients);
  ctx->rand_scale = (c.kind == FB_KIND_RANDK || c.kind == FB_KIND_RANDSEQK)
                        ? static_cast<double>(w) / static_cast<double>(c.k)
                        : 1.0;
  ctx->toplek_P = 1;
  if (c.kind == FB_KIND_TOPLEK && w <= TLB_MAXW_SMEM)
    while (ctx->toplek_P < w || ctx->toplek_P < TK_THREADS) ctx->toplek_P <<= 1;
  // master solve: one cluster (8 CTAs from d >= 128); 32-wide panels while the
  // (d + 1) x 33 panel fits in shared memory, else 16-wide
  // 6 CTAs below d = 512 leave the per-client compressor (one CTA per SM)
  // enough SMs to run in a single wave next to the solve
  ctx->solve_cs = c.d < 128 ? 1 : (c.d < 512 ? 6 : CH_MAX_CLUSTER);
  ctx->solve_nb = solve_panel_bytes<32>(c.d) <= 190 * 1024 ? 32 : 16;
  {
    // panel-owning solve: one or two 32-column panels per CTA of a portable
    // (<= 8) cluster, while the panels fit in shared memory
    const int npan = (c.d + CP_NB - 1) / CP_NB;
    // one panel per CTA (a cluster of up to 16) when the round's compressor
    // CTAs (one per active client, one SM each: the solve CTA's registers
    // leave no room beside it) still fit the other SMs in one wave; else two
    // panels per CTA of a portable cluster
    const int comp_ctas = c.algorithm == FB_ALG_PP ? c.tau : c.n_clients;
    ctx->cp_kp = (npan <= CH_MAX_CLUSTER || (npan <= CP_MAX_CLUSTER && comp_ctas + npan <= ctx->num_sms)) ? 1 : 2;
    ctx->cp_cs = (npan + ctx->cp_kp - 1) / ctx->cp_kp;
    // (three panels or fewer: the cluster-redundant solver is faster)
    ctx->solve_panels = npan >= 4 && c.d <= CP_MAX_D && ctx->cp_cs <= CP_MAX_CLUSTER &&
                        static_cast<size_t>(ctx->cp_kp) * cp_panel_bytes(c.d) <= CP_DYN_SMEM_MAX;
  }
  // d > CP_MAX_D: the global-memory blocked solve (solve_big.cuh)
  ctx->solve_big = c.d > CP_MAX_D;
  if (ctx->solve_big) ctx->solve_panels = false;
  ctx->solve_smem = c.d > CH_MAX_D ? 0
                    : (ctx->solve_nb == 32 ? solve_panel_bytes<32>(c.d) : solve_panel_bytes<16>(c.d));
  int rc = FB_OK;
  auto fail = [&](int code) {
    rc = code;
    g_err = ctx->err;
    fb_destroy(ctx);
    return code;
  };
  if (cudaSetDevice(0) != cudaSuccess) {
    ctx->err = "cudaSetDevice(0) failed";
    return fail(FB_ERR_CUDA);
  }
  int dev = 0;
  int cc_major = 0;
  if (cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cc_major != 10) {
    ctx->err = "libfednl_b200 needs an sm_100 (B200) device";
    return fail(FB_ERR_CUDA);
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev);
#define CKC(call)                                                     \
  do {                                                                \
    cudaError_t e_ = (call);                                          \
    if (e_ != cudaSuccess) {                                          \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);  \
      return fail(FB_ERR_CUDA);                                       \
    }                                                                 \
  } while (0)
  {
    int lo = 0, hi = 0;
    CKC(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ctx->prio_high = hi;
  }
  CKC(cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking));
  CKC(cudaStreamCreateWithFlags(&ctx->st2, cudaStreamNonBlocking));
  CKC(cudaStreamCreateWithFlags(&ctx->st_body, cudaStreamNonBlocking));
  CKC(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&ctx->ev_solve_launched, cudaEventDisableTiming));
  for (int i = 0; i < EV_COUNT; ++i) CKC(cudaEventCreate(&ctx->ev_fixed[i]));
  // dynamic shared memory limits are per-function process state: only ever
  // raise them, so contexts of different shapes can coexist
  static size_t max_toplek = 0, max_solve = 0;
  max_toplek = std::max(max_toplek, toplek_smem_bytes(std::max(ctx->toplek_P, 1)));
  max_solve = std::max(max_solve, std::max<size_t>(ctx->solve_smem, 1));
  CKC(cudaFuncSetAttribute(k_hessian_ws<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(HESS_WS_SMEM)));
  CKC(cudaFuncSetAttribute(k_hessian_ws<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(HESS_WS_SMEM)));
  CKC(cudaFuncSetAttribute(k_topk_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(TKS_SMEM)));
#define FB_MC_ATTR(T)                                                                                  \
  CKC(cudaFuncSetAttribute(k_margins_cpc<MC_THREADS, 1, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           static_cast<int>(MC_SMEM_MAX)));                                               \
  CKC(cudaFuncSetAttribute(k_margins_cpc<512, 2, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                           static_cast<int>(MC_SMEM_MAX)));
  FB_MC_ATTR(double)
  FB_MC_ATTR(float)
  FB_MC_ATTR(int8_t)
#undef FB_MC_ATTR
  CKC(cudaFuncSetAttribute(k_big_panel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(BigSmem))));
  CKC(cudaFuncSetAttribute(k_big_back, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(big_back_smem(FB_MAX_D))));
  CKC(cudaFuncSetAttribute(k_ls_trials<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(LS_BATCH * FB_MAX_D * sizeof(double))));
  CKC(cudaFuncSetAttribute(k_ls_trials<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(LS_BATCH * FB_MAX_D * sizeof(double))));
  CKC(cudaFuncSetAttribute(k_ls_trials<int8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(LS_BATCH * FB_MAX_D * sizeof(double))));
  CKC(cudaFuncSetAttribute(k_topk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(tkst_smem_bytes(TKST_MAXW))));
  CKC(cudaFuncSetAttribute(k_tks_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(tkp_smem_bytes(TKST_MAXW))));
  CKC(cudaFuncSetAttribute(k_tks_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(tkp_smem_bytes(TKST_MAXW))));
  static size_t max_fold = 0;
  max_fold = std::max(max_fold, sizeof(int32_t) * (3 * static_cast<size_t>(c.n_clients) + 1));
  CKC(cudaFuncSetAttribute(k_master_fold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(max_fold)));
  CKC(cudaFuncSetAttribute(k_randk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(RK_SMEM_MAX)));
  CKC(cudaFuncSetAttribute(k_toplek, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(max_toplek)));
  CKC(cudaFuncSetAttribute(k_chol_solve<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(std::max(max_solve, solve_panel_bytes<32>(1)))));
  static size_t max_cp = 0;
  max_cp = std::max(max_cp, static_cast<size_t>(ctx->cp_kp) * cp_panel_bytes(c.d));
  CKC(cudaFuncSetAttribute(k_chol_panels<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CKC(cudaFuncSetAttribute(k_chol_panels<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(std::min<size_t>(max_cp + CP_STAMP_BYTES, CP_DYN_SMEM_MAX))));
  CKC(cudaFuncSetAttribute(k_chol_panels<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(std::min<size_t>(max_cp + CP_STAMP_BYTES, CP_DYN_SMEM_MAX))));
  CKC(cudaFuncSetAttribute(k_chol_solve<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(std::max(max_solve, solve_panel_bytes<16>(1)))));

  const int n = ctx->n, d = ctx->d;
  const size_t wn = static_cast<size_t>(w) * n;
  // one-pass sampled-window TopK from TKST_MINW up (c0: w = 45,451): one
  // read of D plus candidate work beats the shared-memory radix's passes
  const bool stream_topk = c.kind == FB_KIND_TOPK && w <= TKST_MAXW &&
                           (w > TKS_MAXW || w >= TKST_MINW);
  ctx->topk_stream = stream_topk;
  // the stream as many small CTAs (about two waves of 8 per SM) + a select
  // kernel when n * w is large (c4); topk_path pins either variant (tests)
  // (the split path's selection keeps a bitmap row in shared memory: w <~ 1.7M)
  ctx->topk_split = stream_topk && tkp_smem_bytes(w) <= 220 * 1024 && (c.topk_path == FB_TOPK_PATH_AUTO
                                        ? static_cast<int64_t>(w) * n >= (int64_t{1} << 26)
                                        : c.topk_path == FB_TOPK_PATH_SPLIT);
  size_t cand_slots = stream_topk ? static_cast<size_t>(n) * TKST_CAP : 1;
  if (ctx->topk_split) {
    // positions per CTA: one wave of two CTAs per SM when that is 8..64
    // ring stages each, else as close to 64 stages as an even split allows
    int64_t L = (static_cast<int64_t>(w) * n) / (2 * ctx->num_sms);
    L = std::min<int64_t>(std::max<int64_t>(L, 8 * TKP_CH), 64 * TKP_CH);
    int64_t S = std::max<int64_t>(1, (w + L / 2) / L);
    S = std::min<int64_t>(S, TKP_MAXSEG);
    int64_t lseg = ((w + S - 1) / S + TKP_CH - 1) / TKP_CH * TKP_CH;
    ctx->tks_lseg = static_cast<int>(lseg);
    ctx->tks_S = static_cast<int>((w + lseg - 1) / lseg);
    ctx->tks_capseg = static_cast<int>(std::min<int64_t>(lseg, TKP_SEGCAP));
    int ns = 2048;
    while (ns < TKW_MAXSAMPLE && ns * 64 <= w) ns *= 2;
    ctx->tks_ns = ns;
    cand_slots = static_cast<size_t>(n) * ctx->tks_S * ctx->tks_capseg;
  }
  const int tau = ctx->tau;
  if (dalloc(ctx, &ctx->ctl, 1) || dalloc(ctx, &ctx->Bt, static_cast<size_t>(n) * d * ctx->ldj) ||
      dalloc(ctx, &ctx->ni_arr, n) || dalloc(ctx, &ctx->lam_arr, n) || dalloc(ctx, &ctx->hess_sched, 2) ||
      dalloc(ctx, &ctx->x, d) || dalloc(ctx, &ctx->x_new, d) || dalloc(ctx, &ctx->pvec, d) ||
      dalloc(ctx, &ctx->zbuf, d) ||
      dalloc(ctx, &ctx->hcoef, static_cast<size_t>(n) * ctx->ldh) ||
      dalloc(ctx, &ctx->gcoef, static_cast<size_t>(n) * ctx->ldh) ||
      dalloc(ctx, &ctx->loss_part, static_cast<size_t>(n) * ctx->nblk) ||
      dalloc(ctx, &ctx->grad, static_cast<size_t>(n) * d) || dalloc(ctx, &ctx->gbar, d) ||
      dalloc(ctx, &ctx->f_cli, n) || dalloc(ctx, &ctx->shift_cli, n) ||
      dalloc(ctx, &ctx->frob_part, static_cast<size_t>(n) * ctx->n_pairs) ||
      dalloc(ctx, &ctx->flags, n) || dalloc(ctx, &ctx->hest, wn) || dalloc(ctx, &ctx->D, wn + 2) ||
      dalloc(ctx, &ctx->hmas, w) || dalloc(ctx, &ctx->hmas2, w) || dalloc(ctx, &ctx->zeros_w, w) ||
      dalloc(ctx, &ctx->eigA, d > EIG_SMEM_MAX_D ? static_cast<size_t>(d) * d : 1) ||
      dalloc(ctx, &ctx->eigV, static_cast<size_t>(d) * d) || dalloc(ctx, &ctx->hclamp, w) ||
      dalloc(ctx, &ctx->rs, static_cast<size_t>(n) * (ctx->nr + 1)) ||
      dalloc(ctx, &ctx->M, static_cast<size_t>(d + 1) * (d + 1)) ||
      dalloc(ctx, &ctx->Lbig, ctx->solve_big ? static_cast<size_t>(d + 1) * (d + 1) : 1) ||
      dalloc(ctx, &ctx->Tbig, ctx->solve_big ? static_cast<size_t>((d + BIG_NB - 1) / BIG_NB) * BIG_NB * BIG_NB : 1) ||
      dalloc(ctx, &ctx->Lg, ctx->solve_panels ? static_cast<size_t>((d + CP_NB - 1) / CP_NB) *
                                                    cp_rows(d) * CP_LS : 1) ||
      dalloc(ctx, &ctx->bitmap, static_cast<size_t>(n) * tks_wbp(w)) || dalloc(ctx, &ctx->count, n) ||
      dalloc(ctx, &ctx->draws, n) ||
      dalloc(ctx, &ctx->idx_list, static_cast<size_t>(n) * ctx->cap) ||
      dalloc(ctx, &ctx->val_list, static_cast<size_t>(n) * ctx->cap) ||
      dalloc(ctx, &ctx->seeds, n) || dalloc(ctx, &ctx->pair_order, ctx->n_pairs) ||
      dalloc(ctx, &ctx->cand_key, cand_slots) || dalloc(ctx, &ctx->cand_pos, cand_slots) ||
      dalloc(ctx, &ctx->tks_win, ctx->topk_split ? n : 1) ||
      dalloc(ctx, &ctx->tks_ticket, n) ||
      dalloc(ctx, &ctx->gt_val, ctx->topk_split ? cand_slots : 1) ||
      dalloc(ctx, &ctx->gt_pos, ctx->topk_split ? cand_slots : 1) ||
      dalloc(ctx, &ctx->tks_seg, ctx->topk_split ? static_cast<size_t>(n) * ctx->tks_S * TKP_CW : 1) ||
      dalloc(ctx, &ctx->tks_eqz, ctx->topk_split ? static_cast<size_t>(n) * tks_wbp(w) : 1) ||
      dalloc(ctx, &ctx->sc, 1) || dalloc(ctx, &ctx->steps_table, 64) ||
      dalloc(ctx, &ctx->trial_x, static_cast<size_t>(LS_BATCH) * d) ||
      dalloc(ctx, &ctx->ls_loss_part, static_cast<size_t>(LS_BATCH) * n * ctx->ls_nblk) ||
      dalloc(ctx, &ctx->subset, std::max(tau, 1)) || dalloc(ctx, &ctx->pool, n) ||
      dalloc(ctx, &ctx->hess_part, c.algorithm == FB_ALG_PP ? static_cast<size_t>(tau) * w : 1) ||
      dalloc(ctx, &ctx->cli_shift, n) ||
      dalloc(ctx, &ctx->cli_gvec, c.algorithm == FB_ALG_PP ? static_cast<size_t>(n) * d : 1) ||
      dalloc(ctx, &ctx->gvec, d) || dalloc(ctx, &ctx->pp_shift, 1) ||
      dalloc(ctx, &ctx->dshift, std::max(tau, 1)) ||
      dalloc(ctx, &ctx->pp_shift_part, static_cast<size_t>(std::max(tau, 1)) * PP_SB) ||
      dalloc(ctx, &ctx->dgvec, static_cast<size_t>(std::max(tau, 1)) * d) ||
      dalloc(ctx, &ctx->scalar, 4) || dalloc(ctx, &ctx->row_grad, ROW_CHUNK) ||
      dalloc(ctx, &ctx->row_f, ROW_CHUNK) ||
      dalloc(ctx, &ctx->row_counts, static_cast<size_t>(ROW_CHUNK) * n) ||
      dalloc(ctx, &ctx->row_ls, ROW_CHUNK)) {
    return fail(FB_ERR_CUDA);
  }
  {  // every client n_i = n_samples, lambda = lam until fb_upload_shards_ex says otherwise
    std::vector<int32_t> nis(n, c.n_samples);
    std::vector<double> lams(n, c.lam);
    CKC(cudaMemcpyAsync(ctx->ni_arr, nis.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->st));
    CKC(cudaMemcpyAsync(ctx->lam_arr, lams.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->st));
    CKC(cudaStreamSynchronize(ctx->st));
  }
  double steps[64];
  for (int i = 0; i < 64; ++i) steps[i] = c.ls_steps_table[i <= 60 ? i : 60];
  CKC(cudaMemcpyAsync(ctx->steps_table, steps, sizeof steps, cudaMemcpyHostToDevice, ctx->st));
  // Hessian tile pairs by decreasing DMMA work (fragment products of their
  // active quadrants, as k_hessian specialises them), ties by pair index
  std::vector<int32_t> order(ctx->n_pairs);
  {
    std::vector<int> cost(ctx->n_pairs, 0);
    for (int J = 0; J < ctx->nb_tiles; ++J)
      for (int I = 0; I <= J; ++I) {
        int cst = 0;
        for (int qd = 0; qd < 4; ++qd) {
          const int rb = 32 * (qd & 1), cb = 32 * (qd >> 1);
          if (I == J && rb > cb) continue;
          const int vr = (c.d - (I * HT + rb) + 7) / 8, vc = (c.d - (J * HT + cb) + 7) / 8;
          if (vr < 1 || vc < 1) continue;
          const int mr = vr >= 3 ? 4 : 2, nc = vc >= 3 ? 4 : 2;
          cst += (I == J && rb == cb) ? mr * (mr + 1) / 2 : mr * nc;
        }
        cost[J * (J + 1) / 2 + I] = cst;
      }
    for (int i = 0; i < ctx->n_pairs; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  }
  CKC(cudaMemcpyAsync(ctx->pair_order, order.data(), sizeof(int32_t) * ctx->n_pairs,
                      cudaMemcpyHostToDevice, ctx->st));
  if (c.kind == FB_KIND_TOPLEK) {
    // numpy's pairwise recursion over n = w (np.sum of the sorted energies):
    // leaves of <= 128 left to right, internal nodes in post-order
    std::vector<int32_t> loff, llen, nl_, nr_;
    std::function<int(int, int)> walk = [&](int o, int n) -> int {  // returns a node code
      if (n <= 128) {
        loff.push_back(o);
        llen.push_back(n);
        return -static_cast<int>(loff.size());  // leaf k -> -(k + 1)
      }
      int n2 = n / 2;
      n2 -= n2 % 8;
      const int a = walk(o, n2), b = walk(o + n2, n - n2);
      nl_.push_back(a);
      nr_.push_back(b);
      return static_cast<int>(nl_.size()) - 1;  // internal node index
    };
    walk(0, static_cast<int>(w));
    const int nlf = static_cast<int>(loff.size()), nnd = static_cast<int>(nl_.size());
    const bool big = w > TLB_MAXW_SMEM;  // k_toplek_big reads the table from global memory
    if (big) {
      const size_t nw = static_cast<size_t>(n) * w;
      ctx->tlb.npw_stride = 9 * static_cast<int64_t>(nlf) + nnd;
      if (dalloc(ctx, &ctx->tlb.key[0], nw) || dalloc(ctx, &ctx->tlb.key[1], nw) ||
          dalloc(ctx, &ctx->tlb.pos[0], nw) || dalloc(ctx, &ctx->tlb.pos[1], nw) ||
          dalloc(ctx, &ctx->tlb.npw, static_cast<size_t>(n) * ctx->tlb.npw_stride))
        return fail(FB_ERR_CUDA);
    }
    if (nlf <= NPW_TAB_LEAVES || big) {
      auto code = [&](int x) { return x < 0 ? -x - 1 : nlf + x; };
      std::vector<int32_t> tab{nlf, nnd};
      tab.insert(tab.end(), loff.begin(), loff.end());
      tab.insert(tab.end(), llen.begin(), llen.end());
      for (int q = 0; q < nnd; ++q) tab.push_back(code(nl_[q]));
      for (int q = 0; q < nnd; ++q) tab.push_back(code(nr_[q]));
      if (dalloc(ctx, &ctx->npw_tab, tab.size())) return fail(FB_ERR_CUDA);
      CKC(cudaMemcpyAsync(ctx->npw_tab, tab.data(), sizeof(int32_t) * tab.size(),
                          cudaMemcpyHostToDevice, ctx->st));
    }
  }
  if (c.kind == FB_KIND_RANDK) {
    const int wbk = static_cast<int>((w + 31) / 32);
    if (!rk_js_smem(c.k, wbk, w) && dalloc(ctx, &ctx->rk_js, static_cast<size_t>(n) * c.k))
      return fail(FB_ERR_CUDA);
    if (rk_global_pool(c.k, w) && dalloc(ctx, &ctx->rk_pool, static_cast<size_t>(n) * w))
      return fail(FB_ERR_CUDA);
  }
  CKC(cudaStreamSynchronize(ctx->st));  // zero fills and the tables are in place
  if (make_tmap(ctx) != FB_OK) return fail(FB_ERR_CUDA);
  *out = ctx;
  return rc;
#undef CKC
}

void fb_destroy(void* handle) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx) return;
  drop_graphs(ctx);
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  if (ctx->st2) cudaStreamSynchronize(ctx->st2);
  if (ctx->comm) nccl_api().CommDestroy(ctx->comm);
  for (auto& pa : ctx->allocs) cache_release(pa.first, pa.second);
  for (auto& e : ctx->ev_ends) if (e) cudaEventDestroy(e);
  for (auto& e : ctx->ev_pool) if (e) cudaEventDestroy(e);
  for (auto& e : ctx->ev_fixed) if (e) cudaEventDestroy(e);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_solve_launched) cudaEventDestroy(ctx->ev_solve_launched);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  if (ctx->st2) cudaStreamDestroy(ctx->st2);
  if (ctx->st_body) cudaStreamDestroy(ctx->st_body);
  delete ctx;
}

int fb_get_status(void* handle, fb_status* out) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !out) return invalid(ctx, "null argument");
  DevCtl h;
  TRY(read_status(ctx, &h));
  out->code = status_to_code(h.code);
  out->round = h.code_round;
  out->pivot_index = h.pivot_index;
  out->client = h.bad_client;
  out->pivot_value = h.pivot_value;
  out->f_start = h.f_start;
  out->f_best = h.f_best;
  return FB_OK;
}

// Shards -> Bt[c][a][j] (feature-major, sample rows padded to ldj).
__global__ void k_transpose_shard(const double* __restrict__ src, double* __restrict__ dst, int d,
                                  int ni, int ldj) {
  __shared__ double tile[32][33];
  const int j0 = blockIdx.x * 32, a0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = j0 + r, a = a0 + threadIdx.x;
    tile[r][threadIdx.x] = (j < ni && a < d) ? src[a + static_cast<int64_t>(j) * d] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int a = a0 + r, j = j0 + threadIdx.x;
    if (a < d && j < ldj) dst[static_cast<int64_t>(a) * ldj + j] = tile[threadIdx.x][r];
  }
}

// Shard upload: worker threads copy shards into pinned staging slots (two per
// worker), DMA them on the worker's own stream and transpose them into Bt.
// Slots, device staging and streams are process-wide and reused by later
// calls; the call returns once every shard is resident.
struct UploadLane {
  double* host[2] = {nullptr, nullptr};
  double* dev[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  size_t cap = 0;
};
struct UploadPool {
  std::mutex mu;
  std::vector<UploadLane> lanes;
};
UploadPool& upload_pool() {
  static UploadPool* p = new UploadPool;  // process lifetime
  return *p;
}
constexpr int UPLOAD_LANES = 8;

int fb_nccl_unique_id(uint8_t* out) {
  if (!out) return invalid(nullptr, "null argument");
  NcclApi& api = nccl_api();
  if (!api.ok) return invalid(nullptr, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  const ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) {
    g_err = std::string("ncclGetUniqueId: ") + api.GetErrorString(r);
    return FB_ERR_CUDA;
  }
  static_assert(sizeof(ncclUniqueId) == FB_NCCL_ID_BYTES, "unique id size");
  std::memcpy(out, &id, sizeof id);
  return FB_OK;
}

int fb_set_shard(void* handle, int32_t world, int32_t rank, const uint8_t* nccl_id) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !nccl_id) return invalid(ctx, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return invalid(ctx, "bad world / rank");
  if (ctx->uploaded || ctx->initialised) return invalid(ctx, "fb_set_shard must precede fb_upload_shards");

  NcclApi& api = nccl_api();
  if (!api.ok) return invalid(ctx, "libnccl.so.2 could not be loaded");
  const int n = ctx->n;
  ctx->world = world;
  ctx->rank = rank;
  ctx->npr = (n + world - 1) / world;
  ctx->c_lo = std::min(n, rank * ctx->npr);
  ctx->c_hi = std::min(n, ctx->c_lo + ctx->npr);
  const size_t n_pad = static_cast<size_t>(world) * ctx->npr;
  // exchange arrays padded to whole blocks (slots >= n are never consumed)
  if (dalloc(ctx, &ctx->grad, n_pad * ctx->d) || dalloc(ctx, &ctx->loss_part, n_pad * ctx->nblk) ||
      dalloc(ctx, &ctx->frob_part, n_pad * ctx->n_pairs) || dalloc(ctx, &ctx->flags, n_pad) ||
      dalloc(ctx, &ctx->idx_list, n_pad * ctx->cap) || dalloc(ctx, &ctx->val_list, n_pad * ctx->cap) ||
      dalloc(ctx, &ctx->count, n_pad) || dalloc(ctx, &ctx->rs, n_pad * (ctx->nr + 1)) ||
      dalloc(ctx, &ctx->ls_loss_part, n_pad * LS_BATCH * ctx->ls_nblk) ||
      dalloc(ctx, &ctx->local_clients, std::max(1, ctx->c_hi - ctx->c_lo)))
    return FB_ERR_CUDA;
  if (dalloc(ctx, &ctx->xcode, world)) return FB_ERR_CUDA;
  if (ctx->cfg.algorithm == FB_ALG_PP) {
    // participants by slot: B and every H_i^k on every rank (replicated
    // client state), the slot outputs exchanged each round
    const int tau = ctx->tau;
    ctx->spr = (tau + world - 1) / world;
    ctx->s_lo = std::min(tau, rank * ctx->spr);
    ctx->s_hi = std::min(tau, ctx->s_lo + ctx->spr);
    const size_t tp = static_cast<size_t>(world) * ctx->spr;
    PpX& x = ctx->ppx;
    if (dalloc(ctx, &ctx->sub_loc, std::max(1, ctx->spr)) || dalloc(ctx, &x.idx, tp * ctx->cap) ||
        dalloc(ctx, &x.val, tp * ctx->cap) || dalloc(ctx, &x.cnt, tp) ||
        dalloc(ctx, &x.rs, tp * (ctx->nr + 1)) || dalloc(ctx, &x.flags, tp) ||
        dalloc(ctx, &x.gvec, tp * ctx->d) || dalloc(ctx, &x.shift, tp) || dalloc(ctx, &x.dg, tp * ctx->d) ||
        dalloc(ctx, &x.ds, tp) || dalloc(ctx, &x.code, world) ||
        dalloc(ctx, &ctx->dgvec_all, static_cast<size_t>(tau) * ctx->d) || dalloc(ctx, &ctx->dshift_all, tau) ||
        (dense_kind(ctx) && dalloc(ctx, &x.dense, tp * static_cast<size_t>(ctx->w))))
      return FB_ERR_CUDA;
  }
  // dense kinds all-gather D every round; exact init all-gathers H_i(x0)
  if (dense_kind(ctx) && ctx->cfg.algorithm != FB_ALG_PP &&
      dalloc(ctx, &ctx->D, n_pad * static_cast<size_t>(ctx->w) + 2))
    return FB_ERR_CUDA;
  if (ctx->cfg.hessian_init == FB_INIT_EXACT && dalloc(ctx, &ctx->hest, n_pad * static_cast<size_t>(ctx->w)))
    return FB_ERR_CUDA;
  std::vector<int32_t> loc(std::max(1, ctx->c_hi - ctx->c_lo));
  for (int c = ctx->c_lo; c < ctx->c_hi; ++c) loc[c - ctx->c_lo] = c;
  CK(cudaMemcpyAsync(ctx->local_clients, loc.data(), sizeof(int32_t) * loc.size(),
                     cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof id);
  NCK(api.CommInitRank(&ctx->comm, world, id, rank));
  drop_graphs(ctx);  // the round graph is rebuilt for the sharded body
  return FB_OK;
}

int fb_bstore_kind(void* handle) {
  const Ctx* ctx = static_cast<const Ctx*>(handle);
  return ctx ? ctx->bkind : -1;
}

int fb_upload_shards(void* handle, const double* const* bmats) {
  return fb_upload_shards_ex(handle, bmats, nullptr, nullptr);
}

int fb_upload_shards_ex(void* handle, const double* const* bmats, const int32_t* n_samples,
                        const double* lam) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !bmats) return invalid(ctx, "null argument");
  const int d = ctx->d, n = ctx->n;
  // FedNL-PP keeps every client's data on every rank (participants by slot)
  const bool all = ctx->cfg.algorithm == FB_ALG_PP;
  const int up_lo = all ? 0 : ctx->c_lo, up_hi = all ? n : ctx->c_hi;
  for (int c = up_lo; c < up_hi; ++c)
    if (!bmats[c]) return invalid(ctx, "null shard pointer");
  std::vector<int32_t> nis(n, ctx->ni);
  std::vector<double> lams(n, ctx->cfg.lam);
  for (int c = 0; c < n; ++c) {
    if (n_samples) {
      if (n_samples[c] < 1 || n_samples[c] > ctx->ni)
        return invalid(ctx, "shard n_samples must be in [1, fb_config.n_samples]");
      nis[c] = n_samples[c];
    }
    if (lam) lams[c] = lam[c];
  }
  CK(cudaMemcpyAsync(ctx->ni_arr, nis.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(ctx->lam_arr, lams.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  const int ni = ctx->ni;
  const size_t bytes = static_cast<size_t>(d) * ni * sizeof(double);  // staging slot: the largest shard
  UploadPool& pool = upload_pool();
  std::lock_guard<std::mutex> guard(pool.mu);
  const int L = std::max(1, std::min(UPLOAD_LANES, n));
  if (static_cast<int>(pool.lanes.size()) < L) pool.lanes.resize(L);
  for (int l = 0; l < L; ++l) {
    UploadLane& ln = pool.lanes[l];
    if (!ln.st) {
      CK(cudaStreamCreateWithFlags(&ln.st, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) CK(cudaEventCreateWithFlags(&ln.done[b], cudaEventDisableTiming));
    }
    if (ln.cap < bytes) {
      for (int b = 0; b < 2; ++b) {
        if (ln.host[b]) cudaFreeHost(ln.host[b]);
        if (ln.dev[b]) cudaFree(ln.dev[b]);
        ln.host[b] = nullptr;
        ln.dev[b] = nullptr;
      }
      ln.cap = 0;
      for (int b = 0; b < 2; ++b) {
        CK(cudaHostAlloc(&ln.host[b], bytes, cudaHostAllocDefault));
        CK(cudaMalloc(&ln.dev[b], bytes));
      }
      ln.cap = bytes;
    }
  }
  // Bt must not be written before ctx->st's zero fills (fb_create) — already
  // synchronised there; later writers of Bt are ordered after this call.
  std::atomic<int> failed{0};
  std::string err;
  std::mutex err_mu;
  auto lane_body = [&](int l) {
    UploadLane& ln = pool.lanes[l];
    int slot = 0;
    for (int c = up_lo + l; c < up_hi && !failed.load(); c += L, slot ^= 1) {
      cudaError_t e = cudaEventSynchronize(ln.done[slot]);  // slot free again
      const size_t cb = static_cast<size_t>(d) * nis[c] * sizeof(double);
      if (e == cudaSuccess) {
        std::memcpy(ln.host[slot], bmats[c], cb);
        e = cudaMemcpyAsync(ln.dev[slot], ln.host[slot], cb, cudaMemcpyHostToDevice, ln.st);
      }
      if (e == cudaSuccess) {
        dim3 grid((ctx->ldj + 31) / 32, (d + 31) / 32);
        k_transpose_shard<<<grid, dim3(32, 8), 0, ln.st>>>(
            ln.dev[slot], ctx->Bt + static_cast<size_t>(c) * d * ctx->ldj, d, nis[c], ctx->ldj);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaEventRecord(ln.done[slot], ln.st);
      if (e != cudaSuccess) {
        std::lock_guard<std::mutex> g(err_mu);
        err = std::string("shard upload: ") + cudaGetErrorString(e);
        failed.store(1);
      }
    }
    cudaError_t e = cudaStreamSynchronize(ln.st);
    if (e != cudaSuccess) {
      std::lock_guard<std::mutex> g(err_mu);
      err = std::string("shard upload: ") + cudaGetErrorString(e);
      failed.store(1);
    }
  };
  std::vector<std::thread> workers;
  for (int l = 1; l < L; ++l) workers.emplace_back(lane_body, l);
  lane_body(0);
  for (auto& t : workers) t.join();
  if (failed.load()) {
    ctx->err = err;
    return FB_ERR_CUDA;
  }
  TRY(choose_bstore(ctx));
  ctx->uploaded = true;
  return FB_OK;
}

int fb_init_state(void* handle, const double* x0) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx) return invalid(ctx, "null argument");
  if (!ctx->uploaded) return invalid(ctx, "shards not uploaded");
  const fb_config& c = ctx->cfg;
  cudaStream_t s = ctx->st;
  const int n = ctx->n, d = ctx->d;
  DevCtl h{};
  h.master_state = mix64(c.run_seed ^ TAG_MASTER);  // derive_stream(seed, TAG_MASTER)
  CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof h, cudaMemcpyHostToDevice, s));
  if (x0) CK(cudaMemcpyAsync(ctx->x, x0, sizeof(double) * d, cudaMemcpyHostToDevice, s));
  else CK(cudaMemsetAsync(ctx->x, 0, sizeof(double) * d, s));
  CK(cudaMemsetAsync(ctx->gvec, 0, sizeof(double) * d, s));
  CK(cudaMemsetAsync(ctx->pp_shift, 0, sizeof(double), s));
  const bool lam_id = c.hessian_init == FB_INIT_LAMBDA_IDENTITY;
  dim3 gi(static_cast<unsigned>((ctx->w + 255) / 256), n + 1);
  k_init_diag<<<gi, 256, 0, s>>>(ctx->w, n, lam_id ? ctx->lam_arr : nullptr, lam_id ? c.lam : 0.0,
                                 ctx->hest, ctx->hmas);
  CKL();
  const bool pp = c.algorithm == FB_ALG_PP;
  if (c.hessian_init == FB_INIT_EXACT || pp) {
    CK(cudaMemsetAsync(ctx->flags, 0, sizeof(int32_t) * n, s));
    const bool shd = sharded(ctx) && !pp;  // PP: every rank holds every client
    const int32_t* loc = shd ? ctx->local_clients : nullptr;
    const int n_loc = shd ? ctx->c_hi - ctx->c_lo : n;
    TRY(launch_margins(ctx, s, ctx->x, loc, n_loc));
    TRY(launch_gradient(ctx, s, ctx->x, loc, n_loc));
    if (c.hessian_init == FB_INIT_EXACT) {
      // D = H - 0 = H exactly; H_i^0 = H_i(x0), master = mean (algorithms.py:207-209, 336-341)
      TRY(launch_hessian(ctx, s, loc, n_loc, ctx->zeros_w, 0, ctx->hest, nullptr));
      if (shd) TRY(gather_clients(ctx, ctx->hest, static_cast<size_t>(ctx->w), ncclFloat64, s));
      k_mean_packed<<<static_cast<unsigned>((ctx->w + 255) / 256), 256, 0, s>>>(ctx->w, n,
                                                                               ctx->hest, ctx->hmas);
      CKL();
    }
    if (pp) {
      TRY(launch_hessian(ctx, s, nullptr, n, ctx->hest, ctx->w, ctx->D, nullptr));
      k_pp_init_client<<<n, 256, 0, s>>>(d, ctx->n_pairs, ctx->hest, ctx->x, ctx->grad,
                                          ctx->frob_part, ctx->cli_shift, ctx->cli_gvec);
      CKL();
      k_pp_init_master<<<1, 256, 0, s>>>(d, n, ctx->cli_shift, ctx->cli_gvec, ctx->gvec,
                                         ctx->pp_shift);
      CKL();
    }
  }
  CK(cudaStreamSynchronize(s));
  ctx->initialised = true;
  return FB_OK;
}

int fb_run_rounds(void* handle, int32_t first_round, int32_t count, double stop_grad_norm,
                  int32_t timed, double* grad_norm, double* f_value, int32_t* ls_steps,
                  int32_t* entry_counts, double* wall_ms, int32_t* rounds_done) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx) return invalid(ctx, "null argument");
  if (!ctx->initialised) return invalid(ctx, "state not initialised");
  if (count < 0 || first_round < 0) return invalid(ctx, "bad round range");
  if (rounds_done) *rounds_done = 0;
  TRY(build_graph(ctx, timed != 0));
  cudaStream_t s = ctx->st;
  const int n = ctx->n;
  DevCtl h;
  TRY(read_status(ctx, &h));
  if (h.code == ST_STOPPED) {  // a previous call's stop: the run may continue
    h.code = 0;
    h.halt = 0;
  }
  if (h.halt) return status_to_code(h.code);
  h.stop_gn = stop_grad_norm;  // the stop rule runs on the device (k_finish / k_pp_advance)
  cudaEvent_t t0;
  CK(cudaEventCreate(&t0));
  CK(cudaEventRecord(t0, s));
  std::vector<double> kt(EV_COUNT, 0.0);
  int timed_rounds = 0;
  int done = 0;
  int rc = FB_OK;
  std::vector<double> rg(ROW_CHUNK), rf(ROW_CHUNK);
  std::vector<int32_t> rls(ROW_CHUNK), rcnt(static_cast<size_t>(ROW_CHUNK) * n);
  if (ctx->ev_ends.empty()) {
    ctx->ev_ends.resize(ROW_CHUNK);
    for (auto& e : ctx->ev_ends) CK(cudaEventCreate(&e));
  }
  if (timed && ctx->ev_pool.empty()) {  // per-kernel event slots, on first use
    ctx->ev_pool.resize(static_cast<size_t>(ROW_CHUNK) * EV_COUNT);
    for (auto& e : ctx->ev_pool) CK(cudaEventCreate(&e));
  }
  std::vector<cudaEvent_t>& ends = ctx->ev_ends;
  while (done < count && rc == FB_OK) {
    const int chunk = std::min(ROW_CHUNK, count - done);
    h.row_base = first_round + done;
    h.round = first_round + done;
    CK(cudaMemcpyAsync(ctx->ctl, &h, sizeof h, cudaMemcpyHostToDevice, s));
    // rows without an end event of their own (inside a multi-round launch)
    // get their wall time interpolated between the launch ends around them
    std::vector<char> has_end(chunk, 0);
    for (int i = 0; i < chunk;) {
      if (!timed && ctx->gexec_multi && chunk - i >= GRAPH_ROUNDS) {
        CK(cudaGraphLaunch(ctx->gexec_multi, s));
        i += GRAPH_ROUNDS;
        CK(cudaEventRecord(ends[i - 1], s));
        has_end[i - 1] = 1;
        continue;
      }
      if (timed) {
        for (int e = 0; e < EV_COUNT; ++e)
          if (ctx->ev_node[e])
            CK(cudaGraphExecEventRecordNodeSetEvent(ctx->gexec, ctx->ev_node[e],
                                                    ctx->ev_pool[static_cast<size_t>(i) * EV_COUNT + e]));
      }
      CK(cudaGraphLaunch(ctx->gexec, s));
      CK(cudaEventRecord(ends[i], s));
      has_end[i] = 1;
      ++i;
    }
    TRY(read_status(ctx, &h));
    const int completed = h.round - (first_round + done);
    CK(cudaMemcpyAsync(rg.data(), ctx->row_grad, sizeof(double) * chunk, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(rf.data(), ctx->row_f, sizeof(double) * chunk, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(rls.data(), ctx->row_ls, sizeof(int32_t) * chunk, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(rcnt.data(), ctx->row_counts, sizeof(int32_t) * chunk * n,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int take = std::min(completed, chunk);
    bool stop = false;
    for (int i = 0; i < take; ++i) {
      const int o = done + i;
      if (grad_norm) grad_norm[o] = rg[i];
      if (f_value) f_value[o] = rf[i];
      if (ls_steps) ls_steps[o] = rls[i];
      if (entry_counts)
        memcpy(entry_counts + static_cast<size_t>(o) * n, rcnt.data() + static_cast<size_t>(i) * n,
               sizeof(int32_t) * n);
      if (wall_ms) {
        int j1 = i;  // the next row with an end event (a launch's last round)
        while (!has_end[j1]) ++j1;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, t0, ends[j1]));
        if (j1 != i) {  // inside a multi-round launch: between its start and end
          const int j0 = j1 - GRAPH_ROUNDS;  // the previous launch's last row
          float ms0 = 0.f;
          if (j0 >= 0) CK(cudaEventElapsedTime(&ms0, t0, ends[j0]));
          else ms0 = o > 0 && wall_ms ? static_cast<float>(wall_ms[o - 1]) : 0.f;
          ms = ms0 + (ms - ms0) * static_cast<float>(i - j0) / static_cast<float>(GRAPH_ROUNDS);
        }
        wall_ms[o] = ms;
      }
      if (timed && ctx->ev_node[EV_START] && !h.halt) {
        const cudaEvent_t* ev = &ctx->ev_pool[static_cast<size_t>(i) * EV_COUNT];
        auto el = [&](int a, int b) {
          if (!ctx->ev_node[a] || !ctx->ev_node[b]) return 0.0;
          float v = 0.f;
          if (cudaEventElapsedTime(&v, ev[a], ev[b]) != cudaSuccess) return 0.0;
          return static_cast<double>(v);
        };
        kt[0] += el(EV_START, EV_ORACLE_END);
        kt[1] += el(EV_ORACLE_END, EV_HESS_END);
        kt[2] += el(EV_HESS_END, EV_REDUCE_END);
        kt[3] += el(EV_COMP_START, EV_COMP_END);
        kt[4] += (ctx->cfg.algorithm == FB_ALG_PP) ? el(EV_START, EV_SOLVE_END)
                                                    : el(EV_REDUCE_END, EV_SOLVE_END);
        kt[5] += el(EV_FOLD_START, EV_FOLD_END);
        kt[6] += el(EV_START, EV_END);
        ++timed_rounds;
      }
      if (stop_grad_norm >= 0.0 && rg[i] <= stop_grad_norm) {
        done += i + 1;
        stop = true;
        break;
      }
    }
    if (stop) break;
    done += take;
    if (h.code == ST_STOPPED) {  // cannot happen without a row <= stop_grad_norm
      rc = FB_ERR_CUDA;
      ctx->err = "device stop without a stopping row";
      break;
    }
    if (h.code != 0) {
      rc = status_to_code(h.code);
      break;
    }
    if (take < chunk) {
      rc = FB_ERR_CUDA;
      ctx->err = "round graph stopped without a status";
      break;
    }
  }
  cudaGetLastError();
  cudaEventDestroy(t0);
  if (rc == FB_OK && h.code == ST_STOPPED) TRY(clear_status(ctx));  // stopped, not failed
  if (timed && timed_rounds > 0) {
    fb_profile& p = ctx->prof;
    p.rounds = timed_rounds;
    p.launches_per_round = ctx->launches_per_round;
    p.ms_oracle = kt[0] / timed_rounds;
    p.ms_hessian = kt[1] / timed_rounds;
    p.ms_reduce = kt[2] / timed_rounds;
    p.ms_compress = kt[3] / timed_rounds;
    p.ms_solve = kt[4] / timed_rounds;
    p.ms_fold = kt[5] / timed_rounds;
    p.ms_round = kt[6] / timed_rounds;
  }
  if (rounds_done) *rounds_done = done;
  if (rc != FB_OK && ctx->err.empty()) ctx->err = "round failed (see fb_get_status)";
  return rc;
}

int fb_get_profile(void* handle, fb_profile* out) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !out) return invalid(ctx, "null argument");
  *out = ctx->prof;
  return FB_OK;
}

int fb_final_eval(void* handle, double* grad_norm, double* f_value) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx) return invalid(ctx, "null argument");
  cudaStream_t s = ctx->st;
  DevCtl h;
  TRY(read_status(ctx, &h));
  if (h.halt) return status_to_code(h.code);
  const bool shd = sharded(ctx);
  const int32_t* loc = shd ? ctx->local_clients : nullptr;
  const int n_loc = shd ? ctx->c_hi - ctx->c_lo : ctx->n;
  TRY(launch_margins(ctx, s, ctx->x, loc, n_loc));
  TRY(launch_gradient(ctx, s, ctx->x, loc, n_loc));
  if (shd) {
    TRY(gather_clients(ctx, ctx->grad, ctx->d, ncclFloat64, s));
    TRY(gather_clients(ctx, ctx->loss_part, ctx->nblk, ncclFloat64, s));
  }
  TRY(launch_reduce(ctx, s, ctx->x, nullptr, ctx->n, ctx->n, false, nullptr, nullptr));
  RoundScalars sc;
  CK(cudaMemcpyAsync(&sc, ctx->sc, sizeof sc, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (grad_norm) *grad_norm = sc.grad_norm;
  if (f_value) *f_value = sc.f_mean;
  return FB_OK;
}

// ---------------------------------------------------------------- state taps
#define COPY_OUT(dst, src, bytes)                                                   \
  do {                                                                              \
    CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyDeviceToHost, ctx->st));    \
    CK(cudaStreamSynchronize(ctx->st));                                             \
  } while (0)
#define COPY_IN(dst, src, bytes)                                                    \
  do {                                                                              \
    CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyHostToDevice, ctx->st));    \
    CK(cudaStreamSynchronize(ctx->st));                                             \
  } while (0)

int fb_get_x(void* handle, double* x) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !x) return invalid(ctx, "null argument");
  COPY_OUT(x, ctx->x, sizeof(double) * ctx->d);
  return FB_OK;
}
int fb_set_x(void* handle, const double* x) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !x) return invalid(ctx, "null argument");
  COPY_IN(ctx->x, x, sizeof(double) * ctx->d);
  return FB_OK;
}
int fb_get_client_hest(void* handle, int32_t c0, int32_t c1, double* out) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !out || c0 < 0 || c1 > ctx->n || c0 > c1) return invalid(ctx, "bad client range");
  COPY_OUT(out, ctx->hest + static_cast<size_t>(c0) * ctx->w, sizeof(double) * ctx->w * (c1 - c0));
  return FB_OK;
}
int fb_set_client_hest(void* handle, int32_t c0, int32_t c1, const double* in) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !in || c0 < 0 || c1 > ctx->n || c0 > c1) return invalid(ctx, "bad client range");
  COPY_IN(ctx->hest + static_cast<size_t>(c0) * ctx->w, in, sizeof(double) * ctx->w * (c1 - c0));
  return FB_OK;
}
int fb_get_master_hest(void* handle, double* out) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !out) return invalid(ctx, "null argument");
  COPY_OUT(out, ctx->hmas, sizeof(double) * ctx->w);
  return FB_OK;
}
int fb_set_master_hest(void* handle, const double* in) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !in) return invalid(ctx, "null argument");
  COPY_IN(ctx->hmas, in, sizeof(double) * ctx->w);
  return FB_OK;
}
int fb_get_pp_state(void* handle, double* shift, double* gvec, double* cli_shift,
                    double* cli_gvec) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx) return invalid(ctx, "null argument");
  if (shift) COPY_OUT(shift, ctx->pp_shift, sizeof(double));
  if (gvec) COPY_OUT(gvec, ctx->gvec, sizeof(double) * ctx->d);
  if (cli_shift) COPY_OUT(cli_shift, ctx->cli_shift, sizeof(double) * ctx->n);
  if (cli_gvec && ctx->cfg.algorithm == FB_ALG_PP)
    COPY_OUT(cli_gvec, ctx->cli_gvec, sizeof(double) * ctx->n * ctx->d);
  return FB_OK;
}
int fb_get_round_diff(void* handle, int32_t cid, double* out) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !out || cid < 0 || cid >= ctx->n) return invalid(ctx, "bad client");
  COPY_OUT(out, ctx->D + static_cast<size_t>(cid) * ctx->w, sizeof(double) * ctx->w);
  return FB_OK;
}
int fb_get_round_delta(void* handle, int32_t cid, uint32_t* idx, double* val, int32_t* count) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || cid < 0 || cid >= ctx->n) return invalid(ctx, "bad client");
  int32_t cnt = 0;
  COPY_OUT(&cnt, ctx->count + cid, sizeof(int32_t));
  if (count) *count = cnt;
  const int kind = ctx->cfg.kind;
  if (kind == FB_KIND_IDENTITY || kind == FB_KIND_NATURAL) {
    if (val && cnt > 0) COPY_OUT(val, ctx->D + static_cast<size_t>(cid) * ctx->w, sizeof(double) * ctx->w);
    return FB_OK;
  }
  if (idx && cnt > 0)
    COPY_OUT(idx, ctx->idx_list + static_cast<size_t>(cid) * ctx->cap, sizeof(uint32_t) * cnt);
  if (val && cnt > 0)
    COPY_OUT(val, ctx->val_list + static_cast<size_t>(cid) * ctx->cap, sizeof(double) * cnt);
  return FB_OK;
}
int fb_get_round_scalars(void* handle, double* out5, double* client_shift) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !out5) return invalid(ctx, "null argument");
  RoundScalars sc;
  COPY_OUT(&sc, ctx->sc, sizeof sc);
  out5[0] = sc.grad_norm;
  out5[1] = sc.f_mean;
  out5[2] = sc.shift_mean;
  out5[3] = sc.decrement;
  out5[4] = sc.xx;
  if (client_shift) COPY_OUT(client_shift, ctx->shift_cli, sizeof(double) * ctx->n);
  return FB_OK;
}

int fb_get_round_grads(void* handle, double* mean_grad, double* client_grads) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx) return invalid(ctx, "null argument");
  if (mean_grad) COPY_OUT(mean_grad, ctx->gbar, sizeof(double) * ctx->d);
  if (client_grads) COPY_OUT(client_grads, ctx->grad, sizeof(double) * ctx->d * ctx->n);
  return FB_OK;
}

// ------------------------------------------------------------- leaf ops

// flags (nonfinite | nonzero) of injected packed differences
__global__ void k_diff_flags(const double* __restrict__ D, int64_t w, int32_t* __restrict__ flags) {
  const int c = blockIdx.y;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int f = 0;
  if (t < w) {
    const double v = D[static_cast<int64_t>(c) * w + t];
    if (!isfinite(v)) f |= 1;
    if (v != 0.0) f |= 2;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(&flags[c], f);
}

int fb_compress(void* handle, const double* diffs, const uint64_t* seeds, uint32_t* idx,
                double* val, int32_t* count, int32_t* draws) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !diffs || !seeds) return invalid(ctx, "null argument");
  cudaStream_t s = ctx->st;
  TRY(clear_status(ctx));
  const int n = ctx->n;
  const int64_t w = ctx->w;
  CK(cudaMemcpyAsync(ctx->D, diffs, sizeof(double) * w * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->seeds, seeds, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(ctx->flags, 0, sizeof(int32_t) * n, s));
  k_diff_flags<<<dim3(static_cast<unsigned>((w + 255) / 256), n), 256, 0, s>>>(ctx->D, w, ctx->flags);
  CKL();
  std::vector<int32_t> fl(n);
  CK(cudaMemcpyAsync(fl.data(), ctx->flags, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int c = 0; c < n; ++c) {
    if (fl[c] & 1) {
      DevCtl h;
      TRY(read_status(ctx, &h));
      h.bad_client = c;
      h.code = ST_NONFINITE;
      h.halt = 0;
      CK(cudaMemcpy(ctx->ctl, &h, sizeof h, cudaMemcpyHostToDevice));
      ctx->err = "cannot compress a matrix with non-finite entries";
      return FB_ERR_NONFINITE;
    }
  }
  TRY(launch_compress(ctx, s, nullptr, n, ctx->seeds, nullptr, false, false));
  std::vector<int32_t> cnt(n);
  CK(cudaMemcpyAsync(cnt.data(), ctx->count, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  if (draws) CK(cudaMemcpyAsync(draws, ctx->draws, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  DevCtl h;
  TRY(read_status(ctx, &h));
  if (h.code == ST_TOPLEK_ZERO) {
    TRY(clear_status(ctx));
    ctx->err = "toplek plan needs positive total energy";
    return FB_ERR_INVALID;
  }
  if (count) memcpy(count, cnt.data(), sizeof(int32_t) * n);
  const bool dense = ctx->cfg.kind == FB_KIND_IDENTITY || ctx->cfg.kind == FB_KIND_NATURAL;
  for (int c = 0; c < n; ++c) {
    if (cnt[c] == 0) continue;
    if (dense) {
      if (val) CK(cudaMemcpyAsync(val + static_cast<size_t>(c) * w, ctx->D + static_cast<size_t>(c) * w,
                                  sizeof(double) * w, cudaMemcpyDeviceToHost, s));
    } else {
      if (idx) CK(cudaMemcpyAsync(idx + static_cast<size_t>(c) * w, ctx->idx_list + static_cast<size_t>(c) * ctx->cap,
                                  sizeof(uint32_t) * cnt[c], cudaMemcpyDeviceToHost, s));
      if (val) CK(cudaMemcpyAsync(val + static_cast<size_t>(c) * w, ctx->val_list + static_cast<size_t>(c) * ctx->cap,
                                  sizeof(double) * cnt[c], cudaMemcpyDeviceToHost, s));
    }
  }
  CK(cudaStreamSynchronize(s));
  return FB_OK;
}

int fb_oracle_eval(void* handle, const double* x, double* f, double* grad, double* hess_packed) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !x) return invalid(ctx, "null argument");
  if (!ctx->uploaded) return invalid(ctx, "shards not uploaded");
  cudaStream_t s = ctx->st;
  const int n = ctx->n, d = ctx->d;
  DevCtl h;
  TRY(read_status(ctx, &h));
  if (h.halt || h.code) TRY(clear_status(ctx));  // a previous failure's code too
  CK(cudaMemcpyAsync(ctx->x_new, x, sizeof(double) * d, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(ctx->flags, 0, sizeof(int32_t) * n, s));
  TRY(launch_margins(ctx, s, ctx->x_new, nullptr, n));
  TRY(launch_gradient(ctx, s, ctx->x_new, nullptr, n));
  if (hess_packed) TRY(launch_hessian(ctx, s, nullptr, n, ctx->zeros_w, 0, ctx->D, nullptr));
  // f via the reduction kernel without touching the row buffers or status
  k_reduce<<<reduce_grid(d), RED_THREADS, 0, s>>>(ctx->ctl, n, nullptr, n, d, ctx->ni_arr, ctx->nblk, ctx->n_pairs,
                              ctx->x_new, ctx->lam_arr, ctx->grad, ctx->loss_part, nullptr,
                              ctx->flags, ctx->gbar, ctx->f_cli, ctx->shift_cli, ctx->sc, nullptr,
                              nullptr, nullptr, 0);
  CKL();
  if (f) CK(cudaMemcpyAsync(f, ctx->f_cli, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  if (grad) CK(cudaMemcpyAsync(grad, ctx->grad, sizeof(double) * n * d, cudaMemcpyDeviceToHost, s));
  if (hess_packed)
    CK(cudaMemcpyAsync(hess_packed, ctx->D, sizeof(double) * n * ctx->w, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return FB_OK;
}

// Diagnostic: per-phase clock64 cycles of one shifted solve (rank 0, thread 0):
// [setup, A, syncA, pull, B, B-writeback, C, syncC, back-solve, back-total, -, -];
// cluster size override (0 = default).
int fb_solve_phase_cycles(void* handle, const double* h_packed, double shift, const double* rhs,
                          int32_t cluster, long long* cycles, float* ms) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !h_packed || !rhs || !cycles) return invalid(ctx, "null argument");
  cudaStream_t s = ctx->st;
  const int saved = ctx->solve_cs;
  if (cluster > 0) ctx->solve_cs = cluster;
  long long* dbg = nullptr;
  constexpr int NDBG = 16 + 64 * 16;  // phase cycles + per-panel timestamps
  CK(cudaMalloc(&dbg, NDBG * sizeof(long long)));
  CK(cudaMemset(dbg, 0, NDBG * sizeof(long long)));
  CK(cudaMemcpyAsync(ctx->D, h_packed, sizeof(double) * ctx->w, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->scalar, &shift, sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->zbuf, rhs, sizeof(double) * ctx->d, cudaMemcpyHostToDevice, s));
  const bool old = cluster > 0;
  TRY(launch_solve(ctx, s, ctx->D, ctx->scalar, ctx->zbuf, nullptr, ctx->pvec, nullptr, 2, 1, nullptr,
                   nullptr, old));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // plain timing first (no instrumentation), then the instrumented run
  float plain_ms = 0.f;
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(e0, s));
    TRY(launch_solve(ctx, s, ctx->D, ctx->scalar, ctx->zbuf, nullptr, ctx->pvec, nullptr, 2, 1,
                     rep ? dbg : nullptr, nullptr, old));
    CK(cudaEventRecord(e1, s));
    if (rep == 0) {
      CK(cudaStreamSynchronize(s));
      CK(cudaEventElapsedTime(&plain_ms, e0, e1));
    }
  }
  CK(cudaStreamSynchronize(s));
  if (ms) *ms = plain_ms;
  CK(cudaMemcpy(cycles, dbg, (cluster == 0 ? NDBG : 12) * sizeof(long long), cudaMemcpyDeviceToHost));
  cudaFree(dbg);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->solve_cs = saved;
  return FB_OK;
}

int fb_eigen_clamp(void* handle, const double* a_packed, double floor, double* out_packed,
                   double* eigvals, double* eigvecs) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !a_packed || !out_packed) return invalid(ctx, "null argument");
  cudaStream_t s = ctx->st;
  const int d = ctx->d;
  DevCtl h;
  TRY(read_status(ctx, &h));
  if (h.halt || h.code) TRY(clear_status(ctx));  // a previous failure's code too
  CK(cudaMemcpyAsync(ctx->D, a_packed, sizeof(double) * ctx->w, cudaMemcpyHostToDevice, s));
  k_eig_clamp<<<1, EIG_THREADS, eig_smem_bytes(d), s>>>(ctx->ctl, d, ctx->D, nullptr, floor, ctx->eigA,
                                                       ctx->eigV, ctx->hclamp, ctx->zbuf, 1);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  TRY(read_status(ctx, &h));
  if (h.code == ST_EIGEN) {
    ctx->err = "Jacobi did not converge in 30 sweeps";
    h.halt = 0;
    h.code = 0;
    CK(cudaMemcpy(ctx->ctl, &h, sizeof h, cudaMemcpyHostToDevice));
    return FB_ERR_EIGEN;
  }
  COPY_OUT(out_packed, ctx->hclamp, sizeof(double) * ctx->w);
  if (eigvals) COPY_OUT(eigvals, ctx->zbuf, sizeof(double) * d);
  if (eigvecs) {  // V^T rows are the eigenvectors: column-major V is V^T row-major
    COPY_OUT(eigvecs, ctx->eigV, sizeof(double) * d * d);
  }
  return FB_OK;
}

int fb_shifted_solve(void* handle, const double* h_packed, double shift, const double* rhs,
                     double* z) {
  Ctx* ctx = static_cast<Ctx*>(handle);
  if (!ctx || !h_packed || !rhs || !z) return invalid(ctx, "null argument");
  cudaStream_t s = ctx->st;
  const int d = ctx->d;
  DevCtl h;
  TRY(read_status(ctx, &h));
  if (h.halt || h.code) TRY(clear_status(ctx));  // a previous failure's code too
  CK(cudaMemcpyAsync(ctx->D, h_packed, sizeof(double) * ctx->w, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->scalar, &shift, sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(ctx->zbuf, rhs, sizeof(double) * d, cudaMemcpyHostToDevice, s));
  TRY(launch_solve(ctx, s, ctx->D, ctx->scalar, ctx->zbuf, nullptr, ctx->pvec, nullptr, 2, 1));
  CK(cudaStreamSynchronize(s));
  TRY(read_status(ctx, &h));
  if (h.code == ST_NOT_PD) {
    ctx->err = "matrix is not positive definite";
    // keep pivot info readable via fb_get_status, but un-halt the context
    h.halt = 0;
    CK(cudaMemcpy(ctx->ctl, &h, sizeof h, cudaMemcpyHostToDevice));
    return FB_ERR_NOT_PD;
  }
  COPY_OUT(z, ctx->pvec, sizeof(double) * d);
  return FB_OK;
}

// ------------------------------------------------------ context-free PRG

__global__ void k_prg_u64(uint64_t seed, int count, uint64_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = scramble(seed + static_cast<uint64_t>(i + 1) * GOLDEN);
}
__global__ void k_prg_randrange(uint64_t seed, const uint64_t* bounds, int nb, int reps,
                                uint64_t* out, uint64_t* next) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  Prg p(seed);
  for (int r = 0; r < reps; ++r) out[static_cast<int64_t>(b) * reps + r] = p.randrange(bounds[b]);
  next[b] = p.next_u64();
}
__global__ void k_prg_pshuffle(uint64_t seed, int64_t n, int k, int64_t* out, int64_t* pool) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Prg p(seed);
  for (int64_t i = 0; i < n; ++i) pool[i] = i;
  for (int i = 0; i < k; ++i) {
    const int64_t j = i + static_cast<int64_t>(p.randrange(static_cast<uint64_t>(n - i)));
    const int64_t t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
    out[i] = pool[i];
  }
}
__global__ void k_round_seeds(uint64_t run_seed, int n, int rnd, uint64_t* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) out[c] = round_seed(run_seed, c, rnd);
}

#define G_CK(call)                                                                  \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                   \
      return FB_ERR_CUDA;                                                           \
    }                                                                               \
  } while (0)

int fb_prg_u64(uint64_t seed, int32_t count, uint64_t* out) {
  if (!out || count < 0) return invalid(nullptr, "bad argument");
  uint64_t* d = nullptr;
  G_CK(cudaMalloc(&d, sizeof(uint64_t) * std::max(count, 1)));
  k_prg_u64<<<(count + 255) / 256 + 1, 256>>>(seed, count, d);
  G_CK(cudaGetLastError());
  G_CK(cudaMemcpy(out, d, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost));
  cudaFree(d);
  return FB_OK;
}
int fb_prg_randrange(uint64_t seed, const uint64_t* bounds, int32_t n_bounds, int32_t reps,
                     uint64_t* out, uint64_t* next) {
  if (!bounds || !out || !next || n_bounds < 0 || reps < 0) return invalid(nullptr, "bad argument");
  for (int i = 0; i < n_bounds; ++i)
    if (bounds[i] == 0) return invalid(nullptr, "bound must be positive");
  uint64_t *db, *dout, *dnext;
  G_CK(cudaMalloc(&db, sizeof(uint64_t) * std::max(n_bounds, 1)));
  G_CK(cudaMalloc(&dout, sizeof(uint64_t) * std::max(n_bounds * reps, 1)));
  G_CK(cudaMalloc(&dnext, sizeof(uint64_t) * std::max(n_bounds, 1)));
  G_CK(cudaMemcpy(db, bounds, sizeof(uint64_t) * n_bounds, cudaMemcpyHostToDevice));
  k_prg_randrange<<<(n_bounds + 63) / 64 + 1, 64>>>(seed, db, n_bounds, reps, dout, dnext);
  G_CK(cudaGetLastError());
  G_CK(cudaMemcpy(out, dout, sizeof(uint64_t) * n_bounds * reps, cudaMemcpyDeviceToHost));
  G_CK(cudaMemcpy(next, dnext, sizeof(uint64_t) * n_bounds, cudaMemcpyDeviceToHost));
  cudaFree(db);
  cudaFree(dout);
  cudaFree(dnext);
  return FB_OK;
}
int fb_prg_partial_shuffle(uint64_t seed, int64_t n, int32_t k, int64_t* out) {
  if (!out || k < 0 || k > n || n > (int64_t(1) << 28)) return invalid(nullptr, "bad argument");
  int64_t *dout, *dpool;
  G_CK(cudaMalloc(&dout, sizeof(int64_t) * std::max(k, 1)));
  G_CK(cudaMalloc(&dpool, sizeof(int64_t) * std::max<int64_t>(n, 1)));
  k_prg_pshuffle<<<1, 32>>>(seed, n, k, dout, dpool);
  G_CK(cudaGetLastError());
  G_CK(cudaMemcpy(out, dout, sizeof(int64_t) * k, cudaMemcpyDeviceToHost));
  cudaFree(dout);
  cudaFree(dpool);
  return FB_OK;
}
int fb_round_seeds(uint64_t run_seed, int32_t n_clients, int32_t rnd, uint64_t* out) {
  if (!out || n_clients < 0 || rnd < 0) return invalid(nullptr, "bad argument");
  uint64_t* d;
  G_CK(cudaMalloc(&d, sizeof(uint64_t) * std::max(n_clients, 1)));
  k_round_seeds<<<(n_clients + 255) / 256 + 1, 256>>>(run_seed, n_clients, rnd, d);
  G_CK(cudaGetLastError());
  G_CK(cudaMemcpy(out, d, sizeof(uint64_t) * n_clients, cudaMemcpyDeviceToHost));
  cudaFree(d);
  return FB_OK;
}

int fb_debug_counters(int32_t enable, long long* out) {
  if (out) G_CK(cudaMemcpyFromSymbol(out, g_dbg, sizeof(long long) * 32));
  if (out) G_CK(cudaMemcpyFromSymbol(out + 32, g_dbg_cta, sizeof(long long) * 1024));
  if (out) G_CK(cudaMemcpyFromSymbol(out + 32 + 1024, g_dbg_span, sizeof(long long) * 2048));
  long long zero[32] = {};
  G_CK(cudaMemcpyToSymbol(g_dbg, zero, sizeof zero));
  const int on = enable ? 1 : 0;
  G_CK(cudaMemcpyToSymbol(g_dbg_on, &on, sizeof on));
  return FB_OK;
}

int fb_debug_timeline(unsigned long long* out) {
  if (out) G_CK(cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl)));
  unsigned long long init[TL_SLOTS][2];
  for (int i = 0; i < TL_SLOTS; ++i) {
    init[i][0] = ~0ull;
    init[i][1] = 0ull;
  }
  G_CK(cudaMemcpyToSymbol(g_tl, init, sizeof init));
  return FB_OK;
}

int fb_fp64_peak(double* dmma_tflops, double* dfma_tflops) {
  return fp64_peak_measure(dmma_tflops, dfma_tflops, &g_err);
}

}  // extern "C"
