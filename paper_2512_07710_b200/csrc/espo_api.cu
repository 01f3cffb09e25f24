#include <cstdio>
#include <cstdlib>
// espo_api.cu — libespo host side: the C ABI of include/espo.h (context, validation,
// workspace, launches, NCCL). Kernels live in the k_*.cuh headers of this directory.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: no-ops unless a profiler is attached

#include "common.cuh"
#include "k_dlogits.cuh"
#include "k_rowstats.cuh"
#include "k_rowlist.cuh"
#include "k_seq.cuh"
#include "k_lmhead.cuh"
#include "k_lmhead2.cuh"
#include "k_reward.cuh"
#include "k_tpx.cuh"
#include "k_gemm.cuh"
#include "k_compact.cuh"
#include "k_fwdgrad.cuh"
#include "workspace.cuh"

#include <cublas_v2.h>
#include <cudaTypedefs.h>

using namespace espo;

// ------------------------------------------------------------------------------ NCCL
// Resolved at run time from libnccl.so.2 (the copy torch already loaded, when present),
// so a world == 1 context never needs NCCL and there is no link-time dependency.

// Host-side NVTX range around each public call (what a trainer sees on an nsys / ncu NVTX
// timeline: which ESPO call enqueued which kernels); free when no tool is attached.
struct EspoRange {
  explicit EspoRange(const char* name) { nvtxRangePushA(name); }
  ~EspoRange() { nvtxRangePop(); }
};
#define ESPO_RANGE(name) EspoRange espo_range_(name)

namespace {
typedef struct { char internal[ESPO_UNIQUE_ID_BYTES]; } nccl_uid;
typedef void* nccl_comm;
typedef int (*fn_get_uid)(nccl_uid*);
typedef int (*fn_init_rank)(nccl_comm*, int, nccl_uid, int);
typedef int (*fn_allreduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t);
typedef int (*fn_destroy)(nccl_comm);
typedef int (*fn_allgather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t);
typedef int (*fn_count)(nccl_comm, int*);
constexpr int kNcclFloat64 = 8;  // ncclFloat64
constexpr int kNcclFloat32 = 7;  // ncclFloat32
constexpr int kNcclUint8 = 1;    // ncclUint8
constexpr int kNcclSum = 0;      // ncclSum

struct NcclApi {
  void* lib = nullptr;
  fn_get_uid get_uid = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_allreduce allreduce = nullptr;
  fn_destroy destroy = nullptr;
  fn_allgather allgather = nullptr;
  fn_count count = nullptr;
  bool load() {
    if (lib) return true;
    lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return false;
    get_uid = reinterpret_cast<fn_get_uid>(dlsym(lib, "ncclGetUniqueId"));
    init_rank = reinterpret_cast<fn_init_rank>(dlsym(lib, "ncclCommInitRank"));
    allreduce = reinterpret_cast<fn_allreduce>(dlsym(lib, "ncclAllReduce"));
    destroy = reinterpret_cast<fn_destroy>(dlsym(lib, "ncclCommDestroy"));
    allgather = reinterpret_cast<fn_allgather>(dlsym(lib, "ncclAllGather"));
    count = reinterpret_cast<fn_count>(dlsym(lib, "ncclCommCount"));
    return get_uid && init_rank && allreduce && destroy && allgather;
  }
};
NcclApi g_nccl;

// ------------------------------------------------------------------------------ cuBLAS
// The LM-head backward's two plain GEMMs (dh = dz·W, dW += dzᵀ·h). Resolved at run time from
// libcublas.so.12 (the copy torch already loaded, when present); no link-time dependency.
typedef int (*fn_blas_create)(cublasHandle_t*);
typedef int (*fn_blas_destroy)(cublasHandle_t);
typedef int (*fn_blas_stream)(cublasHandle_t, cudaStream_t);
typedef int (*fn_blas_workspace)(cublasHandle_t, void*, size_t);
typedef int (*fn_blas_gemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                            const void*, const void*, cudaDataType, int, const void*, cudaDataType,
                            int, const void*, void*, cudaDataType, int, cublasComputeType_t,
                            cublasGemmAlgo_t);
struct BlasApi {
  void* lib = nullptr;
  fn_blas_create create = nullptr;
  fn_blas_destroy destroy = nullptr;
  fn_blas_stream set_stream = nullptr;
  fn_blas_workspace set_workspace = nullptr;
  fn_blas_gemm gemm = nullptr;
  bool load() {
    if (lib) return true;
    lib = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return false;
    create = reinterpret_cast<fn_blas_create>(dlsym(lib, "cublasCreate_v2"));
    destroy = reinterpret_cast<fn_blas_destroy>(dlsym(lib, "cublasDestroy_v2"));
    set_stream = reinterpret_cast<fn_blas_stream>(dlsym(lib, "cublasSetStream_v2"));
    set_workspace = reinterpret_cast<fn_blas_workspace>(dlsym(lib, "cublasSetWorkspace_v2"));
    gemm = reinterpret_cast<fn_blas_gemm>(dlsym(lib, "cublasGemmEx"));
    return create && destroy && set_stream && set_workspace && gemm;
  }
};
BlasApi g_blas;
constexpr size_t kBlasWorkspace = size_t(32) << 20;

static_assert(kRedLen == ESPO_REDUCE_LEN, "reduction vector length is part of the ABI");
enum class State { Created, Prepared, Reduced, Finalized };
}  // namespace

struct espo_ctx_s {
  espo_config cfg{};
  int device = 0, rank = 0, world = 1;
  nccl_comm comm = nullptr;     // data-parallel group (loss all-reduce)
  nccl_comm tp_comm = nullptr;  // vocabulary-parallel group (partials all-gather)
  int tp_world = 1;
  int num_sms = 148;
  Workspace ws;
  int64_t cap_T = 0;
  int cap_R = -1;
  int R = 0;
  int64_t T = 0;
  State state = State::Created;
  bool single_pass = false;  // espo_set_mask called: chunks run fwd → K3 → bwd at once
  std::map<int64_t, int64_t> covered;  // fwd chunks: begin → end
  float* hsel = nullptr;         // caller-supplied selection entropies [T] (espo_set_entropies)
  size_t hsel_cap = 0;
  std::map<int64_t, int64_t> hsel_cov;   // their chunks: begin → end
  int64_t n_hsel = 0;
  int64_t n_covered = 0;
  uint64_t launches = 0;
  int fwd_impl = 0, bwd_impl = 0;
  int blocks_per_sm = 0;
  int lmh_parts = 0;  // 0 = auto
  int factored_impl = 0;       // espo_loss_fwd_factored kernel geometry
  // compact mode: a host copy of the rollout layout and the eliminated-group flags, taken
  // asynchronously at prepare, bounds the backward grid by the rows that can carry gradient
  // (when the copy has landed; otherwise the grid covers the whole chunk)
  int64_t* h_so = nullptr;     // pinned [R+1]
  uint8_t* h_cand = nullptr;   // pinned [R]
  int h_cap = 0;
  cudaEvent_t prep_ev = nullptr;
  bool prep_ev_set = false;
  void* blocks_tok = nullptr;  // one allocation for all per-token arrays
  void* blocks_roll = nullptr; // one allocation for all per-rollout arrays
  void* blocks_scalar = nullptr;
  float* lmh_partial = nullptr;  // fused LM-head: [parts][rows] float4, grown on demand
  size_t lmh_cap = 0;
  void* rs_scratch = nullptr;    // reward reshaping hash tables, grown on demand
  int64_t rs_cap = 0;
  int lmh_bwd_rows = 8192;       // LM-head backward dz sub-chunk rows
  int lmh_2cta = 0;              // 1: CTA-pair (cta_group::2) LM-head kernels
  int lmh_bwd_gemm = 0;          // dh / dW: 0 = tcgen05 CTA-pair GEMM, 1 = cuBLAS (A/B), 2 = one CTA
  int gemm_group_m = 0;          // dh GEMM tile order: M-blocks per group (0 = auto)
  int gemm_group_n_dw = 0;       // dW GEMM tile order: N-blocks per group (0 = all)
  int lmh_compact = 1;           // LM-head backward on the rows with gradient only (k_compact.cuh)
  int lmh_impl = 0;              // LM-head fwd / dz: 0 = on the tcgen05 GEMM core (k_gemm.cuh),
                                 // 1 = the dedicated kernels (k_lmhead*.cuh)
  uint8_t* lmh_live = nullptr;   // per 256-row block liveness (fwd on the GEMM core)
  int lmh_mcast = 0;             // LM-head GEMM core on 4-CTA clusters (A multicast to two pairs)
  int lmh_split_k = 1;           // dh GEMM split-K over 2 when it has < 6 waves of tiles
  void* lmh_split = nullptr;     // its fp32 scratch [rows][d], grown on demand
  size_t lmh_split_cap = 0;
  int lmh_tile256 = 0;           // LM-head GEMM-core tiles: 0 = 256 × 512 (one accumulator),
                                 // 1 = 256 × 256 (double-buffered, epilogue overlapped)
  int lmh_group_m = 0, lmh_hints = 0;   // LM-head fwd / dz on the GEMM core: raster (0 = auto),
                                        // L2 policies
  int lmh_sync = 8 | (2 << 16);  // their soft lockstep (chunk of K-steps | slack << 16; 0 = off)
  int gemm_half_release = 1;     // CTA-pair 256 × 512 GEMMs: accumulator released in halves
  int gemm_dyn = 1;              // CTA-pair GEMMs: dynamic tile scheduler (atomic counter)
  int gemm_tma_red = 1;          // dW GEMM: epilogue adds into dW with a TMA reduce
  int* gemm_tctr = nullptr;      // its counter
  int gemm_sync_dw = -1;         // dW GEMM's own lockstep (chunk | slack << 16; −1 = as dh)
  int gemm_sync_set = 0;         // ESPO_OPT_GEMM_SYNC given (else: auto, on at d > 4096)
  size_t lmh_live_cap = 0;
  int gemm_sync_chunk = 0, gemm_sync_slack = 2;  // GEMM soft lockstep (0 = off), k_gemm.cuh
  void* gemm_sync = nullptr;     // per-wave progress counters
  size_t gemm_sync_cap = 0;
  void* lmh_cmp = nullptr;       // row list, counts, gathered h rows and records, grown on demand
  size_t lmh_cmp_cap = 0;
  int gemm_hints_dh = -1, gemm_hints_dw = -1;   // L2 policies of the two GEMMs (−1 = auto)
  void* lmh_dz = nullptr;        // [lmh_bwd_rows][round_up(V, 256)] bf16, grown on demand
  size_t lmh_dz_cap = 0;
  cublasHandle_t blas = nullptr;
  void* blas_ws = nullptr;
  // vocabulary-parallel exchange over peer memory (k_tpx.cuh)
  void* x_buf = nullptr;              // this rank's exchange buffer
  int64_t x_cap = 0;                  // rows per (slot, rank) block
  int x_world = 0;                    // tp_world the buffer was sized for
  bool tp_p2p = false;                // connected
  int tp_rank = 0;
  uint8_t** d_xpeer = nullptr;        // device [tp_world]: exchange bases of all ranks
  float4** d_xgath = nullptr;         // device [tp_world]: their partial regions
  std::vector<void*> x_opened;        // IPC-mapped peer buffers (closed at destroy)
  uint32_t x_send_epoch = 0, x_recv_epoch = 0;
  int64_t peer_timeout_ms = 120000;   // bound on every peer-memory wait (ESPO_OPT_PEER_TIMEOUT_MS)
  // context parallelism (rollouts split across CP ranks by token blocks)
  int cp_rank = 0, cp_world = 1;
  nccl_comm cp_comm = nullptr;        // nullptr with cp_world > 1: same-device emulation
  bool cp_gathered = false;           // espo_cp_gather_local ran for this step
};

namespace {
inline cudaStream_t S(espo_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

espo_status cuda_status(cudaError_t e, int line = 0) {
  if (e != cudaSuccess && std::getenv("ESPO_DEBUG"))     // diagnostics only: which call failed
    std::fprintf(stderr, "[libespo] espo_api.cu:%d: %s (%s)\n", line, cudaGetErrorName(e),
                 cudaGetErrorString(e));
  return e == cudaSuccess ? ESPO_OK
                          : (e == cudaErrorMemoryAllocation ? ESPO_ERR_OUT_OF_MEMORY : ESPO_ERR_CUDA);
}

#define ESPO_CUDA(x)                                  \
  do {                                                \
    cudaError_t e_ = (x);                             \
    if (e_ != cudaSuccess) return cuda_status(e_, __LINE__); \
  } while (0)

#define ESPO_LAUNCHED(ctx)                                   \
  do {                                                       \
    (ctx)->launches++;                                       \
    cudaError_t e_ = cudaGetLastError();                     \
    if (e_ != cudaSuccess) return cuda_status(e_, __LINE__); \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
size_t dsize(int dt) { return dt == ESPO_BF16 ? 2 : 4; }
size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

espo_status validate_config(const espo_config& c) {
  if (c.vocab < 2) return ESPO_ERR_INVALID_ARGUMENT;
  if (c.n_buckets < 1 || c.n_buckets > ESPO_MAX_BUCKETS) return ESPO_ERR_INVALID_ARGUMENT;
  if (c.split_den <= 0 || c.split_num < 0 || c.split_num > c.split_den) return ESPO_ERR_INVALID_ARGUMENT;
  if (c.partition < 0 || c.partition > 2 || c.ratio_mode < 0 || c.ratio_mode > 1 || c.norm < 0 ||
      c.norm > 1)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (!(c.alpha >= 0.f) || !(c.eps_min >= 0.f) || !(c.adv_eps >= 0.0) || !(c.zv_var_eps >= 0.0) ||
      !(c.logit_scale > 0.f) || !std::isfinite(c.logit_scale) || !(c.log_ratio_clamp >= 0.f))
    return ESPO_ERR_INVALID_ARGUMENT;
  if ((c.logits_dtype != ESPO_F32 && c.logits_dtype != ESPO_BF16) ||
      (c.grad_dtype != ESPO_F32 && c.grad_dtype != ESPO_BF16))
    return ESPO_ERR_INVALID_ARGUMENT;
  if (c.vocab_local < 0 || (c.vocab_local > 0 && (c.vocab_begin < 0 ||
                                                   int64_t(c.vocab_begin) + c.vocab_local > c.vocab)))
    return ESPO_ERR_INVALID_ARGUMENT;
  if (c.zv_mode < 0 || c.zv_mode > 1 || !(c.zvp_beta >= 0.f) || !std::isfinite(c.zvp_beta) ||
      !std::isfinite(c.zvp_threshold))
    return ESPO_ERR_INVALID_ARGUMENT;
  return ESPO_OK;
}

espo_status ensure_workspace(espo_ctx_t c, int R, int64_t T) {
  if (T > c->cap_T) {
    if (c->blocks_tok) cudaFree(c->blocks_tok);
    c->blocks_tok = nullptr;
    const int64_t cap = std::max<int64_t>(T, 1);
    // 6 f32 + 2 i32 + 3 u8 arrays, each 256-byte aligned
    const size_t a4 = round_up(size_t(cap) * 4, 256), a1 = round_up(size_t(cap), 256);
    const size_t a32 = round_up(size_t(cap) * 32, 256);
    const bool sharded = c->cfg.vocab_local > 0;
    const size_t a16 = sharded ? round_up(size_t(cap) * 16, 256) : 0;
    const size_t agath = c->tp_comm ? round_up(size_t(cap) * 16 * c->tp_world, 256) : 0;
    ESPO_CUDA(cudaMalloc(&c->blocks_tok, 9 * a4 + 4 * a1 + a32 + a16 + agath));
    char* p = static_cast<char*>(c->blocks_tok);
    auto take = [&](size_t n) { char* r = p; p += n; return r; };
    c->ws.lse = reinterpret_cast<float*>(take(a4));
    c->ws.lp = reinterpret_cast<float*>(take(a4));
    c->ws.H = reinterpret_cast<float*>(take(a4));
    c->ws.q = reinterpret_cast<float*>(take(a4));
    c->ws.old = reinterpret_cast<float*>(take(a4));
    c->ws.coef = reinterpret_cast<float*>(take(a4));
    c->ws.y = reinterpret_cast<int32_t*>(take(a4));
    c->ws.row_seq = reinterpret_cast<int32_t*>(take(a4));
    c->ws.flag = reinterpret_cast<uint8_t*>(take(a1));
    c->ws.bucket = reinterpret_cast<uint8_t*>(take(a1));
    c->ws.clip = reinterpret_cast<uint8_t*>(take(a1));
    c->ws.pmask = reinterpret_cast<uint8_t*>(take(a1));
    c->ws.list = take(a32);
    c->ws.zlist = reinterpret_cast<int32_t*>(take(a4));
    c->ws.partial = sharded ? reinterpret_cast<float*>(take(a16)) : nullptr;
    c->ws.gathered = c->tp_comm ? reinterpret_cast<float*>(take(agath)) : nullptr;
    c->cap_T = cap;
  }
  if (R > c->cap_R) {
    if (c->blocks_roll) cudaFree(c->blocks_roll);
    c->blocks_roll = nullptr;
    const int cap = std::max(R, 1);
    const size_t a8 = round_up(size_t(cap + 1) * 8, 256), a1 = round_up(size_t(cap), 256);
    const size_t a4 = round_up(size_t(cap) * 4, 256);
    const size_t ath = round_up(size_t(cap) * (kMaxK - 1) * 4, 256);
    const size_t ared = round_up(size_t(cap) * kRedLen * 8, 256);
    ESPO_CUDA(cudaMalloc(&c->blocks_roll, 3 * a8 + 4 * a1 + a4 + ath + ared));
    char* p = static_cast<char*>(c->blocks_roll);
    auto take = [&](size_t n) { char* r = p; p += n; return r; };
    c->ws.seq_off = reinterpret_cast<int64_t*>(take(a8));
    c->ws.adv = reinterpret_cast<double*>(take(a8));
    c->ws.J = reinterpret_cast<double*>(take(a8));
    c->ws.cand = reinterpret_cast<uint8_t*>(take(a1));
    c->ws.zsign = reinterpret_cast<int8_t*>(take(a1));
    c->ws.ghead = reinterpret_cast<uint8_t*>(take(a1));
    c->ws.active = reinterpret_cast<uint8_t*>(take(a1));
    c->ws.nb = reinterpret_cast<int32_t*>(take(a4));
    c->ws.theta = reinterpret_cast<float*>(take(ath));
    c->ws.red_r = reinterpret_cast<double*>(take(ared));
    c->cap_R = cap;
  }
  return ESPO_OK;
}

int grid_for(espo_ctx_t c, const void* kernel, int threads) {
  int per_sm = c->blocks_per_sm;
  if (per_sm <= 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0) != cudaSuccess ||
        occ <= 0)
      occ = 1;
    per_sm = occ;
  }
  return per_sm * c->num_sms;
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

void espo_config_default(espo_config* cfg, int32_t vocab) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->vocab = vocab;
  cfg->alpha = 0.4f;
  cfg->eps_min = 0.01f;
  cfg->n_buckets = 2;
  cfg->split_num = 4;
  cfg->split_den = 5;
  cfg->partition = ESPO_PART_QUANTILE;
  cfg->ratio_mode = ESPO_RATIO_GSPO_TOKEN;
  cfg->norm = ESPO_NORM_SEQ;
  cfg->std_unbiased = 0;
  cfg->adv_eps = 1e-6;
  cfg->zv_var_eps = 0.0;
  cfg->logit_scale = 1.0f;
  cfg->log_ratio_clamp = 20.0f;
  cfg->logits_dtype = ESPO_BF16;
  cfg->grad_dtype = ESPO_BF16;
  cfg->zero_fill_inactive_rows = 1;
  cfg->zv_mode = ESPO_ZV_MASK;
  cfg->zvp_beta = 0.05f;
  cfg->zvp_threshold = 0.5f;
}

const char* espo_status_string(espo_status s) {
  switch (s) {
    case ESPO_OK: return "ESPO_OK";
    case ESPO_ERR_INVALID_ARGUMENT: return "ESPO_ERR_INVALID_ARGUMENT";
    case ESPO_ERR_ALIGNMENT: return "ESPO_ERR_ALIGNMENT";
    case ESPO_ERR_GROUPS_NOT_CONTIGUOUS: return "ESPO_ERR_GROUPS_NOT_CONTIGUOUS";
    case ESPO_ERR_BAD_STATE: return "ESPO_ERR_BAD_STATE";
    case ESPO_ERR_NONFINITE_INPUT: return "ESPO_ERR_NONFINITE_INPUT";
    case ESPO_ERR_TOKEN_OUT_OF_RANGE: return "ESPO_ERR_TOKEN_OUT_OF_RANGE";
    case ESPO_ERR_OUT_OF_MEMORY: return "ESPO_ERR_OUT_OF_MEMORY";
    case ESPO_ERR_CUDA: return "ESPO_ERR_CUDA";
    case ESPO_ERR_NCCL: return "ESPO_ERR_NCCL";
    case ESPO_ERR_UNSUPPORTED: return "ESPO_ERR_UNSUPPORTED";
    case ESPO_ERR_BLAS: return "ESPO_ERR_BLAS";
    case ESPO_ERR_PEER_TIMEOUT: return "ESPO_ERR_PEER_TIMEOUT";
  }
  return "ESPO_ERR_UNKNOWN";
}

espo_status espo_get_unique_id(void* out_id) {
  if (!out_id) return ESPO_ERR_INVALID_ARGUMENT;
  if (!g_nccl.load()) return ESPO_ERR_NCCL;
  nccl_uid id;
  if (g_nccl.get_uid(&id) != 0) return ESPO_ERR_NCCL;
  std::memcpy(out_id, &id, sizeof(id));
  return ESPO_OK;
}

espo_status espo_create(const espo_config* cfg, const void* nccl_unique_id, int32_t rank,
                        int32_t world, int32_t cuda_device, espo_ctx_t* out) {
  ESPO_RANGE("espo_create");
  if (!cfg || !out) return ESPO_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return ESPO_ERR_INVALID_ARGUMENT;
  // world > 1 needs the NCCL id; world == 1 may pass one too (a one-rank communicator: the
  // collective code path runs, e.g. to validate the NCCL plumbing on a single GPU)
  if (world > 1 && nccl_unique_id == nullptr) return ESPO_ERR_INVALID_ARGUMENT;
  espo_status st = validate_config(*cfg);
  if (st != ESPO_OK) return st;
  int ndev = 0;
  ESPO_CUDA(cudaGetDeviceCount(&ndev));
  if (cuda_device < 0 || cuda_device >= ndev) return ESPO_ERR_INVALID_ARGUMENT;
  DevGuard g(cuda_device);
  espo_ctx_t c = new (std::nothrow) espo_ctx_s();
  if (!c) return ESPO_ERR_OUT_OF_MEMORY;
  c->cfg = *cfg;
  c->device = cuda_device;
  c->rank = rank;
  c->world = world;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  cudaError_t e = cudaMalloc(&c->blocks_scalar, 1024);
  if (e != cudaSuccess) {
    delete c;
    return cuda_status(e);
  }
  char* p = static_cast<char*>(c->blocks_scalar);
  c->ws.red = reinterpret_cast<double*>(p);
  c->ws.bwd_scale = reinterpret_cast<float*>(p + 512);
  c->ws.dpre = reinterpret_cast<double*>(p + 256);
  c->ws.err = reinterpret_cast<int*>(p + 768);
  c->ws.count = reinterpret_cast<int*>(p + 896);
  cudaMemset(c->blocks_scalar, 0, 1024);
  if (nccl_unique_id) {
    if (!g_nccl.load()) {
      espo_destroy(c);
      return ESPO_ERR_NCCL;
    }
    nccl_uid id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    if (g_nccl.init_rank(&c->comm, world, id, rank) != 0) {
      c->comm = nullptr;
      espo_destroy(c);
      return ESPO_ERR_NCCL;
    }
  }
  *out = c;
  return ESPO_OK;
}

espo_status espo_destroy(espo_ctx_t c) {
  ESPO_RANGE("espo_destroy");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  {
    DevGuard g(c->device);
    cudaDeviceSynchronize();
    if (c->comm) g_nccl.destroy(c->comm);
    if (c->tp_comm) g_nccl.destroy(c->tp_comm);
    if (c->cp_comm) g_nccl.destroy(c->cp_comm);
    if (c->blocks_tok) cudaFree(c->blocks_tok);
    if (c->blocks_roll) cudaFree(c->blocks_roll);
    if (c->blocks_scalar) cudaFree(c->blocks_scalar);
    if (c->lmh_partial) cudaFree(c->lmh_partial);
    if (c->rs_scratch) cudaFree(c->rs_scratch);
    if (c->lmh_dz) cudaFree(c->lmh_dz);
    if (c->lmh_cmp) cudaFree(c->lmh_cmp);
    if (c->lmh_split) cudaFree(c->lmh_split);
    if (c->hsel) cudaFree(c->hsel);
    if (c->lmh_live) cudaFree(c->lmh_live);
    if (c->gemm_sync) cudaFree(c->gemm_sync);
    if (c->gemm_tctr) cudaFree(c->gemm_tctr);
    if (c->blas) g_blas.destroy(c->blas);
    if (c->blas_ws) cudaFree(c->blas_ws);
    for (void* q : c->x_opened) cudaIpcCloseMemHandle(q);
    if (c->d_xpeer) cudaFree(c->d_xpeer);
    if (c->x_buf) cudaFree(c->x_buf);
    if (c->h_so) cudaFreeHost(c->h_so);
    if (c->h_cand) cudaFreeHost(c->h_cand);
    if (c->prep_ev) cudaEventDestroy(c->prep_ev);
  }
  delete c;
  return ESPO_OK;
}

espo_status espo_set_option(espo_ctx_t c, int32_t option, int64_t value) {
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  switch (option) {
    case ESPO_OPT_FWD_IMPL:
      if (value < 0 || value > 11) return ESPO_ERR_INVALID_ARGUMENT;
      c->fwd_impl = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_BWD_IMPL:
      if (value < 0 || value > 11) return ESPO_ERR_INVALID_ARGUMENT;
      c->bwd_impl = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_BLOCKS_PER_SM:
      if (value < 0 || value > 32) return ESPO_ERR_INVALID_ARGUMENT;
      c->blocks_per_sm = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_LMHEAD_PARTS:
      if (value < 0 || value > 64) return ESPO_ERR_INVALID_ARGUMENT;
      c->lmh_parts = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_LMHEAD_2CTA:
      if (value < 0 || value > 1) return ESPO_ERR_INVALID_ARGUMENT;
      c->lmh_2cta = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_FACTORED_IMPL:
      if (value < 0 || value > 6) return ESPO_ERR_INVALID_ARGUMENT;
      c->factored_impl = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_LMHEAD_BWD_GEMM:
      if (value < 0 || value > 7) return ESPO_ERR_INVALID_ARGUMENT;
      c->lmh_bwd_gemm = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_GEMM_HINTS:     // low 8 bits: dh, next 8 bits: dW (each A | B<<2 | C<<4); −1 auto
      if (value < -1 || value > 0xFFFF) return ESPO_ERR_INVALID_ARGUMENT;
      c->gemm_hints_dh = value < 0 ? -1 : int(value & 0xFF);
      c->gemm_hints_dw = value < 0 ? -1 : int((value >> 8) & 0xFF);
      return ESPO_OK;
    case ESPO_OPT_GEMM_SYNC: {    // chunk (K-steps) | slack << 16 (dh and dW); bits 32+: the
                                  // same for dW alone (0 = as dh); 0 = off
      if (value == -1) {          // back to the automatic choice
        c->gemm_sync_chunk = 0;
        c->gemm_sync_slack = 2;
        c->gemm_sync_dw = -1;
        c->gemm_sync_set = 0;
        return ESPO_OK;
      }
      const int64_t lo = value & 0xFFFFFFFFll, hi = value >> 32;
      if (value < 0 || (lo & 0xFFFF) > 4096 || (lo >> 16) > 64 || (hi & 0xFFFF) > 4096 ||
          (hi >> 16) > 64)
        return ESPO_ERR_INVALID_ARGUMENT;
      c->gemm_sync_chunk = int(lo & 0xFFFF);
      c->gemm_sync_slack = (lo >> 16) ? int(lo >> 16) : 2;
      c->gemm_sync_dw = hi ? int((hi & 0xFFFF) | ((hi >> 16 ? hi >> 16 : 2) << 16)) : -1;
      c->gemm_sync_set = 1;
      return ESPO_OK;
    }
    case ESPO_OPT_LMHEAD_RASTER:  // bits 0-15 group_m (0 = 8; negative = N-groups), 16-23 hints
      if (value < 0 || (value & 0xFFFF) > 1024) return ESPO_ERR_INVALID_ARGUMENT;
      c->lmh_group_m = int(value & 0xFFFF);
      c->lmh_hints = int((value >> 16) & 0xFF);
      c->lmh_tile256 = int((value >> 24) & 1);
      c->lmh_mcast = int((value >> 25) & 1);
      c->lmh_split_k = int(((value >> 26) & 1) ^ 1);   // bit 26: no split-K for dh
      c->lmh_sync = ((value >> 27) & 1) ? 0 : 8 | (2 << 16);   // bit 27: no lockstep
      c->gemm_half_release = int(((value >> 28) & 1) ^ 1);    // bit 28: whole-accumulator release
      c->gemm_dyn = int(((value >> 29) & 1) ^ 1);             // bit 29: static round robin
      c->gemm_tma_red = int(((value >> 30) & 1) ^ 1);         // bit 30: dW read-add-write on the SMs
      return ESPO_OK;
    case ESPO_OPT_LMHEAD_IMPL:
      if (value < 0 || value > 1) return ESPO_ERR_INVALID_ARGUMENT;
      c->lmh_impl = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_LMHEAD_COMPACT:
      if (value < 0 || value > 1) return ESPO_ERR_INVALID_ARGUMENT;
      c->lmh_compact = static_cast<int>(value);
      return ESPO_OK;
    case ESPO_OPT_GEMM_GROUP_M:   // bits 0-15: dh M-groups; bits 16-31: dW N-groups (0 = auto)
      if (value < 0 || (value & 0xFFFF) > 1024 || (value >> 16) > 1024) return ESPO_ERR_INVALID_ARGUMENT;
      c->gemm_group_m = static_cast<int>(value & 0xFFFF);
      c->gemm_group_n_dw = static_cast<int>(value >> 16);
      return ESPO_OK;
    case ESPO_OPT_PEER_TIMEOUT_MS:
      if (value < 1 || value > int64_t(24) * 3600 * 1000) return ESPO_ERR_INVALID_ARGUMENT;
      c->peer_timeout_ms = value;
      return ESPO_OK;
    case ESPO_OPT_LMHEAD_BWD_ROWS:
      if (value < 0 || value > (1 << 20) || value % kLmBM) return ESPO_ERR_INVALID_ARGUMENT;
      c->lmh_bwd_rows = value ? static_cast<int>(value) : 8192;
      return ESPO_OK;
  }
  return ESPO_ERR_INVALID_ARGUMENT;
}

uint64_t espo_launch_count(espo_ctx_t c) { return c ? c->launches : 0; }

int32_t espo_comm_size(espo_ctx_t c) {
  if (!c) return -1;
  if (!c->comm) return 1;
  int n = -1;
  if (!g_nccl.count || g_nccl.count(c->comm, &n) != 0) return -1;
  return n;
}

espo_status espo_prepare(espo_ctx_t c, const float* rewards, const int32_t* group_ids,
                         const int64_t* seq_offsets, int32_t n_rollouts, int64_t n_tokens,
                         float* adv_out, uint8_t* zv_out, espo_stream_t stream) {
  ESPO_RANGE("espo_prepare");
  if (!c || !rewards || !group_ids || !seq_offsets) return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rollouts < 0 || n_tokens < 0 || n_tokens > (int64_t(1) << 40))
    return ESPO_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  // CP: the per-token arrays hold cp_world equal blocks (in-place all-gather at finalize)
  const int64_t tb = (n_tokens + c->cp_world - 1) / c->cp_world;
  espo_status st = ensure_workspace(c, n_rollouts, std::max<int64_t>(n_tokens, tb * c->cp_world));
  if (st != ESPO_OK) return st;
  cudaStream_t s = S(stream);
  ESPO_CUDA(cudaMemsetAsync(c->ws.err, 0, sizeof(int), s));
  c->R = n_rollouts;
  c->T = n_tokens;
  c->covered.clear();
  c->n_covered = 0;
  c->hsel_cov.clear();
  c->n_hsel = 0;
  c->single_pass = false;
  c->cp_gathered = false;
  PrepParams p;
  p.rewards = rewards;
  p.group_ids = group_ids;
  p.seq_offsets = seq_offsets;
  p.R = n_rollouts;
  p.T = n_tokens;
  p.std_unbiased = c->cfg.std_unbiased;
  p.adv_eps = c->cfg.adv_eps;
  p.zv_var_eps = c->cfg.zv_var_eps;
  p.zv_mode = c->cfg.zv_mode;
  p.zvp_threshold = c->cfg.zvp_threshold;
  p.adv_out = adv_out;
  p.zv_out = zv_out;
  p.ws = c->ws;
  k_prepare_groups<<<(n_rollouts + 1 + 255) / 256, 256, 0, s>>>(p);
  ESPO_LAUNCHED(c);
  if (n_rollouts > 0) {
    k_row_seq<<<n_rollouts, 256, 0, s>>>(c->ws, n_rollouts);
    ESPO_LAUNCHED(c);
  }
  c->prep_ev_set = false;
  // under stream capture the host copy would become a graph node whose landing the host
  // cannot observe at capture time: skip it (the backward grid then covers whole chunks)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  ESPO_CUDA(cudaStreamIsCapturing(s, &cap));
  if (!c->cfg.zero_fill_inactive_rows && n_rollouts > 0 && cap == cudaStreamCaptureStatusNone) {
    if (n_rollouts > c->h_cap) {
      if (c->h_so) cudaFreeHost(c->h_so);
      if (c->h_cand) cudaFreeHost(c->h_cand);
      c->h_so = nullptr;
      c->h_cand = nullptr;
      c->h_cap = 0;
      ESPO_CUDA(cudaMallocHost(&c->h_so, size_t(n_rollouts + 1) * sizeof(int64_t)));
      ESPO_CUDA(cudaMallocHost(&c->h_cand, size_t(n_rollouts)));
      c->h_cap = n_rollouts;
    }
    if (!c->prep_ev) ESPO_CUDA(cudaEventCreateWithFlags(&c->prep_ev, cudaEventDisableTiming));
    ESPO_CUDA(cudaMemcpyAsync(c->h_so, seq_offsets, size_t(n_rollouts + 1) * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, s));
    ESPO_CUDA(cudaMemcpyAsync(c->h_cand, c->ws.cand, size_t(n_rollouts), cudaMemcpyDeviceToHost, s));
    ESPO_CUDA(cudaEventRecord(c->prep_ev, s));
    c->prep_ev_set = true;
  }
  c->state = State::Prepared;
  return ESPO_OK;
}

}  // extern "C"

namespace {
// vocabulary columns held by this context: [v0, v0 + Vl)
inline int shard_begin(espo_ctx_t c) { return c->cfg.vocab_local > 0 ? c->cfg.vocab_begin : 0; }
inline int shard_width(espo_ctx_t c) {
  return c->cfg.vocab_local > 0 ? c->cfg.vocab_local : c->cfg.vocab;
}

espo_status check_fwd_args(espo_ctx_t c, const void* logits, int64_t ld, const int32_t* tokens,
                           const float* old_logp, int64_t row_begin, int64_t n_rows,
                           bool single_pass_call = false) {
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  // single-pass mode admits only espo_loss_fwd_bwd; the other modes never admit it
  if (c->state != State::Prepared || c->single_pass != single_pass_call) return ESPO_ERR_BAD_STATE;
  if (n_rows < 0 || n_rows > INT32_MAX || row_begin < 0 || row_begin + n_rows > c->T)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rows == 0) return ESPO_OK;
  if (!logits || !tokens || !old_logp) return ESPO_ERR_INVALID_ARGUMENT;
  const size_t es = dsize(c->cfg.logits_dtype);
  if (ld < shard_width(c)) return ESPO_ERR_INVALID_ARGUMENT;
  if (!aligned16(logits) || (size_t(ld) * es) % 16 != 0) return ESPO_ERR_ALIGNMENT;
  return ESPO_OK;
}

// context parallelism: CP rank k owns token rows [k·Tb, min(T, (k+1)·Tb)), Tb = ⌈T / cp⌉
inline int64_t cp_block(const espo_ctx_s* c) { return (c->T + c->cp_world - 1) / c->cp_world; }
inline int64_t cp_lo(const espo_ctx_s* c) { return std::min(c->T, c->cp_rank * cp_block(c)); }
inline int64_t cp_hi(const espo_ctx_s* c) { return std::min(c->T, (c->cp_rank + 1) * cp_block(c)); }

espo_status check_coverage(espo_ctx_t c, int64_t b, int64_t e) {
  if (c->cp_world > 1 && (b < cp_lo(c) || e > cp_hi(c))) return ESPO_ERR_INVALID_ARGUMENT;
  auto it = c->covered.upper_bound(b);
  if (it != c->covered.begin()) {
    auto pv = std::prev(it);
    if (pv->second > b) return ESPO_ERR_BAD_STATE;
  }
  if (it != c->covered.end() && it->first < e) return ESPO_ERR_BAD_STATE;
  return ESPO_OK;
}

espo_status launch_combine(espo_ctx_t c, const float* partials, int n_shards, int64_t row_begin,
                           int64_t n_rows, cudaStream_t s);

// K2 (+ its row-list pre-pass) over one chunk; writes statistics, or partials if `partial`.
espo_status launch_sweep_fwd(espo_ctx_t c, const void* logits, int64_t ld, const int32_t* tokens,
                             const float* old_logp, const uint8_t* mask, int64_t row_begin,
                             int64_t n_rows, float* partial, cudaStream_t s,
                             float4* const* xbase = nullptr, int nx = 0, int64_t xoff = 0) {
  FwdParams p;
  p.xbase = xbase;
  p.nx = nx;
  p.xoff = xoff;
  p.logits = logits;
  p.ld = ld;
  p.tokens = tokens;
  p.old_logp = old_logp;
  p.mask = mask;
  p.row_begin = row_begin;
  p.n_rows = n_rows;
  p.V = shard_width(c);
  p.lam_log2e = c->cfg.logit_scale * kLog2e;
  p.partial = partial;
  p.ws = c->ws;
  const int V = c->cfg.vocab, v0 = shard_begin(c);
  const bool bf = c->cfg.logits_dtype == ESPO_BF16;
  FwdRec* list = static_cast<FwdRec*>(c->ws.list);
  ESPO_CUDA(cudaMemsetAsync(c->ws.count, 0, 2 * sizeof(int), s));
  const int pre_grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  if (bf)
    k_fwd_rows<__nv_bfloat16><<<pre_grid, 256, 0, s>>>(logits, ld, tokens, old_logp, mask, row_begin,
                                                       n_rows, V, v0, p.V, p.lam_log2e, c->ws, list,
                                                       c->ws.count);
  else
    k_fwd_rows<float><<<pre_grid, 256, 0, s>>>(logits, ld, tokens, old_logp, mask, row_begin, n_rows,
                                               V, v0, p.V, p.lam_log2e, c->ws, list, c->ws.count);
  ESPO_LAUNCHED(c);
  if (c->fwd_impl >= 9 && c->fwd_impl <= 11 && partial == nullptr && nx == 0) {
    // tiled: (listed row, 32 KB tile) blocks → per-tile partials → k_fwd_combine
    const int epv = bf ? 8 : 4;
    const int ntiles = (((p.V + epv - 1) / epv) + 256 * 8 - 1) / (256 * 8);
    const int64_t grid = n_rows * int64_t(ntiles);
    if (grid > INT32_MAX) return ESPO_ERR_INVALID_ARGUMENT;
    const size_t need = size_t(ntiles) * size_t(n_rows) * 16;
    if (need > c->lmh_cap) {
      if (c->lmh_partial) cudaFree(c->lmh_partial);
      c->lmh_partial = nullptr;
      c->lmh_cap = 0;
      ESPO_CUDA(cudaMalloc(&c->lmh_partial, need));
      c->lmh_cap = need;
    }
    float4* part = reinterpret_cast<float4*>(c->lmh_partial);
#define ESPO_FTILE(MB)                                                                                        \
    if (bf) k_rowstats_tile<__nv_bfloat16, 8, MB><<<unsigned(grid), 256, 0, s>>>(p, list, c->ws.count, ntiles, part); \
    else k_rowstats_tile<float, 8, MB><<<unsigned(grid), 256, 0, s>>>(p, list, c->ws.count, ntiles, part);
    if (c->fwd_impl == 9) { ESPO_FTILE(4) } else if (c->fwd_impl == 10) { ESPO_FTILE(3) } else { ESPO_FTILE(2) }
#undef ESPO_FTILE
    ESPO_LAUNCHED(c);
    return launch_combine(c, c->lmh_partial, ntiles, row_begin, n_rows, s);
  }
  if (c->fwd_impl == 1) {
    if (bf) {
      auto k = k_rowstats_ldg<__nv_bfloat16, 8>;
      k<<<grid_for(c, (const void*)k, 256), 256, 0, s>>>(p, list, c->ws.count);
    } else {
      auto k = k_rowstats_ldg<float, 8>;
      k<<<grid_for(c, (const void*)k, 256), 256, 0, s>>>(p, list, c->ws.count);
    }
  } else {
    cudaError_t le = bf ? launch_rowstats_tma<__nv_bfloat16>(p, list, c->ws.count, c->num_sms, c->blocks_per_sm, c->fwd_impl, s)
                        : launch_rowstats_tma<float>(p, list, c->ws.count, c->num_sms, c->blocks_per_sm, c->fwd_impl, s);
    if (le != cudaSuccess) return cuda_status(le);
  }
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

espo_status launch_combine(espo_ctx_t c, const float* partials, int n_shards, int64_t row_begin,
                           int64_t n_rows, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  k_fwd_combine<<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(partials), n_shards, row_begin,
                                     n_rows, c->ws);
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

TpxParams tpx_params(espo_ctx_t c, uint32_t epoch) {
  TpxParams x;
  x.peer = c->d_xpeer;
  x.local = static_cast<uint8_t*>(c->x_buf);
  x.tp_rank = c->tp_rank;
  x.tp_world = c->x_world;
  x.cap = c->x_cap;
  x.epoch = epoch;
  x.slot = int(epoch & 1u);
  x.timeout_ns = uint64_t(c->peer_timeout_ms) * 1000000ull;
  return x;
}

// peer-memory TP, first half: slot free → fused sweep (partials stored to every rank) → signal
espo_status p2p_send(espo_ctx_t c, const void* logits, int64_t ld, const int32_t* tokens,
                     const float* old_logp, const uint8_t* mask, int64_t row_begin,
                     int64_t n_rows, cudaStream_t s) {
  const TpxParams x = tpx_params(c, ++c->x_send_epoch);
  k_tpx_wait_consumed<<<1, 32, 0, s>>>(x, c->ws.err);
  ESPO_LAUNCHED(c);
  const int64_t xoff = (int64_t(x.slot) * x.tp_world + x.tp_rank) * x.cap;
  espo_status st = launch_sweep_fwd(c, logits, ld, tokens, old_logp, mask, row_begin, n_rows,
                                    nullptr, s, c->d_xgath, x.tp_world, xoff);
  if (st != ESPO_OK) return st;
  k_tpx_signal<<<1, 32 * ((x.tp_world + 31) / 32), 0, s>>>(x);
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

// second half: wait for every rank's partials → combine → post consumed
espo_status p2p_recv(espo_ctx_t c, int64_t row_begin, int64_t n_rows, cudaStream_t s) {
  const TpxParams x = tpx_params(c, ++c->x_recv_epoch);
  const int grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  k_tpx_combine<<<grid, 256, 0, s>>>(x, row_begin, n_rows, c->ws);
  ESPO_LAUNCHED(c);
  k_tpx_post<<<1, 32 * ((x.tp_world + 31) / 32), 0, s>>>(x);
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

// Forward of one chunk (arguments and coverage already checked); records the coverage.
espo_status fwd_chunk(espo_ctx_t c, const void* logits, int64_t ld, const int32_t* tokens,
                      const float* old_logp, const uint8_t* mask, int64_t row_begin,
                      int64_t n_rows, cudaStream_t s) {
  espo_status st;
  const bool sharded = c->cfg.vocab_local > 0 && c->cfg.vocab_local < c->cfg.vocab;
  if (sharded && c->tp_p2p) {
    if (n_rows > c->x_cap) return ESPO_ERR_INVALID_ARGUMENT;
    if ((st = p2p_send(c, logits, ld, tokens, old_logp, mask, row_begin, n_rows, s)) != ESPO_OK) return st;
    if ((st = p2p_recv(c, row_begin, n_rows, s)) != ESPO_OK) return st;
  } else if (sharded) {
    // vocabulary-parallel: partial → all-gather over the TP group → combine
    float* part = c->ws.partial;
    float* gath = c->ws.gathered;
    if ((st = launch_sweep_fwd(c, logits, ld, tokens, old_logp, mask, row_begin, n_rows, part, s)) != ESPO_OK)
      return st;
    if (g_nccl.allgather(part, gath, size_t(n_rows) * 4, kNcclFloat32, c->tp_comm, s) != 0)
      return ESPO_ERR_NCCL;
    if ((st = launch_combine(c, gath, c->tp_world, row_begin, n_rows, s)) != ESPO_OK) return st;
  } else {
    if ((st = launch_sweep_fwd(c, logits, ld, tokens, old_logp, mask, row_begin, n_rows, nullptr, s)) != ESPO_OK)
      return st;
  }
  c->covered[row_begin] = row_begin + n_rows;
  c->n_covered += n_rows;
  return ESPO_OK;
}

SeqParams seq_params(espo_ctx_t c, int64_t row_lo, int64_t row_hi) {
  const espo_config& cf = c->cfg;
  SeqParams sp;
  sp.R = c->R;
  sp.row_lo = row_lo;
  sp.row_hi = row_hi;
  sp.V = cf.vocab;
  sp.alpha = cf.alpha;
  sp.eps_min = cf.eps_min;
  sp.K = cf.n_buckets;
  sp.split_num = cf.split_num;
  sp.split_den = cf.split_den;
  sp.partition = cf.partition;
  sp.ratio_mode = cf.ratio_mode;
  sp.norm = cf.norm;
  sp.log_ratio_clamp = cf.log_ratio_clamp;
  sp.inv_logV = 1.0 / std::log(static_cast<double>(cf.vocab));
  sp.zvp_beta = cf.zvp_beta;
  sp.ws = c->ws;
  if (c->n_hsel > 0) sp.ws.H = c->hsel;    // caller-supplied selection entropies (K3 only)
  return sp;
}
}  // namespace

extern "C" {

espo_status espo_loss_fwd(espo_ctx_t c, const void* logits, int64_t ld, const int32_t* tokens,
                          const float* old_logp, const uint8_t* mask, int64_t row_begin,
                          int64_t n_rows, uint32_t flags, espo_stream_t stream) {
  ESPO_RANGE("espo_loss_fwd");
  if (flags != 0) return ESPO_ERR_INVALID_ARGUMENT;
  espo_status st = check_fwd_args(c, logits, ld, tokens, old_logp, row_begin, n_rows);
  if (st != ESPO_OK || n_rows == 0) return st;
  const bool sharded = c->cfg.vocab_local > 0 && c->cfg.vocab_local < c->cfg.vocab;
  if (sharded && !c->tp_comm && !c->tp_p2p) return ESPO_ERR_BAD_STATE;  // use partial + combine
  if (c->single_pass) return ESPO_ERR_BAD_STATE;           // use espo_loss_fwd_bwd
  if ((st = check_coverage(c, row_begin, row_begin + n_rows)) != ESPO_OK) return st;
  DevGuard g(c->device);
  return fwd_chunk(c, logits, ld, tokens, old_logp, mask, row_begin, n_rows, S(stream));
}

espo_status espo_loss_fwd_partial(espo_ctx_t c, const void* logits, int64_t ld,
                                  const int32_t* tokens, const float* old_logp,
                                  const uint8_t* mask, int64_t row_begin, int64_t n_rows,
                                  float* partial, espo_stream_t stream) {
  ESPO_RANGE("espo_loss_fwd_partial");
  espo_status st = check_fwd_args(c, logits, ld, tokens, old_logp, row_begin, n_rows);
  if (st != ESPO_OK || n_rows == 0) return st;
  if (!partial || !aligned16(partial)) return ESPO_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  return launch_sweep_fwd(c, logits, ld, tokens, old_logp, mask, row_begin, n_rows, partial, S(stream));
}

espo_status espo_loss_fwd_combine(espo_ctx_t c, const float* partials, int32_t n_shards,
                                  int64_t row_begin, int64_t n_rows, espo_stream_t stream) {
  ESPO_RANGE("espo_loss_fwd_combine");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Prepared || c->single_pass) return ESPO_ERR_BAD_STATE;
  if (n_rows < 0 || n_rows > INT32_MAX || row_begin < 0 || row_begin + n_rows > c->T ||
      n_shards < 1 || n_shards > 1024)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rows == 0) return ESPO_OK;
  if (!partials || !aligned16(partials)) return ESPO_ERR_INVALID_ARGUMENT;
  espo_status st = check_coverage(c, row_begin, row_begin + n_rows);
  if (st != ESPO_OK) return st;
  DevGuard g(c->device);
  if ((st = launch_combine(c, partials, n_shards, row_begin, n_rows, S(stream))) != ESPO_OK) return st;
  c->covered[row_begin] = row_begin + n_rows;
  c->n_covered += n_rows;
  return ESPO_OK;
}

}  // extern "C"

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool make_map_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t pitch_bytes, uint32_t box_rows) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_encode),
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {uint32_t(kLmBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && std::getenv("ESPO_DEBUG"))
    std::fprintf(stderr, "[libespo] cuTensorMapEncodeTiled failed (%d): rows %llu cols %llu pitch %llu box %u\n",
                 int(r), (unsigned long long)rows, (unsigned long long)cols,
                 (unsigned long long)pitch_bytes, box_rows);
  return r == CUDA_SUCCESS;
}
// fp32 [rows, cols] (row pitch in bytes) as 32 × 32 boxes with 128-byte swizzle: the target of
// the dW GEMM's TMA-reduce epilogue
bool make_map_f32_box32(CUtensorMap* map, void* base, uint64_t rows, uint64_t cols,
                        uint64_t pitch_bytes) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_encode),
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
// vocabulary parts per row block: enough CTAs for ≥ 2 waves; beyond that the best split
// measured on B200 (tools/bench_lmhead.py, n = 32,768, V = 151,936) is 4 parts for d ≤ 4096
// and 2 for d = 8192 (fewer parts keep fewer W tiles live in L2, more parts keep fewer A row
// blocks live)
int lmhead_parts(const espo_ctx_s* c, int mblocks, int ntiles, int d) {
  int parts = (2 * c->num_sms + mblocks - 1) / mblocks;
  parts = std::max(parts, std::max(2, std::min(4, 16384 / d)));
  if (c->lmh_parts > 0) parts = c->lmh_parts;
  return std::max(1, std::min(parts, std::min(64, ntiles)));
}

// C[M, N] (+)= A·B on the tcgen05 GEMM (k_gemm.cuh); maps built by the caller for the
// operands' majorness (K-major A: box {64 K, 128 M}; MN-major: boxes {64 MN, 64 K}).
// pair: CTA-pair kernel (256 × 256 tiles per cluster of 2), else one CTA per 128 × 256 tile.
// M-tiles per raster group of the LM-head GEMM-core kernels: 32 at d ≤ 4096, 64 above
// (tools/bench_lmhead_fwd_ab.py, tools/gemm_sweep.py: sustained A/B on one B200)
int lmh_raster(const espo_ctx_s* c, int d) {
  (void)d;
  return c->lmh_group_m > 0 ? c->lmh_group_m : 16;
}

// Clusters of `csize` CTAs (one per SM at this smem size) that can be resident at once: a
// persistent grid must not exceed it — a cluster that is not resident only starts when a
// resident one exits, i.e. after the whole tile loop (GPCs whose SM count is not a multiple
// of the cluster size leave SMs idle). Cached per kernel; falls back to SMs / csize.
template <typename K>
int max_resident_clusters(K kernel, int csize, int threads, size_t smem, int num_sms,
                          int& cache) {
  if (cache > 0) return cache;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(csize * (num_sms / csize)), 1, 1);
  cfg.blockDim = dim3(unsigned(threads), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = unsigned(csize);
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = num_sms / csize;
  }
  cache = std::min(n, num_sms / csize);
  if (std::getenv("ESPO_DEBUG"))
    std::fprintf(stderr, "[libespo] resident clusters of %d CTAs (%zu B smem): %d (SMs %d)\n",
                 csize, smem, cache, num_sms);
  return cache;
}

struct GemmDyn {          // device-side row count of compacted operands (k_compact.cuh)
  const int* count = nullptr;
  int base = 0, which = 0;   // which: 1 = M, 2 = K
  const int* row_map = nullptr;
};

template <bool kAMN, bool kBMN, int kOut>
espo_status launch_umma_gemm(espo_ctx_t c, const CUtensorMap& ma, const CUtensorMap& mb, int M,
                             int N, int64_t K, void* C, int64_t ldc, int kind, int group_m,
                             int hints, cudaStream_t s, const GemmDyn& dyn = GemmDyn(),
                             const LmEpi* lm = nullptr, float* split_out = nullptr,
                             int64_t split_ld = 0, int sync_opt = -1,
                             const CUtensorMap* mc = nullptr) {
  // kind: 0 = one CTA per 128 × 256 tile, 1 = CTA pair 256 × 256, 2 = CTA pair 256 × 512,
  // 3 = two CTA pairs per cluster sharing A by multicast, 256 × 512 tiles each
  static unsigned long long attr = 0, attr2 = 0, attr3 = 0, attr4 = 0;
  const bool pair = kind != 0;
  const int tn = (kind == 2 || kind == 3) ? 512 : kGmBN;
  GemmParams p;
  p.lm = lm ? *lm : LmEpi{};
  p.ksplit = split_out ? 2 : 1;                 // split-K over 2 (kOutF32 on pairs only)
  p.split_out = split_out;
  p.split_ld = split_ld;
  p.half_release = c->gemm_half_release;
  p.tile_ctr = nullptr;
  // C through TMA reduce-add (kOutAddF32 on pairs, when the caller passed C's tensor map)
  p.tma_red = (kOut == kOutAddF32 && mc != nullptr && c->gemm_tma_red) ? 1 : 0;
  const CUtensorMap& mcc = mc ? *mc : ma;      // unused unless tma_red
  const size_t smem512 = kOut == kOutAddF32 ? G2<512>::kSmemRed : G2<512>::kSmem;
  const size_t smem256 = kOut == kOutAddF32 ? G2<256>::kSmemRed : G2<256>::kSmem;
  if (split_out && (kOut != kOutF32 || kind == 0)) return ESPO_ERR_INVALID_ARGUMENT;
  if ((kOut == kOutLmFwd || kOut == kOutLmDz) && kind == 0) return ESPO_ERR_INVALID_ARGUMENT;
  p.dyn_count = dyn.count;
  p.dyn_base = dyn.base;
  p.dyn_which = dyn.which;
  p.row_map = dyn.row_map;
  p.M = M;
  p.N = N;
  p.K = int(K);
  const int bm = pair ? 2 * kGmBM : kGmBM;
  p.mblk = (M + bm - 1) / bm;
  p.nblk = (N + tn - 1) / tn;
  p.kblk = int((K + kGmBK - 1) / kGmBK);
  p.group_m = std::max(1, group_m);
  p.group_n = group_m < 0 ? -group_m : 0;     // group_m < 0 selects N-groups of −group_m
  p.hint_a = hints & 3;          // hints: 2 bits each for A, B, C
  p.hint_b = (hints >> 2) & 3;
  p.hint_c = (hints >> 4) & 3;
  p.C = C;
  p.ldc = ldc;
  const int64_t tiles = int64_t(p.mblk) * p.nblk;
  if (tiles == 0 || p.kblk == 0) return ESPO_OK;
  if (tiles > INT32_MAX) return ESPO_ERR_INVALID_ARGUMENT;
  p.sync = nullptr;
  // soft lockstep: the caller's setting (chunk | slack << 16, 0 = off) or the context option
  const int sync_chunk = sync_opt >= 0 ? (sync_opt & 0xFFFF) : c->gemm_sync_chunk;
  p.sync_chunk = std::max(1, sync_chunk);
  p.sync_slack = std::max(1, sync_opt >= 0 ? (sync_opt >> 16) : c->gemm_sync_slack);
  p.sync_timeout_ns = 200000;
  static int res2 = 0, res3 = 0, res4 = 0;   // resident clusters per kernel (this process's GPU)
  if (kind == 3) {
    ESPO_CUDA(ensure_smem_attr(k_umma_gemm4<kAMN, kBMN, kOut, 512>, int(smem512), attr4));
    const int64_t super = int64_t(p.mblk) * ((p.nblk + 1) / 2);
    const int clusters = int(std::min<int64_t>(
        super, max_resident_clusters(k_umma_gemm4<kAMN, kBMN, kOut, 512>, 4, kG2Threads,
                                     smem512, c->num_sms, res4)));
    k_umma_gemm4<kAMN, kBMN, kOut, 512><<<4 * clusters, kG2Threads, smem512, s>>>(ma, mb, mcc, p);
  } else if (pair) {
    if (kind == 2) ESPO_CUDA(ensure_smem_attr(k_umma_gemm2<kAMN, kBMN, kOut, 512>, int(smem512), attr3));
    else ESPO_CUDA(ensure_smem_attr(k_umma_gemm2<kAMN, kBMN, kOut, 256>, int(smem256), attr2));
    const int clusters = int(std::min<int64_t>(
        tiles, kind == 2 ? max_resident_clusters(k_umma_gemm2<kAMN, kBMN, kOut, 512>, 2, kG2Threads,
                                                 smem512, c->num_sms, res3)
                         : max_resident_clusters(k_umma_gemm2<kAMN, kBMN, kOut, 256>, 2, kG2Threads,
                                                 smem256, c->num_sms, res2)));
    if (c->gemm_dyn) {                         // dynamic tile scheduler: a zeroed counter
      if (!c->gemm_tctr) ESPO_CUDA(cudaMalloc(&c->gemm_tctr, sizeof(int)));
      ESPO_CUDA(cudaMemsetAsync(c->gemm_tctr, 0, sizeof(int), s));
      p.tile_ctr = c->gemm_tctr;
    }
    if (sync_chunk > 0) {                      // one zeroed progress counter per wave
      const int64_t waves = (tiles + clusters - 1) / clusters;
      if (size_t(waves) * 4 > c->gemm_sync_cap) {
        if (c->gemm_sync) cudaFree(c->gemm_sync);
        c->gemm_sync = nullptr;
        c->gemm_sync_cap = 0;
        ESPO_CUDA(cudaMalloc(&c->gemm_sync, size_t(waves) * 4));
        c->gemm_sync_cap = size_t(waves) * 4;
      }
      ESPO_CUDA(cudaMemsetAsync(c->gemm_sync, 0, size_t(waves) * 4, s));
      p.sync = static_cast<unsigned*>(c->gemm_sync);
    }
    if (kind == 2)
      k_umma_gemm2<kAMN, kBMN, kOut, 512><<<2 * clusters, kG2Threads, smem512, s>>>(ma, mb, mcc, p);
    else
      k_umma_gemm2<kAMN, kBMN, kOut, 256><<<2 * clusters, kG2Threads, smem256, s>>>(ma, mb, mcc, p);
  } else {
    ESPO_CUDA(ensure_smem_attr(k_umma_gemm<kAMN, kBMN, kOut>, int(kGmSmem), attr));
    const int grid = int(std::min<int64_t>(tiles, c->num_sms));
    k_umma_gemm<kAMN, kBMN, kOut><<<grid, kGmThreads, kGmSmem, s>>>(ma, mb, p);
  }
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}
}  // namespace

extern "C" {

espo_status espo_lmhead_fwd(espo_ctx_t c, const void* hidden, int64_t ldh, const void* weight,
                            int64_t ldw, int32_t d, const int32_t* tokens, const float* old_logp,
                            const uint8_t* mask, int64_t row_begin, int64_t n_rows,
                            espo_stream_t stream) {
  ESPO_RANGE("espo_lmhead_fwd");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Prepared || c->single_pass) return ESPO_ERR_BAD_STATE;
  if (n_rows < 0 || n_rows > INT32_MAX || row_begin < 0 || row_begin + n_rows > c->T || d < 1)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rows == 0) return ESPO_OK;
  if (!hidden || !weight || !tokens || !old_logp || ldh < d || ldw < d) return ESPO_ERR_INVALID_ARGUMENT;
  if (!aligned16(hidden) || !aligned16(weight) || (ldh * 2) % 16 || (ldw * 2) % 16)
    return ESPO_ERR_ALIGNMENT;
  if (c->cfg.vocab_local > 0 && c->cfg.vocab_local < c->cfg.vocab) return ESPO_ERR_UNSUPPORTED;
  espo_status st = check_coverage(c, row_begin, row_begin + n_rows);
  if (st != ESPO_OK) return st;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  const int V = c->cfg.vocab;
  const int mblocks = int((n_rows + kLmBM - 1) / kLmBM);
  const int ntiles = (V + kLmBN - 1) / kLmBN;
  const int parts = lmhead_parts(c, mblocks, ntiles, d);
  if (mblocks > 65535) return ESPO_ERR_INVALID_ARGUMENT;
  const size_t need = size_t(parts) * size_t(n_rows) * 16;
  if (need > c->lmh_cap) {
    if (c->lmh_partial) cudaFree(c->lmh_partial);
    c->lmh_partial = nullptr;
    ESPO_CUDA(cudaMalloc(&c->lmh_partial, need));
    c->lmh_cap = need;
  }
  const int pre_grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  if (c->lmh_impl == 0) {
    // on the tcgen05 GEMM core: CTA-pair 256 × 512 tiles of z = h·Wᵀ in a grouped raster, each
    // tile's rows reduced to a partial {R, S, W, u_y} (k_gemm.cuh kOutLmFwd), then merged over
    // the tiles like vocabulary shards; M-tiles without a valid row are skipped
    const int tw = c->lmh_tile256 ? 256 : 512;
    const int nt = 2 * ((V + tw - 1) / tw);   // one partial per (tile, column half)
    const int nlive = int((n_rows + 255) / 256);
    const size_t needp = size_t(nt) * size_t(n_rows) * 16;
    if (needp > c->lmh_cap) {
      if (c->lmh_partial) cudaFree(c->lmh_partial);
      c->lmh_partial = nullptr;
      c->lmh_cap = 0;
      ESPO_CUDA(cudaMalloc(&c->lmh_partial, needp));
      c->lmh_cap = needp;
    }
    if (size_t(nlive) > c->lmh_live_cap) {
      if (c->lmh_live) cudaFree(c->lmh_live);
      c->lmh_live = nullptr;
      c->lmh_live_cap = 0;
      ESPO_CUDA(cudaMalloc(&c->lmh_live, size_t(nlive)));
      c->lmh_live_cap = size_t(nlive);
    }
    CUtensorMap mh, mw;
    if (!make_map_bf16(&mh, hidden, uint64_t(n_rows), uint64_t(d), uint64_t(ldh) * 2, kGmBM) ||
        !make_map_bf16(&mw, weight, uint64_t(V), uint64_t(d), uint64_t(ldw) * 2, 128))
      return ESPO_ERR_CUDA;
    k_lmh_rows<<<pre_grid, 256, 0, s>>>(tokens, old_logp, mask, row_begin, n_rows, V, c->ws);
    ESPO_LAUNCHED(c);
    k_block_live<<<nlive, 256, 0, s>>>(c->ws.flag + row_begin, int(n_rows), 256, c->lmh_live);
    ESPO_LAUNCHED(c);
    LmEpi lm{};
    lm.tokens = tokens;
    lm.flag = c->ws.flag + row_begin;
    lm.mlive = c->lmh_live;
    lm.partial = reinterpret_cast<float4*>(c->lmh_partial);
    lm.lamL = c->cfg.logit_scale * kLog2e;
    lm.V = V;
    lm.n_rows = int(n_rows);
    lm.err = c->ws.err;
    st = launch_umma_gemm<false, false, kOutLmFwd>(c, mh, mw, int(n_rows), V, d, nullptr, 0,
                                                   c->lmh_tile256 ? 1 : c->lmh_mcast ? 3 : 2,
                                                   lmh_raster(c, d), c->lmh_hints, s, GemmDyn(), &lm,
                                                   nullptr, 0, c->lmh_sync);
    if (st != ESPO_OK) return st;
    {
      const int grid = static_cast<int>(std::min<int64_t>((n_rows + 7) / 8, int64_t(c->num_sms) * 16));
      k_fwd_combine64<<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(c->lmh_partial), nt,
                                           row_begin, n_rows, c->ws);
      ESPO_LAUNCHED(c);
    }
    c->covered[row_begin] = row_begin + n_rows;
    c->n_covered += n_rows;
    return ESPO_OK;
  }
  CUtensorMap mh, mw;
  if (!make_map_bf16(&mh, hidden, uint64_t(n_rows), uint64_t(d), uint64_t(ldh) * 2, kLmBM) ||
      !make_map_bf16(&mw, weight, uint64_t(V), uint64_t(d), uint64_t(ldw) * 2, c->lmh_2cta ? kLmBN / 2 : kLmBN))
    return ESPO_ERR_CUDA;
  k_lmh_rows<<<pre_grid, 256, 0, s>>>(tokens, old_logp, mask, row_begin, n_rows, V, c->ws);
  ESPO_LAUNCHED(c);
  static unsigned long long attr_mask = 0, attr_mask2 = 0;
  ESPO_CUDA(ensure_smem_attr(k_lmhead_fwd, int(kLmSmem), attr_mask));
  ESPO_CUDA(ensure_smem_attr(k_lmhead2_fwd, int(kL2Smem), attr_mask2));
  LmParams lp{};
  lp.n_rows = int(n_rows);
  lp.row_begin = row_begin;
  lp.d = d;
  lp.V = V;
  lp.ntiles = ntiles;
  lp.parts = parts;
  lp.lam_log2e = c->cfg.logit_scale * kLog2e;
  lp.tokens = tokens;
  lp.partial = c->lmh_partial;
  lp.ws = c->ws;
  if (c->lmh_2cta)   // CTA pairs: (2·part + rank, row-block pair), cluster (2, 1, 1)
    k_lmhead2_fwd<<<dim3(2 * parts, (mblocks + 1) / 2), kLmThreads, kL2Smem, s>>>(mh, mw, lp);
  else
    k_lmhead_fwd<<<dim3(parts, mblocks), kLmThreads, kLmSmem, s>>>(mh, mw, lp);
  ESPO_LAUNCHED(c);
  if ((st = launch_combine(c, c->lmh_partial, parts, row_begin, n_rows, s)) != ESPO_OK) return st;
  c->covered[row_begin] = row_begin + n_rows;
  c->n_covered += n_rows;
  return ESPO_OK;
}

espo_status espo_lmhead_bwd(espo_ctx_t c, const void* hidden, int64_t ldh, const void* weight,
                            int64_t ldw, int32_t d, void* dhidden, int64_t lddh, int32_t dh_dtype,
                            float* dweight, int64_t lddw, const float* grad_loss_dev,
                            int64_t row_begin, int64_t n_rows, espo_stream_t stream) {
  ESPO_RANGE("espo_lmhead_bwd");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Finalized) return ESPO_ERR_BAD_STATE;
  if (n_rows < 0 || n_rows > INT32_MAX || row_begin < 0 || row_begin + n_rows > c->T || d < 1)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rows == 0) return ESPO_OK;
  if (!hidden || !weight || ldh < d || ldw < d) return ESPO_ERR_INVALID_ARGUMENT;
  if (dh_dtype != ESPO_F32 && dh_dtype != ESPO_BF16) return ESPO_ERR_INVALID_ARGUMENT;
  if ((dhidden && lddh < d) || (dweight && lddw < d)) return ESPO_ERR_INVALID_ARGUMENT;
  if (!aligned16(hidden) || !aligned16(weight) || (ldh * 2) % 16 || (ldw * 2) % 16 ||
      (dhidden && (!aligned16(dhidden) || (lddh * int64_t(dsize(dh_dtype))) % 16)) ||
      (dweight && (!aligned16(dweight) || (lddw * 4) % 16)))
    return ESPO_ERR_ALIGNMENT;
  if (c->cfg.vocab_local > 0 && c->cfg.vocab_local < c->cfg.vocab) return ESPO_ERR_UNSUPPORTED;
  if (c->cp_world > 1 && (row_begin < cp_lo(c) || row_begin + n_rows > cp_hi(c)))
    return ESPO_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  const int V = c->cfg.vocab;
  const int ntiles = (V + kLmBN - 1) / kLmBN;
  // dz scratch pitch: a multiple of the dz tile width (256, or 512 on the GEMM core)
  const int64_t ldz = c->lmh_impl == 0 ? round_up(size_t(V), 512) : int64_t(ntiles) * kLmBN;
  const int sub = int(std::min<int64_t>(c->lmh_bwd_rows, round_up(size_t(n_rows), kLmBM)));
  const size_t need = size_t(sub) * size_t(ldz) * 2;
  if (need > c->lmh_dz_cap) {
    if (c->lmh_dz) cudaFree(c->lmh_dz);
    c->lmh_dz = nullptr;
    c->lmh_dz_cap = 0;
    ESPO_CUDA(cudaMalloc(&c->lmh_dz, need));
    c->lmh_dz_cap = need;
  }
  const bool use_blas = c->lmh_bwd_gemm == 1;
  if (use_blas) {
    if (!c->blas) {
      if (!g_blas.load()) return ESPO_ERR_BLAS;
      if (g_blas.create(&c->blas) != 0) {
        c->blas = nullptr;
        return ESPO_ERR_BLAS;
      }
      ESPO_CUDA(cudaMalloc(&c->blas_ws, kBlasWorkspace));
      if (g_blas.set_workspace(c->blas, c->blas_ws, kBlasWorkspace) != 0) return ESPO_ERR_BLAS;
    }
    if (g_blas.set_stream(c->blas, s) != 0) return ESPO_ERR_BLAS;
  }
  // per-row records {g, −lse·log2e, g·q, y} for the whole chunk (K5's k_bwd_recs, zero-filling)
  BwdRec* rec = static_cast<BwdRec*>(c->ws.list);
  const int pre_grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  k_bwd_recs<<<pre_grid, 256, 0, s>>>(row_begin, n_rows, grad_loss_dev, 1, 0, V, c->ws, rec);
  ESPO_LAUNCHED(c);
  static unsigned long long attr_mask = 0, attr_mask2 = 0;
  ESPO_CUDA(ensure_smem_attr(k_lmhead_dz, int(kLmSmem), attr_mask));
  ESPO_CUDA(ensure_smem_attr(k_lmhead2_dz, int(kL2Smem), attr_mask2));
  CUtensorMap mw, mw_mn, mw_k128;
  if (!make_map_bf16(&mw, weight, uint64_t(V), uint64_t(d), uint64_t(ldw) * 2, c->lmh_2cta ? kLmBN / 2 : kLmBN) ||
      !make_map_bf16(&mw_mn, weight, uint64_t(V), uint64_t(d), uint64_t(ldw) * 2, 64) ||
      !make_map_bf16(&mw_k128, weight, uint64_t(V), uint64_t(d), uint64_t(ldw) * 2, 128))
    return ESPO_ERR_CUDA;
  const float one = 1.f, zero = 0.f;
  const char* hb = static_cast<const char*>(hidden);
  // rows with gradient only (k_compact.cuh): default for the tcgen05 GEMMs when d % 8 == 0
  const bool compact = !use_blas && c->lmh_compact && d % 8 == 0;
  int* list = nullptr;
  int* total = nullptr;
  __nv_bfloat16* hc = nullptr;
  BwdRec* rec_c = nullptr;
  const int64_t ldc = round_up(size_t(d), 8);
  if (compact) {
    const int nb = int((n_rows + kCmpBlock - 1) / kCmpBlock);
    const size_t need_c = round_up(size_t(n_rows) * 4, 256) + round_up(size_t(nb + 1) * 4, 256) +
                          round_up(size_t(sub) * ldc * 2, 256) + size_t(sub) * sizeof(BwdRec);
    if (need_c > c->lmh_cmp_cap) {
      if (c->lmh_cmp) cudaFree(c->lmh_cmp);
      c->lmh_cmp = nullptr;
      c->lmh_cmp_cap = 0;
      ESPO_CUDA(cudaMalloc(&c->lmh_cmp, need_c));
      c->lmh_cmp_cap = need_c;
    }
    uint8_t* b = static_cast<uint8_t*>(c->lmh_cmp);
    list = reinterpret_cast<int*>(b);
    b += round_up(size_t(n_rows) * 4, 256);
    total = reinterpret_cast<int*>(b);              // [0] = total, [1 ..] = block counts
    b += round_up(size_t(nb + 1) * 4, 256);
    hc = reinterpret_cast<__nv_bfloat16*>(b);
    b += round_up(size_t(sub) * ldc * 2, 256);
    rec_c = reinterpret_cast<BwdRec*>(b);
    k_cmp_count<<<nb, kCmpBlock, 0, s>>>(rec, int(n_rows), total + 1);
    ESPO_LAUNCHED(c);
    k_cmp_scatter<<<nb, kCmpBlock, 0, s>>>(rec, int(n_rows), total + 1, nb, list, total);
    ESPO_LAUNCHED(c);
    if (dhidden) {   // rows without gradient: dh = 0 (the GEMM writes only the listed rows)
      k_zero_rows<<<int(n_rows), 256, 0, s>>>(rec, int(n_rows), dhidden,
                                              lddh * int64_t(dsize(dh_dtype)), d * int(dsize(dh_dtype)));
      ESPO_LAUNCHED(c);
    }
  }
  for (int64_t r0 = 0; r0 < n_rows; r0 += sub) {
    // compact: r0 indexes the list of rows with gradient (sub-chunks past the count exit at
    // once on the device); otherwise it is the chunk row
    const int n = int(std::min<int64_t>(sub, n_rows - r0));
    const int mblocks = (n + kLmBM - 1) / kLmBM;
    const int parts = lmhead_parts(c, mblocks, ntiles, d);
    const char* hsrc = compact ? reinterpret_cast<const char*>(hc) : hb + r0 * ldh * 2;
    const int64_t hld = compact ? ldc : ldh;
    if (compact) {
      k_cmp_gather<<<n, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(hidden), ldh, d, rec, list,
                                     total, int(r0), n, hc, ldc, rec_c);
      ESPO_LAUNCHED(c);
    }
    CUtensorMap mh;
    if (!make_map_bf16(&mh, hsrc, uint64_t(n), uint64_t(d), uint64_t(hld) * 2, kLmBM))
      return ESPO_ERR_CUDA;
    LmParams lp{};
    lp.n_rows = n;
    lp.row_begin = row_begin + r0;
    lp.d = d;
    lp.V = V;
    lp.ntiles = ntiles;
    lp.parts = parts;
    lp.lam_log2e = c->cfg.logit_scale * kLog2e;
    lp.rec = compact ? rec_c : rec + r0;
    lp.dz = static_cast<__nv_bfloat16*>(c->lmh_dz);
    lp.ldz = ldz;
    lp.ws = c->ws;
    if (compact) {
      lp.dyn_count = total;
      lp.dyn_base = int(r0);
    }
    if (c->lmh_impl == 0) {    // recompute on the GEMM core, dz epilogue (kOutLmDz)
      LmEpi lm{};
      lm.rec = lp.rec;
      lm.dz = lp.dz;
      lm.ldz = ldz;
      lm.lamL = lp.lam_log2e;
      lm.V = V;
      lm.n_rows = n;
      lm.err = c->ws.err;
      GemmDyn dz_dyn;
      if (compact) {             // rows up to the next 256 (their records are zero): dz = 0
        dz_dyn.count = total;
        dz_dyn.base = int(r0);
        dz_dyn.which = 3;
      }
      const espo_status st = launch_umma_gemm<false, false, kOutLmDz>(
          c, mh, mw_k128, n, int(ldz), d, nullptr, 0, c->lmh_tile256 ? 1 : c->lmh_mcast ? 3 : 2,
          lmh_raster(c, d), c->lmh_hints, s, dz_dyn, &lm, nullptr, 0,
          c->gemm_dyn ? 0 : c->lmh_sync);   // dz: with the dynamic scheduler, no lockstep (measured)
      if (st != ESPO_OK) return st;
    } else if (c->lmh_2cta) {
      k_lmhead2_dz<<<dim3(2 * parts, (mblocks + 1) / 2), kLmThreads, kL2Smem, s>>>(mh, mw, lp);
      ESPO_LAUNCHED(c);
    } else {
      k_lmhead_dz<<<dim3(parts, mblocks), kLmThreads, kLmSmem, s>>>(mh, mw, lp);
      ESPO_LAUNCHED(c);
    }
    // z = h·Wᵀ (dz already carries λ, as K5's) ⇒ dh = dz·W and dW = dzᵀ·h
    if (!use_blas) {
      CUtensorMap mdz_k, mdz_mn, mh_mn;
      if (!make_map_bf16(&mdz_k, c->lmh_dz, uint64_t(n), uint64_t(ldz), uint64_t(ldz) * 2, kGmBM) ||
          !make_map_bf16(&mdz_mn, c->lmh_dz, uint64_t(n), uint64_t(ldz), uint64_t(ldz) * 2, 64) ||
          !make_map_bf16(&mh_mn, hsrc, uint64_t(n), uint64_t(d), uint64_t(hld) * 2, 64))
        return ESPO_ERR_CUDA;
      espo_status st;
      // tile kinds (ESPO_OPT_LMHEAD_BWD_GEMM): 0 → dh on 256 × 512 pair tiles (long K) and dW
      // on 256 × 256 pair tiles; 2 → one CTA per 128 × 256; 3 → 256 × 256 pairs for both;
      // 4 → 256 × 512 pairs for both
      // (tools/gemm_sweep.py, sustained A/B on one B200: d = 4096 → dW 256-wide pair tiles in
      // N-groups of 8 blocks; d = 8192 → 512-wide pair tiles in N-groups of 2)
      const int g = c->lmh_bwd_gemm;
      const bool wide_dw = d > 4096;
      const int kind_dh = g == 2 ? 0 : g == 3 ? 1 : (g == 5 || g == 6) ? 3 : 2;
      const int kind_dw = g == 2 ? 0 : g == 3 ? 1 : g == 4 ? 2 : g == 5 ? 3 : g == 7 ? 1 :
                          (wide_dw ? 2 : 1);
      // tile order: dh has a long K (the vocabulary) and few tiles: groups of 8 M-blocks keep
      // the resident tiles' A and B panels small; dW (K = rows): N fastest, so every M-block
      // of dz is read once while h stays in L2
      const int g_dh = c->gemm_group_m > 0 ? c->gemm_group_m : (wide_dw ? 16 : 8);
      // soft lockstep of dh / dW: the option if given, else on (16 K-steps, slack 2) above
      // d = 4096 (sustained sweep: d = 8192 sub-chunk 52.5 → 50.0 ms; at d = 4096 it costs 2–5 %)
      const int sync_auto = (!c->gemm_sync_set && wide_dw) ? (16 | (2 << 16)) : -1;
      const int sync_dh = sync_auto;
      const int sync_dw = c->gemm_sync_dw >= 0 ? c->gemm_sync_dw : sync_auto;
      // dW: groups of gemm_group_n_dw N-blocks (0 = N fastest over all of d)
      const int g_dw = c->gemm_group_n_dw > 0 ? -c->gemm_group_n_dw
                                              : (g == 0 ? (wide_dw ? -2 : -8) : g == 7 ? -8 : 1);
      // L2 policies (2 bits each: A | B << 2 | C << 4; 1 = evict_first, 2 = evict_last):
      // dh streams both panels once per wave; dW streams dz and the dW read-add-write while
      // every tile re-reads h (64 MB at n = 8192, d = 4096), which should stay in L2
      const int hint_dh = c->gemm_hints_dh >= 0 ? c->gemm_hints_dh : 0;
      const int hint_dw = c->gemm_hints_dw >= 0 ? c->gemm_hints_dw : (1 | (2 << 2) | (1 << 4));
      GemmDyn dyn_m, dyn_k;
      if (compact) {
        dyn_m.count = dyn_k.count = total;
        dyn_m.base = dyn_k.base = int(r0);
        dyn_m.which = 1;
        dyn_k.which = 2;
        dyn_m.row_map = list + r0;
      }
      if (dhidden) {   // dh[n, d] = dz[n, V] · W[V, d]: A = dz K-major, B = W MN-major
        char* dh = static_cast<char*>(dhidden) + (compact ? 0 : r0 * lddh * int64_t(dsize(dh_dtype)));
        // dh has few, long tiles (K = the vocabulary): at 8192 rows and d = 4096 only 256
        // pair tiles = 3.5 waves of 74 pairs (the 4th half empty). Below 6 waves, split K in
        // two (deterministic: K-half 1 into a scratch, added by k_split_fixup)
        float* split = nullptr;
        if (dh_dtype == ESPO_F32 && kind_dh != 0 && d % 4 == 0 && c->lmh_split_k) {
          const int64_t tiles = int64_t((n + 255) / 256) * ((d + (kind_dh == 1 ? 255 : 511)) / (kind_dh == 1 ? 256 : 512));
          if (tiles < 6 * (c->num_sms / 2)) {
            const size_t need_s = size_t(n) * size_t(d) * 4;
            if (need_s > c->lmh_split_cap) {
              if (c->lmh_split) cudaFree(c->lmh_split);
              c->lmh_split = nullptr;
              c->lmh_split_cap = 0;
              ESPO_CUDA(cudaMalloc(&c->lmh_split, need_s));
              c->lmh_split_cap = need_s;
            }
            split = static_cast<float*>(c->lmh_split);
          }
        }
        st = dh_dtype == ESPO_BF16
                 ? launch_umma_gemm<false, true, kOutBF16>(c, mdz_k, mw_mn, n, d, ldz, dh, lddh, kind_dh, g_dh, hint_dh, s, dyn_m,
                                                           nullptr, nullptr, 0, sync_dh)
                 : launch_umma_gemm<false, true, kOutF32>(c, mdz_k, mw_mn, n, d, ldz, dh, lddh, kind_dh, g_dh, hint_dh, s, dyn_m,
                                                          nullptr, split, d, sync_dh);
        if (st != ESPO_OK) return st;
        if (split) {
          const int grid = c->num_sms * 8;
          k_split_fixup<<<grid, 256, 0, s>>>(reinterpret_cast<float*>(dh), lddh, split, d, n, d,
                                             dyn_m.count, dyn_m.base, dyn_m.row_map);
          ESPO_LAUNCHED(c);
        }
      }
      if (dweight) {   // dW[V, d] += dzᵀ[V, n] · h[n, d]: A = dz MN-major, B = h MN-major
        CUtensorMap mdw;
        const bool red = c->gemm_tma_red && kind_dw != 0 &&
                         make_map_f32_box32(&mdw, dweight, uint64_t(V), uint64_t(d), uint64_t(lddw) * 4);
        st = launch_umma_gemm<true, true, kOutAddF32>(c, mdz_mn, mh_mn, V, d, n, dweight, lddw, kind_dw, g_dw, hint_dw, s, dyn_k,
                                                      nullptr, nullptr, 0, sync_dw, red ? &mdw : nullptr);
        if (st != ESPO_OK) return st;
      }
      continue;
    }
    if (dhidden) {   // column-major view: dhᵀ[d, n] = Wᵀ[d, V] · dzᵀ[V, n]
      char* dh = static_cast<char*>(dhidden) + r0 * lddh * int64_t(dsize(dh_dtype));
      if (g_blas.gemm(c->blas, CUBLAS_OP_N, CUBLAS_OP_N, d, n, V, &one, weight, CUDA_R_16BF,
                      int(ldw), c->lmh_dz, CUDA_R_16BF, int(ldz), &zero, dh,
                      dh_dtype == ESPO_BF16 ? CUDA_R_16BF : CUDA_R_32F, int(lddh),
                      CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != 0)
        return ESPO_ERR_BLAS;
    }
    if (dweight) {   // column-major view: dWᵀ[d, V] += hᵀ[d, n] · dz[n, V]
      if (g_blas.gemm(c->blas, CUBLAS_OP_N, CUBLAS_OP_T, d, V, n, &one, hb + r0 * ldh * 2,
                      CUDA_R_16BF, int(ldh), c->lmh_dz, CUDA_R_16BF, int(ldz), &one, dweight,
                      CUDA_R_32F, int(lddw), CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT) != 0)
        return ESPO_ERR_BLAS;
    }
  }
  return ESPO_OK;
}

void espo_reward_shaping_default(espo_reward_shaping* p, int32_t max_len) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->max_len = max_len;
  p->buffer = 0;
  p->ngram = 4;
  p->gamma_rep = 1.0f;
  p->rep_thresh = 0.2f;
}

espo_status espo_reshape_rewards(espo_ctx_t c, const espo_reward_shaping* prm,
                                 const float* base_rewards, const int32_t* tokens,
                                 const int64_t* seq_offsets, int32_t n_rollouts,
                                 int64_t n_tokens, float* rewards_out, float* len_pen_out,
                                 float* rep_pen_out, espo_stream_t stream) {
  ESPO_RANGE("espo_reshape_rewards");
  if (!c || !prm || !base_rewards || !seq_offsets || !rewards_out || n_rollouts < 0 ||
      n_tokens < 0 || (n_tokens > 0 && !tokens))
    return ESPO_ERR_INVALID_ARGUMENT;
  if (prm->max_len < 1 || prm->buffer < 0 || prm->buffer > prm->max_len || prm->ngram < 1 ||
      prm->ngram > 16 || !(prm->gamma_rep >= 0.f) || !std::isfinite(prm->gamma_rep) ||
      !std::isfinite(prm->rep_thresh))
    return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rollouts == 0) return ESPO_OK;
  DevGuard g(c->device);
  const int64_t need = std::max<int64_t>(4 * n_tokens, 1);
  if (need > c->rs_cap) {
    if (c->rs_scratch) cudaFree(c->rs_scratch);
    c->rs_scratch = nullptr;
    ESPO_CUDA(cudaMalloc(&c->rs_scratch, size_t(need) * 12));
    c->rs_cap = need;
  }
  ReshapeParams rp;
  rp.base = base_rewards;
  rp.tokens = tokens;
  rp.seq_off = seq_offsets;
  rp.R = n_rollouts;
  rp.max_len = prm->max_len;
  rp.buffer = prm->buffer;
  rp.ngram = prm->ngram;
  rp.gamma_rep = prm->gamma_rep;
  rp.rep_thresh = prm->rep_thresh;
  rp.out = rewards_out;
  rp.len_pen = len_pen_out;
  rp.rep_pen = rep_pen_out;
  rp.keys = static_cast<uint64_t*>(c->rs_scratch);
  rp.first = reinterpret_cast<int32_t*>(static_cast<char*>(c->rs_scratch) + size_t(c->rs_cap) * 8);
  k_reshape_rewards<<<n_rollouts, 256, 0, S(stream)>>>(rp);
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

espo_status espo_attach_tp(espo_ctx_t c, const void* tp_unique_id, int32_t tp_rank,
                           int32_t tp_world) {
  if (!c || !tp_unique_id || tp_world < 1 || tp_rank < 0 || tp_rank >= tp_world)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (c->cfg.vocab_local <= 0 || c->tp_comm) return ESPO_ERR_BAD_STATE;
  if (!g_nccl.load()) return ESPO_ERR_NCCL;
  DevGuard g(c->device);
  nccl_uid id;
  std::memcpy(&id, tp_unique_id, sizeof(id));
  if (g_nccl.init_rank(&c->tp_comm, tp_world, id, tp_rank) != 0) {
    c->tp_comm = nullptr;
    return ESPO_ERR_NCCL;
  }
  c->tp_world = tp_world;
  c->cap_T = 0;  // re-size the workspace at the next prepare (adds the gather buffer)
  return ESPO_OK;
}

espo_status espo_tp_p2p_buffer(espo_ctx_t c, int64_t max_rows, int32_t tp_world,
                               void* ipc_handle_out) {
  if (!c || max_rows < 1 || max_rows > INT32_MAX || tp_world < 1 || tp_world > 1024)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (c->cfg.vocab_local <= 0 || c->tp_p2p || c->x_buf) return ESPO_ERR_BAD_STATE;
  DevGuard g(c->device);
  const size_t bytes = kTpxFlagBytes + size_t(2) * tp_world * size_t(max_rows) * 16;
  ESPO_CUDA(cudaMalloc(&c->x_buf, bytes));
  ESPO_CUDA(cudaMemset(c->x_buf, 0, bytes));
  c->x_cap = max_rows;
  c->x_world = tp_world;
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    ESPO_CUDA(cudaIpcGetMemHandle(&h, c->x_buf));
    std::memcpy(ipc_handle_out, &h, sizeof(h));
  }
  return ESPO_OK;
}

}  // extern "C"

namespace {
espo_status tpx_finish_connect(espo_ctx_t c, const std::vector<uint8_t*>& bases, int32_t tp_rank) {
  const int w = int(bases.size());
  std::vector<void*> host(2 * w);
  for (int k = 0; k < w; ++k) {
    host[k] = bases[k];
    host[w + k] = bases[k] + kTpxFlagBytes;
  }
  ESPO_CUDA(cudaMalloc(&c->d_xpeer, host.size() * sizeof(void*)));
  ESPO_CUDA(cudaMemcpy(c->d_xpeer, host.data(), host.size() * sizeof(void*), cudaMemcpyHostToDevice));
  c->d_xgath = reinterpret_cast<float4**>(c->d_xpeer + w);
  c->tp_rank = tp_rank;
  c->tp_p2p = true;
  c->x_send_epoch = c->x_recv_epoch = 0;
  return ESPO_OK;
}
}  // namespace

extern "C" {

espo_status espo_tp_p2p_open(espo_ctx_t c, const void* ipc_handles, int32_t tp_rank,
                             int32_t tp_world) {
  if (!c || !ipc_handles || tp_rank < 0 || tp_rank >= tp_world) return ESPO_ERR_INVALID_ARGUMENT;
  if (!c->x_buf || c->x_world != tp_world || c->tp_p2p) return ESPO_ERR_BAD_STATE;
  DevGuard g(c->device);
  std::vector<uint8_t*> bases(tp_world);
  for (int k = 0; k < tp_world; ++k) {
    if (k == tp_rank) {
      bases[k] = static_cast<uint8_t*>(c->x_buf);
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(ipc_handles) + size_t(k) * ESPO_IPC_HANDLE_BYTES, sizeof(h));
    void* q = nullptr;
    ESPO_CUDA(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
    c->x_opened.push_back(q);
    bases[k] = static_cast<uint8_t*>(q);
  }
  return tpx_finish_connect(c, bases, tp_rank);
}

espo_status espo_tp_p2p_connect_local(espo_ctx_t c, const espo_ctx_t* ranks, int32_t tp_rank,
                                      int32_t tp_world) {
  if (!c || !ranks || tp_rank < 0 || tp_rank >= tp_world || ranks[tp_rank] != c)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (!c->x_buf || c->x_world != tp_world || c->tp_p2p) return ESPO_ERR_BAD_STATE;
  std::vector<uint8_t*> bases(tp_world);
  for (int k = 0; k < tp_world; ++k) {
    if (!ranks[k] || !ranks[k]->x_buf || ranks[k]->device != c->device ||
        ranks[k]->x_cap != c->x_cap || ranks[k]->x_world != tp_world)
      return ESPO_ERR_INVALID_ARGUMENT;
    bases[k] = static_cast<uint8_t*>(ranks[k]->x_buf);
  }
  DevGuard g(c->device);
  return tpx_finish_connect(c, bases, tp_rank);
}

espo_status espo_tp_p2p_unmap(espo_ctx_t c) {
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  cudaDeviceSynchronize();
  for (void* q : c->x_opened) cudaIpcCloseMemHandle(q);
  c->x_opened.clear();
  if (c->d_xpeer) cudaFree(c->d_xpeer);
  c->d_xpeer = nullptr;
  c->d_xgath = nullptr;
  c->tp_p2p = false;
  return ESPO_OK;
}

espo_status espo_loss_fwd_p2p_send(espo_ctx_t c, const void* logits, int64_t ld,
                                   const int32_t* tokens, const float* old_logp,
                                   const uint8_t* mask, int64_t row_begin, int64_t n_rows,
                                   espo_stream_t stream) {
  ESPO_RANGE("espo_loss_fwd_p2p_send");
  espo_status st = check_fwd_args(c, logits, ld, tokens, old_logp, row_begin, n_rows);
  if (st != ESPO_OK || n_rows == 0) return st;
  if (!c->tp_p2p || c->single_pass) return ESPO_ERR_BAD_STATE;
  if (n_rows > c->x_cap) return ESPO_ERR_INVALID_ARGUMENT;
  if ((st = check_coverage(c, row_begin, row_begin + n_rows)) != ESPO_OK) return st;
  DevGuard g(c->device);
  return p2p_send(c, logits, ld, tokens, old_logp, mask, row_begin, n_rows, S(stream));
}

espo_status espo_loss_fwd_p2p_recv(espo_ctx_t c, int64_t row_begin, int64_t n_rows,
                                   espo_stream_t stream) {
  ESPO_RANGE("espo_loss_fwd_p2p_recv");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Prepared || !c->tp_p2p || c->single_pass) return ESPO_ERR_BAD_STATE;
  if (n_rows < 0 || n_rows > c->x_cap || row_begin < 0 || row_begin + n_rows > c->T)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rows == 0) return ESPO_OK;
  espo_status st = check_coverage(c, row_begin, row_begin + n_rows);
  if (st != ESPO_OK) return st;
  if (c->x_recv_epoch >= c->x_send_epoch) return ESPO_ERR_BAD_STATE;   // recv before its send
  DevGuard g(c->device);
  if ((st = p2p_recv(c, row_begin, n_rows, S(stream))) != ESPO_OK) return st;
  c->covered[row_begin] = row_begin + n_rows;
  c->n_covered += n_rows;
  return ESPO_OK;
}

espo_status espo_attach_cp(espo_ctx_t c, const void* cp_unique_id, int32_t cp_rank,
                           int32_t cp_world) {
  if (!c || cp_world < 1 || cp_rank < 0 || cp_rank >= cp_world) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->cp_world > 1 || c->state != State::Created) return ESPO_ERR_BAD_STATE;
  if (cp_unique_id) {
    if (!g_nccl.load()) return ESPO_ERR_NCCL;
    DevGuard g(c->device);
    nccl_uid id;
    std::memcpy(&id, cp_unique_id, sizeof(id));
    if (g_nccl.init_rank(&c->cp_comm, cp_world, id, cp_rank) != 0) {
      c->cp_comm = nullptr;
      return ESPO_ERR_NCCL;
    }
  }
  c->cp_rank = cp_rank;
  c->cp_world = cp_world;
  return ESPO_OK;
}

espo_status espo_cp_gather_local(espo_ctx_t c, const espo_ctx_t* ranks, int32_t cp_world,
                                 espo_stream_t stream) {
  ESPO_RANGE("espo_cp_gather_local");
  if (!c || !ranks || cp_world != c->cp_world || cp_world < 2 || ranks[c->cp_rank] != c)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (c->cp_comm || c->state != State::Prepared) return ESPO_ERR_BAD_STATE;
  for (int k = 0; k < cp_world; ++k)
    if (!ranks[k] || ranks[k]->device != c->device || ranks[k]->T != c->T ||
        ranks[k]->cp_rank != k || ranks[k]->state != State::Prepared)
      return ESPO_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  const int64_t tb = cp_block(c);
  for (int k = 0; k < cp_world; ++k) {
    if (k == c->cp_rank) continue;
    const int64_t lo = std::min(c->T, k * tb), n = std::min(c->T, (k + 1) * tb) - lo;
    if (n <= 0) continue;
    const Workspace& w = ranks[k]->ws;
    ESPO_CUDA(cudaMemcpyAsync(c->ws.lp + lo, w.lp + lo, n * 4, cudaMemcpyDeviceToDevice, s));
    ESPO_CUDA(cudaMemcpyAsync(c->ws.H + lo, w.H + lo, n * 4, cudaMemcpyDeviceToDevice, s));
    ESPO_CUDA(cudaMemcpyAsync(c->ws.old + lo, w.old + lo, n * 4, cudaMemcpyDeviceToDevice, s));
    ESPO_CUDA(cudaMemcpyAsync(c->ws.flag + lo, w.flag + lo, n, cudaMemcpyDeviceToDevice, s));
  }
  c->cp_gathered = true;
  return ESPO_OK;
}

namespace {
// K3 + the fixed-order K4 reduction into ws.red (the rank-local kRedLen fp64 terms); the CP
// all-gather of the per-token values K3 reads comes first.
espo_status reduce_local(espo_ctx_t c, cudaStream_t s) {
  if (c->cp_comm && c->T > 0) {
    // context parallelism: in-place all-gather of the per-token values K3 reads (13 B/token)
    const size_t tb = size_t(cp_block(c)), off = size_t(c->cp_rank) * tb;
    float* f32s[3] = {c->ws.lp, c->ws.H, c->ws.old};
    for (float* f : f32s)
      if (g_nccl.allgather(f + off, f, tb, kNcclFloat32, c->cp_comm, s) != 0) return ESPO_ERR_NCCL;
    if (g_nccl.allgather(c->ws.flag + off, c->ws.flag, tb, kNcclUint8, c->cp_comm, s) != 0)
      return ESPO_ERR_NCCL;
  }
  if (c->R > 0) {
    if (!c->single_pass || c->T == 0) {   // single-pass chunks ran K3 already
      k_seq_reduce<<<c->R, kSeqThreads, 0, s>>>(seq_params(c, 0, c->T));
      ESPO_LAUNCHED(c);
    }
    k_reduce_rollouts<<<kRedLen, 256, 0, s>>>(c->ws, c->R);
    ESPO_LAUNCHED(c);
  } else {
    ESPO_CUDA(cudaMemsetAsync(c->ws.red, 0, kRedLen * sizeof(double), s));
  }
  return ESPO_OK;
}

espo_status finalize_check(espo_ctx_t c) {
  const int64_t need = c->cp_world > 1 ? cp_hi(c) - cp_lo(c) : c->T;
  if (c->state != State::Prepared || c->n_covered != need) return ESPO_ERR_BAD_STATE;
  if (c->n_hsel != 0 && c->n_hsel != c->T) return ESPO_ERR_BAD_STATE;   // partial entropies
  if (c->cp_world > 1 && !c->cp_comm && !c->cp_gathered) return ESPO_ERR_BAD_STATE;
  return ESPO_OK;
}
}  // namespace

espo_status espo_loss_finalize(espo_ctx_t c, float* loss_dev, espo_stats* stats_dev,
                               espo_stream_t stream) {
  ESPO_RANGE("espo_loss_finalize");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  espo_status st = finalize_check(c);
  if (st != ESPO_OK) return st;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  const espo_config& cf = c->cfg;
  if ((st = reduce_local(c, s)) != ESPO_OK) return st;
  if (c->comm) {
    if (g_nccl.allreduce(c->ws.red, c->ws.red, kRedLen, kNcclFloat64, kNcclSum, c->comm, s) != 0)
      return ESPO_ERR_NCCL;
  }
  k_finalize_scalar<<<1, 1, 0, s>>>(c->ws, cf.norm, cf.logit_scale, loss_dev, stats_dev);
  ESPO_LAUNCHED(c);
  c->state = State::Finalized;
  return ESPO_OK;
}

espo_status espo_loss_reduce_local(espo_ctx_t c, double* partial_out, espo_stream_t stream) {
  ESPO_RANGE("espo_loss_reduce_local");
  if (!c || !partial_out) return ESPO_ERR_INVALID_ARGUMENT;
  espo_status st = finalize_check(c);
  if (st != ESPO_OK) return st;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  if ((st = reduce_local(c, s)) != ESPO_OK) return st;
  ESPO_CUDA(cudaMemcpyAsync(partial_out, c->ws.red, kRedLen * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
  c->state = State::Reduced;
  return ESPO_OK;
}

espo_status espo_loss_finalize_reduced(espo_ctx_t c, const double* reduced, float* loss_dev,
                                       espo_stats* stats_dev, espo_stream_t stream) {
  ESPO_RANGE("espo_loss_finalize_reduced");
  if (!c || !reduced) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Reduced) return ESPO_ERR_BAD_STATE;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  ESPO_CUDA(cudaMemcpyAsync(c->ws.red, reduced, kRedLen * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
  k_finalize_scalar<<<1, 1, 0, s>>>(c->ws, c->cfg.norm, c->cfg.logit_scale, loss_dev, stats_dev);
  ESPO_LAUNCHED(c);
  c->state = State::Finalized;
  return ESPO_OK;
}

}  // extern "C"

namespace {
espo_status check_bwd_args(espo_ctx_t c, const void* logits, int64_t ld, const void* dlogits,
                           int64_t ldg) {
  if (!logits || !dlogits) return ESPO_ERR_INVALID_ARGUMENT;
  const espo_config& cf = c->cfg;
  const size_t ei = dsize(cf.logits_dtype), eo = dsize(cf.grad_dtype);
  if (ld < shard_width(c) || ldg < shard_width(c)) return ESPO_ERR_INVALID_ARGUMENT;
  if (!aligned16(logits) || !aligned16(dlogits) || (size_t(ld) * ei) % 16 || (size_t(ldg) * eo) % 16)
    return ESPO_ERR_ALIGNMENT;
  if (logits == dlogits && (ld != ldg || ei != eo)) return ESPO_ERR_INVALID_ARGUMENT;
  return ESPO_OK;
}

// Rows of [b, e) that belong to rollouts whose group is not eliminated (an upper bound on the
// rows with gradient), from the host copy taken at prepare — or e − b if it has not landed.
int64_t candidate_rows(espo_ctx_t c, int64_t b, int64_t e, cudaStream_t s) {
  if (!c->prep_ev_set) return e - b;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();          // a capture-related query error must not leak into the
    return e - b;                // ESPO_LAUNCHED check of the launch that follows
  }
  const cudaError_t q = cudaEventQuery(c->prep_ev);
  if (q != cudaSuccess) {
    if (q != cudaErrorNotReady) cudaGetLastError();   // anything else: treat as not landed
    return e - b;
  }
  const int64_t* so = c->h_so;
  const int R = c->R;
  int i = static_cast<int>(std::upper_bound(so, so + R + 1, b) - so) - 1;   // rollout holding row b
  int64_t n = 0;
  for (i = std::max(i, 0); i < R && so[i] < e; ++i)
    if (c->h_cand[i]) n += std::max<int64_t>(0, std::min(e, so[i + 1]) - std::max(b, so[i]));
  return n;
}

// K5 over one chunk (arguments checked).
espo_status launch_bwd(espo_ctx_t c, const void* logits, int64_t ld, void* dlogits, int64_t ldg,
                       const float* grad_loss_dev, int64_t row_begin, int64_t n_rows,
                       cudaStream_t s) {
  const espo_config& cf = c->cfg;
  const bool aliased = logits == dlogits;
  // default: (row, tile) grid when every row is written; in compact mode (rows without
  // gradient untouched) tiles over the compact row lists, 8 rows per block (measured on C3)
  int impl = c->bwd_impl;
  if (impl == 0 && !cf.zero_fill_inactive_rows) impl = 10;
  BwdParams p;
  p.logits = logits;
  p.ld = ld;
  p.dlogits = dlogits;
  p.ldg = ldg;
  p.grad_loss = grad_loss_dev;
  p.row_begin = row_begin;
  p.n_rows = n_rows;
  p.V = shard_width(c);
  p.lam_log2e = cf.logit_scale * kLog2e;
  p.zero_fill = cf.zero_fill_inactive_rows;
  p.aliased = aliased ? 1 : 0;
  p.ws = c->ws;
  const bool bi = cf.logits_dtype == ESPO_BF16, bo = cf.grad_dtype == ESPO_BF16;
  BwdRec* list = static_cast<BwdRec*>(c->ws.list);
  int32_t* zl = c->ws.zlist;
  int* cnt = c->ws.count;
  const int pre_grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  if (impl == 0 || impl == 7 || impl == 8) {
    // tiled (default): per-row records indexed by row, non-persistent (row, tile) grid
    k_bwd_recs<<<pre_grid, 256, 0, s>>>(row_begin, n_rows, grad_loss_dev, p.zero_fill,
                                        shard_begin(c), p.V, c->ws, list);
    ESPO_LAUNCHED(c);
    const int epv = bi ? 8 : 4;
    const int nvec = (p.V + epv - 1) / epv;
    const int vpt = (impl == 7) ? 4 : 8;  // default 0: 32 KB tiles (measured best)
    const int ntiles = (nvec + 256 * vpt - 1) / (256 * vpt);
    const int64_t grid = n_rows * int64_t(ntiles);
    if (grid > INT32_MAX) return ESPO_ERR_INVALID_ARGUMENT;
    if (impl == 8) {   // the default tiles with scalar FP32 (A/B of the packed f32x2)
      if (bi && bo) k_dlogits_tile<__nv_bfloat16, __nv_bfloat16, 8, false><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else if (bi) k_dlogits_tile<__nv_bfloat16, float, 8, false><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else if (bo) k_dlogits_tile<float, __nv_bfloat16, 8, false><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else k_dlogits_tile<float, float, 8, false><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
    } else if (vpt == 4) {
      if (bi && bo) k_dlogits_tile<__nv_bfloat16, __nv_bfloat16, 4><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else if (bi) k_dlogits_tile<__nv_bfloat16, float, 4><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else if (bo) k_dlogits_tile<float, __nv_bfloat16, 4><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else k_dlogits_tile<float, float, 4><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
    } else {
      if (bi && bo) k_dlogits_tile<__nv_bfloat16, __nv_bfloat16, 8><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else if (bi) k_dlogits_tile<__nv_bfloat16, float, 8><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else if (bo) k_dlogits_tile<float, __nv_bfloat16, 8><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
      else k_dlogits_tile<float, float, 8><<<unsigned(grid), 256, 0, s>>>(p, list, ntiles);
    }
    ESPO_LAUNCHED(c);
    return ESPO_OK;
  }
  ESPO_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), s));
  k_bwd_rows<<<pre_grid, 256, 0, s>>>(row_begin, n_rows, grad_loss_dev, p.zero_fill, shard_begin(c),
                                      p.V, c->ws, list, zl, cnt);
  ESPO_LAUNCHED(c);
  if (impl >= 9) {   // tiled over the compact lists, RPB rows per block
    const int rpb = impl == 9 ? 4 : (impl == 10 ? 8 : 16);
    const int epv = bi ? 8 : 4;
    const int ntiles = (((p.V + epv - 1) / epv) + 256 * 8 - 1) / (256 * 8);
    // compact mode writes only rows with gradient: bound the grid by the candidate rows so
    // the blocks past the lists' end are not launched just to exit
    const int64_t bound = p.zero_fill ? n_rows : candidate_rows(c, row_begin, row_begin + n_rows, s);
    if (bound == 0) return ESPO_OK;
    const int64_t grid = (bound + rpb - 1) / rpb * int64_t(ntiles);
    if (grid > INT32_MAX) return ESPO_ERR_INVALID_ARGUMENT;
#define ESPO_TLIST(RPB)                                                                                    \
    if (bi && bo) k_dlogits_tlist<__nv_bfloat16, __nv_bfloat16, 8, RPB><<<unsigned(grid), 256, 0, s>>>(p, list, zl, cnt, ntiles); \
    else if (bi) k_dlogits_tlist<__nv_bfloat16, float, 8, RPB><<<unsigned(grid), 256, 0, s>>>(p, list, zl, cnt, ntiles);         \
    else if (bo) k_dlogits_tlist<float, __nv_bfloat16, 8, RPB><<<unsigned(grid), 256, 0, s>>>(p, list, zl, cnt, ntiles); \
    else k_dlogits_tlist<float, float, 8, RPB><<<unsigned(grid), 256, 0, s>>>(p, list, zl, cnt, ntiles);
    if (rpb == 4) { ESPO_TLIST(4) } else if (rpb == 8) { ESPO_TLIST(8) } else { ESPO_TLIST(16) }
#undef ESPO_TLIST
    ESPO_LAUNCHED(c);
    return ESPO_OK;
  }
  if (impl == 1) {
    if (bi && bo) {
      auto k = k_dlogits_ldg<__nv_bfloat16, __nv_bfloat16, 8>;
      k<<<grid_for(c, (const void*)k, 256), 256, 0, s>>>(p, list, zl, cnt);
    } else if (bi) {
      auto k = k_dlogits_ldg<__nv_bfloat16, float, 8>;
      k<<<grid_for(c, (const void*)k, 256), 256, 0, s>>>(p, list, zl, cnt);
    } else if (bo) {
      auto k = k_dlogits_ldg<float, __nv_bfloat16, 4>;
      k<<<grid_for(c, (const void*)k, 256), 256, 0, s>>>(p, list, zl, cnt);
    } else {
      auto k = k_dlogits_ldg<float, float, 4>;
      k<<<grid_for(c, (const void*)k, 256), 256, 0, s>>>(p, list, zl, cnt);
    }
  } else {
    cudaError_t le;
    const int v = impl;  // 2..5 geometry variants, 6 = 8 warps × 4 × 4 KB
    if (bi && bo) le = launch_dlogits_tma<__nv_bfloat16, __nv_bfloat16>(p, list, zl, cnt, c->num_sms, c->blocks_per_sm, v, s);
    else if (bi) le = launch_dlogits_tma<__nv_bfloat16, float>(p, list, zl, cnt, c->num_sms, c->blocks_per_sm, v, s);
    else if (bo) le = launch_dlogits_tma<float, __nv_bfloat16>(p, list, zl, cnt, c->num_sms, c->blocks_per_sm, v, s);
    else le = launch_dlogits_tma<float, float>(p, list, zl, cnt, c->num_sms, c->blocks_per_sm, v, s);
    if (le != cudaSuccess) return cuda_status(le);
  }
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

}  // namespace

extern "C" {

espo_status espo_loss_bwd(espo_ctx_t c, const void* logits, int64_t ld, void* dlogits, int64_t ldg,
                          const float* grad_loss_dev, int64_t row_begin, int64_t n_rows,
                          espo_stream_t stream) {
  ESPO_RANGE("espo_loss_bwd");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Finalized || c->single_pass) return ESPO_ERR_BAD_STATE;
  if (n_rows < 0 || n_rows > INT32_MAX || row_begin < 0 || row_begin + n_rows > c->T)
    return ESPO_ERR_INVALID_ARGUMENT;
  if (c->cp_world > 1 && n_rows > 0 && (row_begin < cp_lo(c) || row_begin + n_rows > cp_hi(c)))
    return ESPO_ERR_INVALID_ARGUMENT;   // a CP rank owns only its token block
  if (n_rows == 0) return ESPO_OK;
  espo_status st = check_bwd_args(c, logits, ld, dlogits, ldg);
  if (st != ESPO_OK) return st;
  DevGuard g(c->device);
  return launch_bwd(c, logits, ld, dlogits, ldg, grad_loss_dev, row_begin, n_rows, S(stream));
}

espo_status espo_set_entropies(espo_ctx_t c, const float* entropy, int64_t row_begin,
                               int64_t n_rows, espo_stream_t stream) {
  ESPO_RANGE("espo_set_entropies");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Prepared) return ESPO_ERR_BAD_STATE;
  if (c->single_pass || c->cp_world > 1) return ESPO_ERR_UNSUPPORTED;
  if (n_rows < 0 || row_begin < 0 || row_begin + n_rows > c->T) return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rows == 0) return ESPO_OK;
  if (!entropy) return ESPO_ERR_INVALID_ARGUMENT;
  const int64_t b = row_begin, e = row_begin + n_rows;
  auto it = c->hsel_cov.upper_bound(b);            // chunks must not overlap
  if (it != c->hsel_cov.begin() && std::prev(it)->second > b) return ESPO_ERR_BAD_STATE;
  if (it != c->hsel_cov.end() && it->first < e) return ESPO_ERR_BAD_STATE;
  DevGuard g(c->device);
  const size_t need = size_t(std::max<int64_t>(c->T, 1)) * sizeof(float);
  if (need > c->hsel_cap) {
    if (c->hsel) cudaFree(c->hsel);
    c->hsel = nullptr;
    c->hsel_cap = 0;
    ESPO_CUDA(cudaMalloc(&c->hsel, need));
    c->hsel_cap = need;
  }
  cudaStream_t s = S(stream);
  const int grid = int(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  k_set_entropies<<<grid, 256, 0, s>>>(entropy, c->hsel + row_begin, n_rows, c->ws.err);
  ESPO_LAUNCHED(c);
  c->hsel_cov[b] = e;
  c->n_hsel += n_rows;
  return ESPO_OK;
}

espo_status espo_set_mask(espo_ctx_t c, const uint8_t* mask, espo_stream_t stream) {
  ESPO_RANGE("espo_set_mask");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Prepared || c->n_covered != 0 || c->cp_world > 1) return ESPO_ERR_BAD_STATE;
  if (c->n_hsel != 0) return ESPO_ERR_UNSUPPORTED;   // supplied entropies: two-sweep mode only
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  if (c->R > 0) {
    k_mask_counts<<<c->R, 256, 0, s>>>(mask, c->ws, c->R);
    ESPO_LAUNCHED(c);
    k_mask_reduce<<<1, 256, 0, s>>>(c->ws, c->R);
    ESPO_LAUNCHED(c);
  } else {
    ESPO_CUDA(cudaMemsetAsync(c->ws.dpre, 0, 2 * sizeof(double), s));
  }
  if (c->comm) {
    if (g_nccl.allreduce(c->ws.dpre, c->ws.dpre, 2, kNcclFloat64, kNcclSum, c->comm, s) != 0)
      return ESPO_ERR_NCCL;
  }
  k_mask_scale<<<1, 1, 0, s>>>(c->ws, c->cfg.norm, c->cfg.logit_scale);
  ESPO_LAUNCHED(c);
  c->single_pass = true;
  return ESPO_OK;
}

espo_status espo_loss_fwd_bwd(espo_ctx_t c, const void* logits, int64_t ld, const int32_t* tokens,
                              const float* old_logp, void* dlogits, int64_t ldg,
                              const float* grad_loss_dev, int64_t row_begin, int64_t n_rows,
                              espo_stream_t stream) {
  ESPO_RANGE("espo_loss_fwd_bwd");
  espo_status st = check_fwd_args(c, logits, ld, tokens, old_logp, row_begin, n_rows, true);
  if (st != ESPO_OK) return st;
  if (n_rows == 0) return ESPO_OK;
  const bool sharded = c->cfg.vocab_local > 0 && c->cfg.vocab_local < c->cfg.vocab;
  if (sharded && !c->tp_comm && !c->tp_p2p) return ESPO_ERR_BAD_STATE;
  if ((st = check_bwd_args(c, logits, ld, dlogits, ldg)) != ESPO_OK) return st;
  if ((st = check_coverage(c, row_begin, row_begin + n_rows)) != ESPO_OK) return st;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  const int64_t row_end = row_begin + n_rows;
  k_check_chunk<<<1, 1, 0, s>>>(c->ws, row_begin, row_end, c->T);
  ESPO_LAUNCHED(c);
  if ((st = fwd_chunk(c, logits, ld, tokens, old_logp, c->ws.pmask + row_begin, row_begin, n_rows, s)) != ESPO_OK)
    return st;
  k_seq_reduce<<<c->R, kSeqThreads, 0, s>>>(seq_params(c, row_begin, row_end));
  ESPO_LAUNCHED(c);
  return launch_bwd(c, logits, ld, dlogits, ldg, grad_loss_dev, row_begin, n_rows, s);
}

espo_status espo_get_error(espo_ctx_t c, espo_stream_t stream) {
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return ESPO_ERR_CUDA;
  int err = 0;
  e = cudaMemcpy(&err, c->ws.err, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return ESPO_ERR_CUDA;
  e = cudaGetLastError();
  if (e != cudaSuccess) return ESPO_ERR_CUDA;
  return static_cast<espo_status>(err);
}

espo_status espo_export_token_stats(espo_ctx_t c, int64_t row_begin, int64_t n_rows, float* lse,
                                    float* lp, float* H, float* q, float* coef, uint8_t* bucket,
                                    uint8_t* clip, uint8_t* valid, espo_stream_t stream) {
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state == State::Created) return ESPO_ERR_BAD_STATE;
  if (n_rows < 0 || row_begin < 0 || row_begin + n_rows > c->T) return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rows == 0) return ESPO_OK;
  DevGuard g(c->device);
  const int grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, 4096));
  k_export_tokens<<<grid, 256, 0, S(stream)>>>(c->ws, row_begin, n_rows, lse, lp, H, q, coef,
                                                bucket, clip, valid);
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

espo_status espo_export_rollout_stats(espo_ctx_t c, double* adv, uint8_t* zv, uint8_t* active,
                                      double* J_i, int32_t* nb, float* theta, espo_stream_t stream) {
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state == State::Created) return ESPO_ERR_BAD_STATE;
  if (c->R == 0) return ESPO_OK;
  DevGuard g(c->device);
  k_export_rollouts<<<(c->R + 255) / 256, 256, 0, S(stream)>>>(c->ws, c->R, adv, zv, active, J_i,
                                                                 nb, theta);
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

}  // extern "C"

extern "C" {

espo_status espo_loss_fwd_factored(espo_ctx_t c, const void* logits, int64_t ld,
                                   const int32_t* tokens, const float* old_logp,
                                   const uint8_t* mask, void* grad, int64_t ldg, int64_t row_begin,
                                   int64_t n_rows, espo_stream_t stream) {
  ESPO_RANGE("espo_loss_fwd_factored");
  espo_status st = check_fwd_args(c, logits, ld, tokens, old_logp, row_begin, n_rows);
  if (st != ESPO_OK || n_rows == 0) return st;
  if (c->cfg.vocab_local > 0 && c->cfg.vocab_local < c->cfg.vocab) return ESPO_ERR_BAD_STATE;
  if ((st = check_bwd_args(c, logits, ld, grad, ldg)) != ESPO_OK) return st;
  if ((st = check_coverage(c, row_begin, row_begin + n_rows)) != ESPO_OK) return st;
  DevGuard g(c->device);
  cudaStream_t s = S(stream);
  const espo_config& cf = c->cfg;
  FwdParams p;
  p.logits = logits;
  p.ld = ld;
  p.tokens = tokens;
  p.old_logp = old_logp;
  p.mask = mask;
  p.row_begin = row_begin;
  p.n_rows = n_rows;
  p.V = cf.vocab;
  p.lam_log2e = cf.logit_scale * kLog2e;
  p.partial = nullptr;
  p.ws = c->ws;
  const bool bi = cf.logits_dtype == ESPO_BF16, bo = cf.grad_dtype == ESPO_BF16;
  FwdRec* list = static_cast<FwdRec*>(c->ws.list);
  int32_t* zl = cf.zero_fill_inactive_rows ? c->ws.zlist : nullptr;
  ESPO_CUDA(cudaMemsetAsync(c->ws.count, 0, 3 * sizeof(int), s));
  const int pre_grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  if (bi)
    k_fwd_rows<__nv_bfloat16><<<pre_grid, 256, 0, s>>>(logits, ld, tokens, old_logp, mask, row_begin,
                                                       n_rows, cf.vocab, 0, cf.vocab, p.lam_log2e,
                                                       c->ws, list, c->ws.count, zl);
  else
    k_fwd_rows<float><<<pre_grid, 256, 0, s>>>(logits, ld, tokens, old_logp, mask, row_begin, n_rows,
                                               cf.vocab, 0, cf.vocab, p.lam_log2e, c->ws, list,
                                               c->ws.count, zl);
  ESPO_LAUNCHED(c);
  const int al = logits == grad ? 1 : 0;
  // geometry (ESPO_OPT_FACTORED_IMPL): 0 = TMA ring, 20 consumer warps + 1 producer warp,
  // 5 × 40 KB slots (measured best); 1 = CTA of 1024 threads re-reading each row
  // through L2 with plain loads; 2 = 16 warps × 6 × 32 KB; 3 = the default with the TMEM
  // stash of pass 1's exponentials; 4, 5 = two CTAs per SM (thrash the L2); 6 = rolling
  // interleave of pass 2 (row k−1) with pass 1 (row k) (longer L2 reuse distance: slower)
#define ESPO_FG(NT, U)                                                                     \
  {                                                                                            \
    const int grid = c->num_sms * (1024 / NT);                                                  \
    if (bi && bo) k_fwd_grad<__nv_bfloat16, __nv_bfloat16, NT, U><<<grid, NT, 0, s>>>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al); \
    else if (bi) k_fwd_grad<__nv_bfloat16, float, NT, U><<<grid, NT, 0, s>>>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al);         \
    else if (bo) k_fwd_grad<float, __nv_bfloat16, NT, U><<<grid, NT, 0, s>>>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al);         \
    else k_fwd_grad<float, float, NT, U><<<grid, NT, 0, s>>>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al);                         \
  }
#define ESPO_FGR(NC, ST, CH, TM, CPS)                                                           \
  {                                                                                            \
    cudaError_t le;                                                                            \
    if (bi && bo) le = launch_fwd_grad_ring<__nv_bfloat16, __nv_bfloat16, NC, ST, CH, TM>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al, c->num_sms, s, CPS); \
    else if (bi) le = launch_fwd_grad_ring<__nv_bfloat16, float, NC, ST, CH, TM>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al, c->num_sms, s, CPS);         \
    else if (bo) le = launch_fwd_grad_ring<float, __nv_bfloat16, NC, ST, CH, TM>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al, c->num_sms, s, CPS);         \
    else le = launch_fwd_grad_ring<float, float, NC, ST, CH, TM>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al, c->num_sms, s, CPS);                         \
    if (le != cudaSuccess) return cuda_status(le);                                             \
  }
#define ESPO_FGL(NC, ST, CH)                                                                   \
  {                                                                                            \
    cudaError_t le;                                                                            \
    if (bi && bo) le = launch_fwd_grad_roll<__nv_bfloat16, __nv_bfloat16, NC, ST, CH>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al, c->num_sms, s); \
    else if (bi) le = launch_fwd_grad_roll<__nv_bfloat16, float, NC, ST, CH>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al, c->num_sms, s);         \
    else if (bo) le = launch_fwd_grad_roll<float, __nv_bfloat16, NC, ST, CH>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al, c->num_sms, s);         \
    else le = launch_fwd_grad_roll<float, float, NC, ST, CH>(p, list, c->ws.zlist, c->ws.count, grad, ldg, al, c->num_sms, s);                         \
    if (le != cudaSuccess) return cuda_status(le);                                             \
  }
  switch (c->factored_impl) {
    case 6: ESPO_FGL(20, 5, 40960) break;
    case 1: ESPO_FG(1024, 4) break;
    case 2: ESPO_FGR(16, 6, 32768, 0, 1) break;
    case 3: ESPO_FGR(20, 5, 40960, 1, 1) break;
    case 4: ESPO_FGR(10, 5, 20480, 0, 2) break;
    case 5: ESPO_FGR(12, 4, 24576, 0, 2) break;
    default: ESPO_FGR(20, 5, 40960, 0, 1) break;
  }
#undef ESPO_FG
#undef ESPO_FGR
#undef ESPO_FGL
  ESPO_LAUNCHED(c);
  c->covered[row_begin] = row_begin + n_rows;
  c->n_covered += n_rows;
  return ESPO_OK;
}

espo_status espo_loss_row_scale(espo_ctx_t c, const float* grad_loss_dev, float* scale_out,
                                int64_t row_begin, int64_t n_rows, espo_stream_t stream) {
  ESPO_RANGE("espo_loss_row_scale");
  if (!c) return ESPO_ERR_INVALID_ARGUMENT;
  if (c->state != State::Finalized) return ESPO_ERR_BAD_STATE;
  if (n_rows < 0 || row_begin < 0 || row_begin + n_rows > c->T) return ESPO_ERR_INVALID_ARGUMENT;
  if (n_rows == 0) return ESPO_OK;
  if (!scale_out) return ESPO_ERR_INVALID_ARGUMENT;
  DevGuard g(c->device);
  const int grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, int64_t(c->num_sms) * 8));
  k_row_scale<<<grid, 256, 0, S(stream)>>>(row_begin, n_rows, grad_loss_dev, c->ws, scale_out);
  ESPO_LAUNCHED(c);
  return ESPO_OK;
}

}  // extern "C"
