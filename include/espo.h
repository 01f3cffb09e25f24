/*
 * espo.h — C ABI (v1) of libespo: the ESPO policy-loss pass of arXiv 2512.07710
 * ("Each Prompt Matters", §2.4.1 Multi-Stage Zero-Variance Elimination and §2.4.2 ESPO),
 * forward and backward, on NVIDIA B200 (sm_100a).
 *
 * What the library computes (citations: PAPER.md line + section/equation):
 *   - prompt groups, zero-variance (ZV) mask and GRPO advantages
 *       PAPER.md:77-79 (§2.4.1 "all rollouts receive identical rewards ... zero advantage");
 *       PAPER.md:105-107 (§2.4.2 normalised advantage Â, GRPO group normalisation)
 *   - per-token log-prob of the sampled token and token entropy from vocab-wide logits
 *       PAPER.md:111 (Eq. 1 numerator π_θ(y_t|x,y_<t)); PAPER.md:119-121 (Eq. 3 e_t, log|V|)
 *   - per-sequence entropy buckets τ, the length-normalised bucket ratio s_τ (Eq. 2,
 *     PAPER.md:115) and the entropy-adaptive clip ε_τ (Eq. 3)
 *   - the clipped surrogate J_ESPO with the stop-gradient token ratio
 *     (Eq. 1), loss = −J, and d loss / d logits.
 * Readings of silent/garbled passages are listed in DESIGN.md ("Readings", Q1-Q21);
 * the config fields below name the reading they select.
 *
 * Call order per training step (one context per GPU / rank):
 *   espo_prepare  →  espo_loss_fwd on chunks covering every token row exactly once
 *   (any order; a chunk may split a sequence)  →  espo_loss_finalize  →
 *   espo_loss_bwd on chunks (any order, any number of times).
 * Every call is asynchronous on the given CUDA stream; the only host↔device
 * synchronisation is espo_get_error. With world > 1, espo_loss_finalize issues the one
 * NCCL all-reduce of the pass (global active-rollout / token counts and loss terms).
 * Other modes (declared below): single pass (espo_set_mask + espo_loss_fwd_bwd on chunks of
 * whole rollouts), the fused LM head (espo_lmhead_fwd / espo_lmhead_bwd: logits never
 * materialised), vocabulary parallelism (partial + combine, NCCL all-gather, or the fused
 * peer-memory exchange), context parallelism (espo_attach_cp) and reward reshaping.
 *
 * Layout: token rows are packed (cu_seqlens): rollout i owns rows
 * [seq_offsets[i], seq_offsets[i+1]). Logits row t is the distribution that produced
 * tokens[t] (the caller applies the usual one-position shift). A padded [R, L] batch is
 * seq_offsets[i] = i·L with mask = 0 on padding. Logits/dlogits are row-major with a
 * leading dimension `ld`/`ldg` (elements) ≥ vocab.
 *
 * Ownership: all pointer arguments are caller-owned; "device" pointers must be CUDA
 * device memory of the context's device, "host" pointers host memory. Inputs of a chunk
 * call are read before the call's work completes on the stream; the context keeps what
 * it needs (per-token workspace ≈ 72 B/token, per-rollout arrays) until the next prepare.
 *
 * Errors: host-detectable problems (NULL, sizes, alignment, call order, chunk overlap)
 * return a status immediately and enqueue nothing. Data problems found on the device
 * (NaN/+inf logit in a row that is read, non-finite reward, token ∉ [0, vocab), a target
 * logit of −inf, non-contiguous group ids, inconsistent seq_offsets) set a sticky device
 * error word: espo_loss_finalize then writes a NaN loss, and espo_get_error returns the
 * code. Rows of eliminated (ZV) groups and masked rows are never read (garbage is legal).
 * No C++ exception crosses this ABI and nothing aborts. A context is not thread-safe;
 * distinct contexts are independent.
 */
#ifndef ESPO_H_
#define ESPO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESPO_ABI_VERSION 1
#define ESPO_MAX_BUCKETS 4
#define ESPO_UNIQUE_ID_BYTES 128

typedef struct espo_ctx_s* espo_ctx_t;
/* Same type as cudaStream_t; NULL = the legacy default stream. */
typedef struct CUstream_st* espo_stream_t;

typedef enum {
  ESPO_OK = 0,
  ESPO_ERR_INVALID_ARGUMENT = 1,     /* NULL pointer, bad size/enum, chunk outside [0,T) */
  ESPO_ERR_ALIGNMENT = 2,            /* logits/dlogits base or row pitch not 16-byte aligned */
  ESPO_ERR_GROUPS_NOT_CONTIGUOUS = 3,/* group_ids decrease somewhere (device-detected) */
  ESPO_ERR_BAD_STATE = 4,            /* call order violated, rows uncovered or covered twice */
  ESPO_ERR_NONFINITE_INPUT = 5,      /* NaN/+inf logit, −inf target logit, non-finite reward */
  ESPO_ERR_TOKEN_OUT_OF_RANGE = 6,   /* tokens[t] ∉ [0, vocab) */
  ESPO_ERR_OUT_OF_MEMORY = 7,
  ESPO_ERR_CUDA = 8,
  ESPO_ERR_NCCL = 9,
  ESPO_ERR_UNSUPPORTED = 10,
  ESPO_ERR_BLAS = 11,                /* libcublas missing or a cuBLAS call failed */
  ESPO_ERR_PEER_TIMEOUT = 12         /* a TP peer never signalled its partials (peer-memory mode) */
} espo_status;

typedef enum { ESPO_F32 = 0, ESPO_BF16 = 1 } espo_dtype;

/* Eq. 1 denominator reading (Q1). R2 (default): sg[π_θ] as in GSPO-token, so the
 * token ratio's value is s_τ and a singleton bucket is token-level PPO. R1: the printed
 * sg[π_θold] literally, value s_τ·π_θ/π_old. */
typedef enum { ESPO_RATIO_GSPO_TOKEN = 0, ESPO_RATIO_LITERAL_OLD = 1 } espo_ratio_mode;

/* Token grouping (Q3). QUANTILE: per sequence, K buckets split at the K−1 entropy order
 * statistics (K=2: rank ⌊split_num·n/split_den⌋, the 80/20 rule of PAPER.md:95; ties to
 * the lower bucket). WHOLE: one bucket (GSPO-token). SINGLETON: one bucket per token. */
typedef enum { ESPO_PART_QUANTILE = 0, ESPO_PART_WHOLE = 1, ESPO_PART_SINGLETON = 2 } espo_partition;

/* Normaliser (Q2, Q10). SEQ: J = (1/N_active_rollouts) Σ_i (1/nb_i) Σ_τ (1/|y_τ|) Σ_t ℓ_t
 * (PAPER.md:105). TOKEN: J = (1/T_active) Σ_t ℓ_t. */
typedef enum { ESPO_NORM_SEQ = 0, ESPO_NORM_TOKEN = 1 } espo_norm;

/* Zero-variance groups (§2.4.1). MASK (default, north_star): eliminated — Â = 0, rows never
 * read, not counted in N. RLZVP: ZVE stage 3 "advantage reshaping" with the
 * RL-ZVP instantiation of SPEC.md:338-343 — the group's rows are read and token t of rollout
 * i gets Â_t = β·s·(e_t − ē_i)/log|V|, s = +1 if the group's reward < zvp_threshold else −1,
 * ē_i the rollout's mean token entropy; such rollouts count in N. */
typedef enum { ESPO_ZV_MASK = 0, ESPO_ZV_RLZVP = 1 } espo_zv_mode;

typedef struct {
  int32_t vocab;               /* V: row width; log|V| of Eq. 3 (Q6) */
  float alpha;                 /* Eq. 3 α (Q5), default 0.4 */
  float eps_min;               /* floor on ε_τ (Q5), default 0.01; 0 = paper-literal */
  int32_t n_buckets;           /* K ∈ [1, 4], default 2 */
  int32_t split_num, split_den;/* K=2 split fraction, default 4/5 */
  int32_t partition;           /* espo_partition */
  int32_t ratio_mode;          /* espo_ratio_mode */
  int32_t norm;                /* espo_norm */
  int32_t std_unbiased;        /* 0 (default): population std (Q7) */
  double adv_eps;              /* Â = (r−μ)/(σ + adv_eps), default 1e-6 (Q7) */
  double zv_var_eps;           /* 0 (default): ZV iff all rewards compare equal (Q8);
                                  > 0: ZV iff fp64 two-pass variance ≤ zv_var_eps */
  float logit_scale;           /* λ = 1/temperature applied to logits (Q15), default 1 */
  float log_ratio_clamp;       /* clamp of the Eq. 2 mean log-ratio (Q14), default 20; 0=off */
  int32_t logits_dtype;        /* espo_dtype of logits */
  int32_t grad_dtype;          /* espo_dtype of dlogits: any of f32 / bf16 for either logits dtype */
  int32_t zero_fill_inactive_rows; /* 1 (default): bwd writes 0 to rows of masked tokens,
                                      ZV groups and clipped tokens; 0: leaves them as-is */
  int32_t zv_mode;             /* espo_zv_mode, default MASK */
  float zvp_beta;              /* RL-ZVP β, default 0.05 (|Â_t| ≤ β) */
  float zvp_threshold;         /* RL-ZVP success threshold on the uniform reward, default 0.5 */
  int32_t vocab_begin;         /* vocabulary-parallel shard: this context's logits chunks hold */
  int32_t vocab_local;         /* columns [vocab_begin, vocab_begin + vocab_local) of the full
                                  `vocab`; vocab_local = 0 (default): unsharded */
  int32_t reserved[2];
} espo_config;

/* Device-written statistics (all fp64). Per-bucket arrays are indexed by the pre-drop
 * bucket id k (0 = lowest entropy); WHOLE and SINGLETON report everything in k = 0. */
typedef struct {
  double loss;
  double n_active_rollouts;    /* N: rollouts of non-ZV groups with ≥ 1 valid token */
  double n_active_tokens;      /* T_active */
  double n_zv_groups;          /* eliminated prompt groups (ZV ratio) */
  double n_groups;
  double n_clipped_tokens;     /* tokens whose clipped branch zeroes the gradient */
  double mean_abs_logratio;    /* mean |log π_θ − log π_old| (mismatch) */
  double mean_entropy;         /* mean e_t over active tokens (nats) */
  double clip_frac[ESPO_MAX_BUCKETS];
  double mean_ratio[ESPO_MAX_BUCKETS];   /* token-weighted mean of the ratio value */
  double mean_eps[ESPO_MAX_BUCKETS];     /* token-weighted mean of ε_τ */
  double tokens_per_bucket[ESPO_MAX_BUCKETS];
  /* train/inference mismatch of the rollout-engine log-probs (§2.4.4 Router
   * Replay; Δ_t = log π_θ(y_t) − log π_old(y_t) over active tokens): */
  double mean_sq_logratio;     /* mean Δ² */
  double mean_k3;              /* mean (e^Δ − 1 − Δ): k3 estimate of KL(π_old ‖ π_θ) */
} espo_stats;

/* Fills *cfg with the defaults listed above for the given vocab (bf16 logits and grads). */
void espo_config_default(espo_config* cfg, int32_t vocab);

/* Writes a fresh NCCL unique id (ESPO_UNIQUE_ID_BYTES bytes, host memory) for rank 0 to
 * broadcast to the other ranks before espo_create. Loads libnccl.so.2 on first use. */
espo_status espo_get_unique_id(void* out_id);

/* Creates a context on CUDA device `cuda_device`. world == 1: nccl_unique_id must be
 * NULL and NCCL is never touched. world > 1: collective over all ranks (ncclCommInitRank
 * with the broadcast id, host memory). cfg is copied. */
espo_status espo_create(const espo_config* cfg, const void* nccl_unique_id, int32_t rank,
                        int32_t world, int32_t cuda_device, espo_ctx_t* out);
espo_status espo_destroy(espo_ctx_t ctx);

/* Step begin (K1 kernels) — §2.4.1 zero-variance elimination and §2.4.2's advantage.
 * Operation: prompt groups are the maximal runs of equal group_ids (the G rollouts
 * {y_i} ~ π_old of one prompt); a group whose rewards all compare equal (or
 * G = 1) has zero variance and is eliminated ("identical rewards … zero
 * advantage", masked out per PAPER.md:91 / north_star; reading Q8); every other rollout gets
 * the GRPO advantage Â_i = (r_i − μ_g)/(σ_g + adv_eps) ("normalized
 * token-level advantage", formula SPEC.md:335; population std, reading Q7), in fp64.
 * Device inputs: rewards f32[R], group_ids i32[R] (each prompt
 * group is one run of equal ids; ids must be non-decreasing), seq_offsets i64[R+1] with
 * seq_offsets[0] = 0, non-decreasing, seq_offsets[R] = n_tokens. Outputs (device,
 * nullable): adv_out f32[R] (0 for ZV groups), zv_out u8[R] (1 = eliminated group).
 * Resets the sticky error word and the chunk coverage; may grow the workspace
 * (the only call that allocates). With zero_fill_inactive_rows = 0 (compact mode) it also
 * enqueues an asynchronous copy of seq_offsets and the eliminated-group flags into pinned
 * host memory owned by the context (8·(R+1) + R bytes, grown on demand); espo_loss_bwd uses
 * it, once it has landed, only to size its grid (results do not depend on it). Under CUDA
 * stream capture the copy is skipped (the backward grid then covers whole chunks).
 * Errors: NULL input / negative sizes → ESPO_ERR_INVALID_ARGUMENT (nothing enqueued);
 * non-finite reward, decreasing group_ids, inconsistent seq_offsets → sticky device error. */
espo_status espo_prepare(espo_ctx_t ctx, const float* rewards, const int32_t* group_ids,
                         const int64_t* seq_offsets, int32_t n_rollouts, int64_t n_tokens,
                         float* adv_out, uint8_t* zv_out, espo_stream_t stream);

/* Forward sweep over token rows [row_begin, row_begin + n_rows) (K2).
 * Operation: for each row t of an active rollout with mask = 1, one pass over the vocabulary
 * gives lse_t = log Σ_v e^{λz_v}, the log-prob of the sampled token lp_t = λz_{y_t} − lse_t
 * (the Eq. 1 numerator log π_θ(y_t|x, y_<t)), the token entropy
 * e_t = −Σ_v p_v log p_v (Eq. 3's e_t) and q_t = 1 − p_{y_t}; rows of
 * eliminated groups and masked rows are not read. Device inputs,
 * each pointing at row row_begin: logits (dtype cfg.logits_dtype, 16-byte aligned,
 * ld·sizeof(dtype) % 16 == 0, ld ≥ vocab), tokens i32, old_logp f32 (rollout-engine
 * log π_old, nats), mask u8 (nullable = all valid). flags must be 0. Chunks may come in any
 * order and may split a rollout; every row exactly once before espo_loss_finalize.
 * Errors: NULL / misaligned / overlapping chunk → immediate status (nothing enqueued);
 * NaN/+inf logit, −inf target logit, token ∉ [0, vocab) in a read row → sticky device error. */
espo_status espo_loss_fwd(espo_ctx_t ctx, const void* logits, int64_t ld,
                          const int32_t* tokens, const float* old_logp, const uint8_t* mask,
                          int64_t row_begin, int64_t n_rows, uint32_t flags,
                          espo_stream_t stream);

/* After all rows are covered: K3 per sequence, K4 reduction, NCCL all-reduce when world > 1.
 * Operation (§2.4.2): within each rollout the valid tokens are grouped by
 * entropy (K = 2 split at the 80/20 order statistic of PAPER.md:95, reading Q3);
 * per bucket τ, s_τ = exp(mean_{t∈τ}(lp_t − old_t)) (Eq. 2) and
 * ε_τ = max(ε_min, α·mean_{t∈τ} e_t / log|V|) (Eq. 3); per token the clipped
 * surrogate ℓ_t = min(v_t·Â, clip(v_t, 1 ± ε_τ)·Â) with v_t = s_τ (Eq. 1, reading R2);
 * J_i = (1/|τ|)·Σ_τ (1/|y_τ|)·Σ_{t∈τ} ℓ_t and loss = −(1/N)·Σ_i J_i over the N active
 * rollouts (J_ESPO; readings Q2, Q10, Q13). The N and Σ J_i terms (26 fp64) are
 * summed over the DP ranks by one ncclAllReduce. Device outputs, nullable: loss_dev f32[1]
 * (= −J; 0 when no rollout is active; NaN after a device-detected data error), stats_dev
 * espo_stats. Errors: rows not covered / wrong call order → ESPO_ERR_BAD_STATE; NCCL failure
 * → ESPO_ERR_NCCL. */
espo_status espo_loss_finalize(espo_ctx_t ctx, float* loss_dev, espo_stats* stats_dev,
                               espo_stream_t stream);

/* espo_loss_finalize in two halves, for a caller-owned collective (torch.distributed, MPI,
 * a different NCCL communicator) or none. espo_loss_reduce_local runs K3 and the fixed-order
 * K4 reduction and copies this rank's ESPO_REDUCE_LEN fp64 terms to partial_out (device);
 * the caller sums those vectors element-wise over its ranks and passes the sum to
 * espo_loss_finalize_reduced (device, ESPO_REDUCE_LEN fp64), which writes loss/stats like
 * espo_loss_finalize and fixes the backward scale −grad·c_t/N. With the sum of every rank's
 * vector, each rank's dlogits rows are bitwise those of a single context holding all ranks'
 * rollouts (N is an integer count; only the fp64 loss sum depends on the reduction order).
 * The context's own communicator (world > 1) is not used by this pair. States: Prepared with
 * all rows covered → reduce_local → finalize_reduced → bwd; otherwise ESPO_ERR_BAD_STATE. */
#define ESPO_REDUCE_LEN 26
espo_status espo_loss_reduce_local(espo_ctx_t ctx, double* partial_out, espo_stream_t stream);
espo_status espo_loss_finalize_reduced(espo_ctx_t ctx, const double* reduced, float* loss_dev,
                                       espo_stats* stats_dev, espo_stream_t stream);

/* Backward sweep (K5): dlogits = d(grad_loss · loss)/d logits for rows
 * [row_begin, row_begin+n_rows). Operation: only the Eq. 1 numerator π_θ(y_t) carries
 * gradient — every sg[·] is a constant — so row t gets
 * λ·g_t·(onehot(y_t) − softmax(λz_t)) with g_t = −grad_loss·c_t/N, c_t = ∂J_i/∂lp_t =
 * κ_t·Â·v_t/(|τ|·|y_τ|) (κ_t = 0 where the clipped branch of the min is strictly active);
 * rows with c_t = 0 (clipped, masked, eliminated) are written as zeros without being read
 * (or left untouched in compact mode). logits as in espo_loss_fwd (the same values);
 * dlogits (device, cfg.grad_dtype, 16-byte aligned, ldg ≥ vocab) may alias logits when
 * ldg == ld and the dtypes match. grad_loss_dev: device f32[1], nullable = 1.0.
 * Errors: before finalize → ESPO_ERR_BAD_STATE; NULL / misaligned → immediate status. */
espo_status espo_loss_bwd(espo_ctx_t ctx, const void* logits, int64_t ld, void* dlogits,
                          int64_t ldg, const float* grad_loss_dev, int64_t row_begin,
                          int64_t n_rows, espo_stream_t stream);

/* ---- ZVE stage 2: reward reshaping ----
 * final_i = base_i + length_penalty_i + repetition_penalty_i for rollout i with response
 * tokens tokens[seq_offsets[i] .. seq_offsets[i+1]) (device). length_penalty = 0 if
 * len ≤ max_len − buffer, −(len − (max_len − buffer))/buffer on the ramp, −1 from max_len on;
 * repetition_penalty = −gamma_rep·max(0, f − rep_thresh), f = fraction of the len − ngram + 1
 * positions whose n-gram occurred earlier in the response. Arithmetic in fp64, results f32.
 * Run before espo_prepare (the reshaped rewards feed the zero-variance test). May allocate
 * scratch (12 B × 4 × n_tokens) on first use or growth. */
typedef struct {
  int32_t max_len;      /* ≥ 1 */
  int32_t buffer;       /* ramp length; 0 = ⌈max_len / 8⌉ */
  int32_t ngram;        /* 1..16, default 4 */
  float gamma_rep;      /* default 1.0 */
  float rep_thresh;     /* default 0.2 */
  int32_t reserved[3];
} espo_reward_shaping;
void espo_reward_shaping_default(espo_reward_shaping* p, int32_t max_len);
espo_status espo_reshape_rewards(espo_ctx_t ctx, const espo_reward_shaping* params,
                                 const float* base_rewards, const int32_t* tokens,
                                 const int64_t* seq_offsets, int32_t n_rollouts,
                                 int64_t n_tokens, float* rewards_out, float* len_pen_out,
                                 float* rep_pen_out, espo_stream_t stream);

/* ---- vocabulary-parallel ESPO (logits sharded by vocabulary over TP ranks) ----
 * With cfg.vocab_local > 0 every rank holds the same token rows but only its vocabulary
 * columns. The forward sweep then produces, per row, a 16-byte partial
 * {R, S, W, u_y} (base-2 reference, Σ_{v≠y} 2^{u_v−R}, Σ 2^{u_v−R}(u_v−R) over the local
 * columns, and λ·log2(e)·z_y on the rank owning the target, NaN elsewhere); the partials of
 * all shards are combined into the exact row statistics (lse, lp, H, q). The backward sweep
 * writes the local columns of dlogits (no collective). */

/* Forward sweep of the local shard → partials (device f32[n_rows·4]); no coverage update. */
espo_status espo_loss_fwd_partial(espo_ctx_t ctx, const void* logits, int64_t ld,
                                  const int32_t* tokens, const float* old_logp,
                                  const uint8_t* mask, int64_t row_begin, int64_t n_rows,
                                  float* partial, espo_stream_t stream);
/* Combines partials laid out [n_shards][n_rows][4] (device) into the row statistics and
 * records the rows as covered (the same call order rules as espo_loss_fwd). */
espo_status espo_loss_fwd_combine(espo_ctx_t ctx, const float* partials, int32_t n_shards,
                                  int64_t row_begin, int64_t n_rows, espo_stream_t stream);
/* Attaches a tensor-parallel NCCL communicator (collective over the TP ranks, id broadcast by
 * the caller). Afterwards espo_loss_fwd on this context runs partial → ncclAllGather of the
 * partials over the TP group → combine. The DP all-reduce of espo_loss_finalize stays on the
 * communicator given to espo_create. */
espo_status espo_attach_tp(espo_ctx_t ctx, const void* tp_unique_id, int32_t tp_rank,
                           int32_t tp_world);

/* ---- vocabulary-parallel partial exchange over peer memory (NVLink / NVSwitch) ----
 * The alternative to espo_attach_tp: instead of partial sweep → ncclAllGather → combine, the
 * forward sweep's own epilogue stores each row's 16-byte partial {R, S, W, u_y} into the
 * exchange buffer of EVERY TP rank (peer pointers from CUDA IPC), then releases a flag per
 * rank; the combine acquires all ranks' flags for the chunk and merges (PAPER.md:129 Megatron
 * vocab-parallel layout). Two slots alternate between chunks; a slot is
 * rewritten only after every rank posted that it consumed it. Waits are bounded in wall time
 * (ESPO_OPT_PEER_TIMEOUT_MS, default 120 s): a missing peer gives ESPO_ERR_PEER_TIMEOUT
 * (sticky, via espo_get_error) and an invalid step, not a hang.
 *
 * espo_tp_p2p_buffer: allocates this rank's exchange buffer for chunks of ≤ max_rows rows
 *   (4 KB flags + 2·tp_world·max_rows·16 B) and writes its cudaIpcMemHandle_t
 *   (ESPO_IPC_HANDLE_BYTES, nullable) — the caller all-gathers the handles over its TP group.
 * espo_tp_p2p_open: maps the peers' buffers (handles laid out [tp_world][64], own ignored).
 * espo_tp_p2p_connect_local: same-device variant for tests and single-GPU emulation: `ranks`
 *   are the tp_world contexts (one per shard) on this device, each with its buffer allocated.
 * espo_loss_fwd_p2p_send / _recv: the two halves of a chunk's forward (send: wait until the
 *   slot is free, fused sweep + stores, signal; recv: wait for all ranks, combine, post
 *   consumed; records coverage). espo_loss_fwd on a connected context runs both. Every rank
 *   must process the same chunks in the same order. */
#define ESPO_IPC_HANDLE_BYTES 64
espo_status espo_tp_p2p_buffer(espo_ctx_t ctx, int64_t max_rows, int32_t tp_world,
                               void* ipc_handle_out);
espo_status espo_tp_p2p_open(espo_ctx_t ctx, const void* ipc_handles, int32_t tp_rank,
                             int32_t tp_world);
espo_status espo_tp_p2p_connect_local(espo_ctx_t ctx, const espo_ctx_t* ranks, int32_t tp_rank,
                                      int32_t tp_world);
/* Disconnects: unmaps the peers' buffers (call on every rank, then synchronise the ranks,
 * before any rank destroys its context — an exporter must outlive the mappings of it). */
espo_status espo_tp_p2p_unmap(espo_ctx_t ctx);
espo_status espo_loss_fwd_p2p_send(espo_ctx_t ctx, const void* logits, int64_t ld,
                                   const int32_t* tokens, const float* old_logp,
                                   const uint8_t* mask, int64_t row_begin, int64_t n_rows,
                                   espo_stream_t stream);
espo_status espo_loss_fwd_p2p_recv(espo_ctx_t ctx, int64_t row_begin, int64_t n_rows,
                                   espo_stream_t stream);

/* ---- context parallelism (long-CoT rollouts split across ranks by token blocks) ----
 * SURVEY §8(f) row 3's sibling: CP rank k owns the packed token rows [k·Tb, min(T,(k+1)·Tb)),
 * Tb = ⌈T / cp_world⌉ (sequences are cut anywhere). Each rank sweeps only its rows (fwd and
 * bwd calls outside the block → ESPO_ERR_INVALID_ARGUMENT). At espo_loss_finalize the per-token
 * values the per-rollout reduction reads — lp, H, old_logp (f32) and the valid flag (u8):
 * 13 B/token, negligible next to the 2V-byte logits rows — are all-gathered in place over the
 * CP communicator, and every CP rank runs the same per-rollout partition / Eq. 2 / Eq. 3 /
 * surrogate (the entropy split needs all of a rollout's entropies), so each rank holds the
 * coefficients of its own rows and the same loss. Combine with DP through espo_create's
 * communicator (the DP group spans different data; the CP ranks of one group hold the same
 * rollouts). Not with single-pass mode.
 * espo_attach_cp: right after espo_create; cp_unique_id = NCCL id of the CP group, or NULL for
 *   same-device emulation, where espo_cp_gather_local must run (after every rank's forward)
 *   in place of the all-gather: it copies the other ranks' blocks from their contexts. */
espo_status espo_attach_cp(espo_ctx_t ctx, const void* cp_unique_id, int32_t cp_rank,
                           int32_t cp_world);
espo_status espo_cp_gather_local(espo_ctx_t ctx, const espo_ctx_t* ranks, int32_t cp_world,
                                 espo_stream_t stream);

/* ---- caller-supplied selection entropies (reading Q4's alternative) ----
 * By default the entropies that pick each rollout's entropy buckets and set
 * Eq. 3's ε_τ are the sweep's own, of the π_θ logits given to the forward
 * (reading Q4). SPEC.md:460 takes the rollout policy's entropies instead; a trainer that has
 * them (from the inference engine) passes them here: after espo_prepare and before finalize,
 * entropy f32 [n_rows] (device, nats, finite and ≥ 0; −0 is taken as +0) for rows
 * [row_begin, row_begin + n_rows), in chunks of any order that do not overlap (else
 * ESPO_ERR_BAD_STATE). Once called in a step, every row of [0, T) must be covered before
 * finalize (else ESPO_ERR_BAD_STATE). K3 then uses these values wherever the method uses e_t —
 * the partition, ε_τ, RL-ZVP's token advantages and stats.mean_entropy — while
 * lse / lp / q and the exported per-token H stay the sweep's; dlogits keep their form (the
 * entropies are detached). The values are copied (the caller keeps ownership; a T-float
 * buffer is allocated on first use). A negative value → sticky ESPO_ERR_INVALID_ARGUMENT,
 * NaN / ±inf → sticky ESPO_ERR_NONFINITE_INPUT (espo_get_error; the loss is then NaN). Not
 * with single-pass mode or context parallelism (ESPO_ERR_UNSUPPORTED). */
espo_status espo_set_entropies(espo_ctx_t ctx, const float* entropy, int64_t row_begin,
                               int64_t n_rows, espo_stream_t stream);

/* ---- single-pass mode: forward and backward of a chunk in one call ----
 * The loss normaliser D (N active rollouts; T_active in TOKEN mode) depends only on the
 * zero-variance filter and the mask (readings Q10, Q11), and every other
 * coupling (partition, s_τ, ε_τ) is within a rollout. So once D is fixed from the mask, a
 * chunk holding COMPLETE rollouts can run forward → per-rollout K3 → backward at once, and a
 * trainer produces each logits chunk once (no second pass over the logits or recompute of the
 * LM head for the backward).
 *
 * espo_set_mask: after espo_prepare and before any forward call. mask u8[T] (device; NULL =
 * all ones) is copied into the context; D is counted (and all-reduced over the DP
 * communicator when world > 1 — a collective: every rank calls it). Switches the context to
 * single-pass mode until the next espo_prepare: espo_loss_fwd / espo_loss_bwd then return
 * ESPO_ERR_BAD_STATE.
 * espo_loss_fwd_bwd: rows [row_begin, row_begin + n_rows) must start and end on rollout
 * boundaries (device-checked: ESPO_ERR_INVALID_ARGUMENT via espo_get_error and a NaN loss);
 * logits/tokens/old_logp as espo_loss_fwd, dlogits/grad_loss_dev as espo_loss_bwd (in place
 * allowed). Chunks in any order, each row once; espo_loss_finalize afterwards only reduces
 * the loss and statistics. Results are identical to the two-sweep path. */
espo_status espo_set_mask(espo_ctx_t ctx, const uint8_t* mask, espo_stream_t stream);
espo_status espo_loss_fwd_bwd(espo_ctx_t ctx, const void* logits, int64_t ld,
                              const int32_t* tokens, const float* old_logp, void* dlogits,
                              int64_t ldg, const float* grad_loss_dev, int64_t row_begin,
                              int64_t n_rows, espo_stream_t stream);

/* ---- factored gradient (one sweep per row: statistics + the row-local gradient factor) ----
 * The gradient of the loss w.r.t. logits row t factors as
 *   d loss/d z_t = scale_t · G_t,  G_t = onehot(y_t) − softmax(λ z_t),  scale_t = λ·g_t
 * (only the Eq. 1 numerator log π_θ(y_t) carries gradient; g_t = −grad·c_t/D
 * from Eqs. 1-3). G_t needs only the row, scale_t the rollout-level
 * reduction, so a consumer that applies scale_t in its own GEMM (dh = diag(scale)·G·W,
 * dW = Gᵀ·(diag(scale)·h)) reads each logits row once: 2V read + one G row written.
 * espo_loss_fwd_factored: espo_loss_fwd for rows [row_begin, row_begin + n_rows) (same
 * arguments, checks, coverage and errors) that also writes G_t into grad (device,
 * [n_rows, ldg ≥ vocab] of grad_dtype, 16-byte aligned; may alias logits when ldg == ld and
 * the dtypes are equal — the rows' logits are then overwritten). The target entry is
 * q_t = 1 − p_y (no cancellation); rows without gradient (masked, eliminated group, inactive
 * rollout) are zero-filled without being read when zero_fill_inactive_rows, else untouched;
 * clipped rows get their G_t (their scale is 0). In compact mode the untouched rows keep
 * whatever grad held (the Python binding zero-initialises a grad it allocates): a consumer
 * forming diag(scale)·G must either start from a zeroed grad or skip rows whose scale is 0
 * (0·NaN = NaN would otherwise poison dh/dW). Unsharded contexts, not in single-pass mode
 * (ESPO_ERR_BAD_STATE). Statistics agree with espo_loss_fwd's within fp32 rounding (a
 * different summation order), not bitwise.
 * espo_loss_row_scale (after espo_loss_finalize): scale_out[r] = scale_t for rows
 * [row_begin, row_begin + n_rows) (device f32 [n_rows]), 0 for rows without gradient;
 * grad_loss_dev as in espo_loss_bwd. scale_t·G_t equals espo_loss_bwd's row up to the bf16
 * rounding of G_t instead of the product. */
espo_status espo_loss_fwd_factored(espo_ctx_t ctx, const void* logits, int64_t ld,
                                   const int32_t* tokens, const float* old_logp,
                                   const uint8_t* mask, void* grad, int64_t ldg, int64_t row_begin,
                                   int64_t n_rows, espo_stream_t stream);
espo_status espo_loss_row_scale(espo_ctx_t ctx, const float* grad_loss_dev, float* scale_out,
                                int64_t row_begin, int64_t n_rows, espo_stream_t stream);

/* ---- fused LM head + forward statistics (tcgen05) ----
 * Computes the same row statistics as espo_loss_fwd for logits z = hidden · weightᵀ (softmax
 * of λ·z as there) without writing the logits: hidden bf16 [n_rows, ldh ≥ d] (row row_begin of the chunk first),
 * weight bf16 [vocab, ldw ≥ d] (the LM-head matrix, row v = vocabulary entry v), fp32
 * accumulation on the tensor cores; tokens/old_logp/mask as in espo_loss_fwd. 16-byte aligned
 * bases and pitches. Counts as the forward call for these rows. The first call may allocate
 * a small per-row partial buffer (16 B × rows × vocabulary parts) and the GEMM's lockstep
 * counters (4 B per wave of tiles); like espo_lmhead_bwd's scratch they only grow, so a step
 * can be captured into a CUDA graph after one eager step of the same size (no call
 * synchronises with the host; tests/test_gpu_graph.py). Unsharded contexts only. */
espo_status espo_lmhead_fwd(espo_ctx_t ctx, const void* hidden, int64_t ldh, const void* weight,
                            int64_t ldw, int32_t d, const int32_t* tokens, const float* old_logp,
                            const uint8_t* mask, int64_t row_begin, int64_t n_rows,
                            espo_stream_t stream);

/* ---- fused LM head backward (tcgen05 recompute + bf16 dz tile + two tcgen05 GEMMs) ----
 * Gradients of grad_loss·loss through logits z = hidden·weightᵀ for the
 * rows [row_begin, row_begin + n_rows) of a finalized context whose forward ran through
 * espo_lmhead_fwd with the same hidden/weight:
 *   dz    = ∂(grad_loss·loss)/∂z, exactly K5's formula, recomputed tile by tile on the tensor
 *           cores (same pipeline and K order as the forward, so the logits are bitwise the
 *           forward's) and rounded to bf16 into a context-owned scratch of
 *           ESPO_OPT_LMHEAD_BWD_ROWS × round_up(vocab, 256) bf16 (allocated on first use);
 *           rows whose coefficient is 0 (clipped, masked, eliminated: dz_t = 0) are left out —
 *           the rows with gradient are gathered (stable order) and only they are recomputed
 *           and contracted (ESPO_OPT_LMHEAD_COMPACT; scratch 4 B/row + the gathered rows);
 *   dhidden[r, :] = Σ_v dz[r, v]·weight[v, :]          (overwritten; f32 or bf16 per dh_dtype)
 *   dweight[v, :] += Σ_r dz[r, v]·hidden[r, :]          (f32, ACCUMULATED: zero it once)
 * The two contractions are bf16 × bf16 → fp32 GEMMs on the library's own tcgen05 kernel
 * (k_gemm.cuh: TMA-fed, TMEM accumulators; dz is read K-major for dh and MN-major for dW, W
 * and hidden MN-major, so no operand is transposed or copied), on `stream`. Either output may
 * be NULL (skipped). Shapes and alignment as espo_lmhead_fwd; dhidden pitch lddh ≥ d, dweight
 * pitch lddw ≥ d (16-byte aligned). grad_loss_dev as espo_loss_bwd. Errors:
 * ESPO_ERR_BAD_STATE before finalize, ESPO_ERR_UNSUPPORTED on a vocabulary-sharded context,
 * ESPO_ERR_BLAS only with ESPO_OPT_LMHEAD_BWD_GEMM = 1 (cuBLAS A/B path) if cuBLAS fails. */
espo_status espo_lmhead_bwd(espo_ctx_t ctx, const void* hidden, int64_t ldh, const void* weight,
                            int64_t ldw, int32_t d, void* dhidden, int64_t lddh, int32_t dh_dtype,
                            float* dweight, int64_t lddw, const float* grad_loss_dev,
                            int64_t row_begin, int64_t n_rows, espo_stream_t stream);

/* Synchronises `stream`, then returns the sticky device error (ESPO_OK if none) or
 * ESPO_ERR_CUDA if a CUDA error is pending. */
espo_status espo_get_error(espo_ctx_t ctx, espo_stream_t stream);

const char* espo_status_string(espo_status s);

/* ---- introspection (tests / tooling; not needed on the training path) ---- */

/* Copies per-token workspace values of rows [row_begin, row_begin+n_rows) to device
 * arrays (each nullable): lse/lp/H/q f32 (after fwd), coef f32 = ∂J_i/∂lp_t before the
 * global 1/D (after finalize), bucket u8 (stats bucket), clip u8 (1 = gradient clipped),
 * valid u8 (1 = row was read: active rollout and mask = 1). */
espo_status espo_export_token_stats(espo_ctx_t ctx, int64_t row_begin, int64_t n_rows,
                                    float* lse, float* lp, float* H, float* q, float* coef,
                                    uint8_t* bucket, uint8_t* clip, uint8_t* valid,
                                    espo_stream_t stream);

/* Copies per-rollout results to device arrays (each nullable): adv f64, zv u8, active u8,
 * J_i f64 (Σ_t w_t ℓ_t), nb i32 (non-empty buckets), theta f32[R·(K−1)] thresholds. */
espo_status espo_export_rollout_stats(espo_ctx_t ctx, double* adv, uint8_t* zv,
                                      uint8_t* active, double* J_i, int32_t* nb,
                                      float* theta, espo_stream_t stream);

/* Number of kernels this context has launched so far. */
uint64_t espo_launch_count(espo_ctx_t ctx);

/* Ranks in the data-parallel communicator of espo_create (ncclCommCount): 1 for world == 1,
 * −1 on error. */
int32_t espo_comm_size(espo_ctx_t ctx);

/* Kernel-variant switches for A/B measurement. */
typedef enum {
  ESPO_OPT_FWD_IMPL = 0,       /* 0 = TMA bulk-copy smem ring (default), 1 = LDG.128 warp per
                                  row, 2..7 = other ring geometries, 8 = default geometry in
                                  scalar FP32, 9..11 = (row, tile) grid (K2) */
  ESPO_OPT_BWD_IMPL = 1,       /* 0 = tiled (row, 32 KB tile) grid (default), 1 = LDG.128 warp
                                  per row, 2..6 = TMA ring geometries, 7 = 16 KB tiles,
                                  8 = tiles with scalar FP32, 9 = tiles over the compact row
                                  lists (4 rows per block) */
  ESPO_OPT_BLOCKS_PER_SM = 2,  /* persistent grid = blocks_per_sm × SM count (0 = auto) */
  ESPO_OPT_LMHEAD_PARTS = 3,   /* espo_lmhead_fwd/bwd vocabulary parts per row block (0 = auto) */
  ESPO_OPT_LMHEAD_BWD_ROWS = 4,/* espo_lmhead_bwd rows per dz sub-chunk (multiple of 128;
                                  0 = default 8192) */
  ESPO_OPT_LMHEAD_2CTA = 5,    /* 1: LM-head kernels on CTA pairs (tcgen05 cta_group::2,
                                  M = 256 per pair); 0: one CTA per 128-row block */
  ESPO_OPT_FACTORED_IMPL = 6,  /* espo_loss_fwd_factored: 0 = TMA ring (1 producer + 20 consumer
                                  warps, 5 × 40 KB slots, default), 1 = 1024-thread CTA per row
                                  with plain loads, 2 = 16 warps × 6 × 32 KB, 3 = default + TMEM
                                  stash of pass-1 exponentials, 4-5 = two CTAs per SM,
                                  6 = rolling pass-2/pass-1 interleave (A/B) */
  ESPO_OPT_PEER_TIMEOUT_MS = 7,/* bound on every peer-memory wait of the TP exchange, in ms of
                                  device wall time (default 120000); a timeout sets the sticky
                                  ESPO_ERR_PEER_TIMEOUT and invalidates the step (the chunk's
                                  row statistics are not written) */
  ESPO_OPT_LMHEAD_BWD_GEMM = 8,/* espo_lmhead_bwd's dh / dW contractions on the library's
                                  tcgen05 GEMM: 0 = CTA pairs, 256 × 512 tiles for dh (long K) and
                                  256 × 256 for dW (default); 2 = one CTA per 128 × 256 tile;
                                  3 = pairs 256 × 256 for both; 4 = pairs 256 × 512 for both;
                                  5 = 4-CTA clusters (two pairs sharing A by TMA multicast,
                                  256 × 512 each) for both; 6 = those for dh, default dW;
                                  7 = default dh, 256 × 256 dW in N-groups of 8 at any d;
                                  1 = cuBLAS (A/B measurement only) */
  ESPO_OPT_GEMM_GROUP_M = 9,   /* backward GEMM tile order: bits 0-15 = dh M-blocks per raster
                                  group (0 = auto: 8, 16 above d = 4096); bits 16-31 = dW N-blocks per group (0 = all
                                  of d, N fastest) */
  ESPO_OPT_GEMM_HINTS = 10,    /* L2 policies of the backward GEMMs for A/B measurement: bits 0-7
                                  dh, 8-15 dW, each A | B << 2 | C << 4 with 0 = normal,
                                  1 = evict_first, 2 = evict_last; −1 = defaults */
  ESPO_OPT_LMHEAD_COMPACT = 11, /* espo_lmhead_bwd: 1 (default) = recompute and contract only the
                                  rows with gradient (c_t ≠ 0; needs d % 8 == 0), 0 = all rows */
  ESPO_OPT_GEMM_SYNC = 12,     /* soft lockstep of the backward's dh / dW CTA-pair GEMMs:
                                  bits 0-15 = chunk of K-steps (0 = off), bits 16-31 = slack in
                                  chunks (0 = 2); bits 32-47 / 48-63 = the same for the dW GEMM
                                  alone (0 = as above). Not set (or −1): on (16 K-steps, slack 2)
                                  for d > 4096, off below. The LM-head forward / dz GEMMs have their
                                  own (ESPO_OPT_LMHEAD_RASTER bit 27) */
  ESPO_OPT_LMHEAD_IMPL = 13,   /* fused LM-head forward and backward recompute: 0 (default) = on
                                  the tcgen05 GEMM core (CTA-pair 256 × 512 tiles in a grouped
                                  raster, per-tile partials merged like vocabulary shards);
                                  1 = the dedicated kernels (part × row-block grid; ESPO_OPT_LMHEAD_2CTA
                                  / _PARTS apply) */
  ESPO_OPT_LMHEAD_RASTER = 14  /* impl 0: bits 0-15 = M-tiles per raster group (0 = auto: 16),
                                  bits 16-23 = L2 policies (A | B << 2, 1 evict_first, 2
                                  evict_last), bit 24 = 256 × 256 tiles (double-buffered) instead
                                  of 256 × 512, bit 25 = 4-CTA clusters (two pairs sharing A by
                                  TMA multicast), bit 26 = no split-K for the backward's dh GEMM
                                  (default: split in two when it has fewer than 6 waves of
                                  tiles), bit 27 = no soft lockstep of the forward / dz GEMM
                                  (default on: a cluster more than 2 chunks of 8 K-steps ahead
                                  of the slowest cluster of its wave waits, so the wave's
                                  operand panels are read from DRAM once), bit 28 =
                                  every 256 × 512 CTA-pair GEMM (also dh / dW) releases its
                                  accumulator whole instead of in halves (default: the next
                                  tile's first K-steps on columns 0-255 overlap the epilogue's
                                  read of 256-511), bit 29 = static round-robin tile order for
                                  every CTA-pair GEMM (default: a dynamic scheduler — each pair
                                  takes the next tile from an atomic counter, so the tiles in
                                  flight stay a contiguous window of the raster; the backward's
                                  dz recompute then runs without the lockstep), bit 30 = the dW
                                  GEMM's epilogue reads, adds and writes dW on the SMs (default:
                                  it stages 32 × 32 fp32 blocks in shared memory and adds them
                                  into dW with a TMA reduce, cp.reduce.async.bulk.tensor .add) */
} espo_option;
espo_status espo_set_option(espo_ctx_t ctx, int32_t option, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* ESPO_H_ */
