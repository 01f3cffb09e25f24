// k_seq.cuh — K1 (prepare: groups, zero-variance filter, GRPO advantages), K3 (per-sequence
// entropy partition, Eq. 2 ratio, Eq. 3 clip, surrogate and coefficients) and K4
// (deterministic reduction + loss). SURVEY §8(a) a1, a2, a4–a7.
#pragma once
#include "common.cuh"
#include "workspace.cuh"

namespace espo {

struct PrepParams {
  const float* rewards;
  const int32_t* group_ids;
  const int64_t* seq_offsets;
  int R;
  int64_t T;
  int std_unbiased;
  double adv_eps, zv_var_eps;
  int zv_mode;
  float zvp_threshold;
  float* adv_out;   // nullable
  uint8_t* zv_out;  // nullable
  Workspace ws;
};

// K1a — one thread per rollout; the first rollout of each group (a maximal run of equal
// group ids) walks its group sequentially in index order with one IEEE rounding per
// operation (no FMA contraction), so μ, σ and Â are bit-identical to the fp64 oracle.
// PAPER.md:77 (ZV: identical rewards → zero advantage), PAPER.md:105-107 (Â).
__global__ void k_prepare_groups(const PrepParams p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > p.R) return;
  // seq_offsets copy + checks (R+1 entries)
  const int64_t so = p.seq_offsets[i];
  p.ws.seq_off[i] = so;
  if ((i == 0 && so != 0) || (i == p.R && so != p.T) || (i > 0 && so < p.seq_offsets[i - 1]))
    set_error(p.ws.err, ESPO_ERR_INVALID_ARGUMENT);
  if (i == p.R) return;
  const float ri = p.rewards[i];
  if (!isfinite(ri)) set_error(p.ws.err, ESPO_ERR_NONFINITE_INPUT);
  const int gi = p.group_ids[i];
  if (i > 0 && gi < p.group_ids[i - 1]) set_error(p.ws.err, ESPO_ERR_GROUPS_NOT_CONTIGUOUS);
  const bool head = (i == 0) || (p.group_ids[i - 1] != gi);
  if (!head) return;
  int e = i + 1;
  while (e < p.R && p.group_ids[e] == gi) ++e;
  const int n = e - i;
  double mu = 0.0;
  for (int j = i; j < e; ++j) mu = __dadd_rn(mu, static_cast<double>(p.rewards[j]));
  mu = __ddiv_rn(mu, static_cast<double>(n));
  double ss = 0.0;
  bool all_eq = true;
  for (int j = i; j < e; ++j) {
    const double rj = static_cast<double>(p.rewards[j]);
    const double d = __dsub_rn(rj, mu);
    ss = __dadd_rn(ss, __dmul_rn(d, d));
    all_eq = all_eq && (p.rewards[j] == ri);
  }
  const int denom = p.std_unbiased ? n - 1 : n;
  const double var = denom > 0 ? __ddiv_rn(ss, static_cast<double>(denom)) : 0.0;
  const double sigma = __dsqrt_rn(var);
  bool zv;
  if (n < 2) zv = true;
  else if (p.zv_var_eps > 0.0) zv = var <= p.zv_var_eps;
  else zv = all_eq;
  const double den = __dadd_rn(sigma, p.adv_eps);
  const bool zvp = zv && p.zv_mode == ESPO_ZV_RLZVP;
  for (int j = i; j < e; ++j) {
    const double a = zv ? 0.0 : __ddiv_rn(__dsub_rn(static_cast<double>(p.rewards[j]), mu), den);
    p.ws.adv[j] = a;
    p.ws.cand[j] = (zv && !zvp) ? 0 : 1;
    p.ws.zsign[j] = zvp ? (p.rewards[j] < p.zvp_threshold ? 1 : -1) : 0;
    p.ws.ghead[j] = (j == i) ? (zv ? 2 : 1) : 0;
    if (p.adv_out) p.adv_out[j] = static_cast<float>(a);
    if (p.zv_out) p.zv_out[j] = zv ? 1 : 0;
  }
}

// K1b — rollout id of every row (block per rollout).
__global__ void k_row_seq(const Workspace ws, int R) {
  const int i = blockIdx.x;
  const int64_t b = ws.seq_off[i], e = ws.seq_off[i + 1];
  for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) ws.row_seq[t] = i;
}

// ------------------------------------------------------------------------------ K3
struct SeqParams {
  int R;
  int64_t row_lo, row_hi;  // rollouts inside [row_lo, row_hi] only (single-pass chunk)
  int V;
  float alpha, eps_min;
  int K;
  int split_num, split_den;
  int partition, ratio_mode, norm;
  double log_ratio_clamp;
  double inv_logV;
  double zvp_beta;
  Workspace ws;
};

constexpr int kSeqThreads = 512;

// Deterministic block sum (fixed shuffle tree + fixed smem order).
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  T r = 0;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kSeqThreads / 32; ++k) r += sh[k];
    sh[32] = r;
  }
  __syncthreads();
  r = sh[32];
  return r;
}

// rank-th smallest (1-based) H bit pattern among valid rows of [b, e): 4-pass MSB radix
// select over the fp32 bits (H ≥ +0, so the unsigned order is the float order).
__device__ uint32_t radix_select(const float* H, const uint8_t* flag, int64_t b, int64_t e,
                                 int rank, unsigned* hist, int* sel) {
  uint32_t prefix = 0, pmask = 0;
  int k = rank;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) {
      if (flag[t]) {
        const uint32_t key = __float_as_uint(H[t]);
        if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      unsigned c[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { c[j] = hist[lane * 8 + j]; s += c[j]; }
      unsigned incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
      }
      const unsigned excl = incl - s;
      if (excl < static_cast<unsigned>(k) && static_cast<unsigned>(k) <= incl) {
        unsigned cum = excl;
        for (int j = 0; j < 8; ++j) {
          if (cum + c[j] >= static_cast<unsigned>(k)) {
            sel[0] = lane * 8 + j;
            sel[1] = k - static_cast<int>(cum);
            break;
          }
          cum += c[j];
        }
      }
    }
    __syncthreads();
    prefix |= static_cast<uint32_t>(sel[0]) << shift;
    pmask |= 255u << shift;
    k = sel[1];
    __syncthreads();
  }
  return prefix;
}

// K3 — one CTA per rollout. Partition (reading Q3), per-bucket Eq. 2
// ratio s_τ and Eq. 3 clip ε_τ in fp64, then per token the surrogate ℓ_t,
// clip decision κ_t (Q12) and c_t = Â·v_t·κ_t·w_t; J_i = Σ_t w_t ℓ_t.
__global__ void __launch_bounds__(kSeqThreads) k_seq_reduce(const SeqParams p) {
  __shared__ unsigned hist[256];
  __shared__ int sel[2];
  __shared__ double shd[33];
  __shared__ long long shl[33];
  __shared__ double s_s[kMaxK], s_eps[kMaxK], s_w[kMaxK];
  __shared__ float s_theta[kMaxK];
  const int i = blockIdx.x;
  const Workspace& ws = p.ws;
  const int64_t b = ws.seq_off[i], e = ws.seq_off[i + 1];
  if (b < p.row_lo || e > p.row_hi) return;   // another chunk's rollout (single-pass)
  double* red = ws.red_r;  // SoA [kRedLen][R]
  auto put = [&](int k, double v) { if (threadIdx.x == 0) red[int64_t(k) * p.R + i] = v; };

  // n_i = valid rows
  long long cnt = 0;
  for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) cnt += ws.flag[t];
  const long long n = block_sum<long long>(cnt, shl);
  const bool act = ws.cand[i] && n > 0;
  if (!act) {
    if (threadIdx.x == 0) {
      ws.active[i] = 0; ws.nb[i] = 0; ws.J[i] = 0.0;
    }
    for (int k = 0; k < kRedLen; ++k) put(k, 0.0);
    if (threadIdx.x == 0) {
      red[3ll * p.R + i] = ws.ghead[i] == 2 ? 1.0 : 0.0;
      red[4ll * p.R + i] = ws.ghead[i] ? 1.0 : 0.0;
    }
    return;
  }
  const double A = ws.adv[i];
  const int zs = ws.zsign[i];
  // RL-ZVP: ē_i (fp64, fixed order) for Â_t = β·s·(e_t − ē_i)/log|V|
  double hbar = 0.0;
  if (zs != 0) {
    double hl = 0.0;
    for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x)
      if (ws.flag[t]) hl += static_cast<double>(ws.H[t]);
    hbar = block_sum<double>(hl, shd) / static_cast<double>(n);
  }
  const double zscale = p.zvp_beta * static_cast<double>(zs) * p.inv_logV;
  const bool quant = (p.partition == ESPO_PART_QUANTILE) && p.K > 1;
  const bool single = (p.partition == ESPO_PART_SINGLETON);
  const int K = quant ? p.K : 1;

  // ---- O3: thresholds (order statistics of H among valid rows)
  if (quant) {
    for (int k = 1; k < K; ++k) {
      long long rk = (K == 2) ? (static_cast<long long>(p.split_num) * n) / p.split_den
                              : (static_cast<long long>(k) * n) / K;
      if (rk < 1) rk = 1;
      const uint32_t bits = radix_select(ws.H, ws.flag, b, e, static_cast<int>(rk), hist, sel);
      if (threadIdx.x == 0) s_theta[k - 1] = __uint_as_float(bits);
    }
    __syncthreads();
  }
  auto bucket_of = [&](float h) {
    int bk = 0;
    for (int k = 1; k < K; ++k) bk += (h > s_theta[k - 1]) ? 1 : 0;
    return bk;
  };

  // ---- O4: per-bucket sums (fp64, fixed order)
  if (!single) {
    long long c[kMaxK] = {0, 0, 0, 0};
    double dl[kMaxK] = {0, 0, 0, 0}, hs[kMaxK] = {0, 0, 0, 0};
    for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) {
      if (!ws.flag[t]) continue;
      const float h = ws.H[t];
      const int bk = bucket_of(h);
#pragma unroll
      for (int k = 0; k < kMaxK; ++k) {
        if (k == bk) {
          c[k] += 1;
          dl[k] += static_cast<double>(ws.lp[t]) - static_cast<double>(ws.old[t]);
          hs[k] += static_cast<double>(h);
        }
      }
    }
    int nb = 0;
    for (int k = 0; k < K; ++k) {
      const long long ck = block_sum<long long>(c[k], shl);
      const double dk = block_sum<double>(dl[k], shd);
      const double hk = block_sum<double>(hs[k], shd);
      if (threadIdx.x == 0) {
        if (ck > 0) {
          ++nb;
          double m = dk / static_cast<double>(ck);
          if (p.log_ratio_clamp > 0) m = fmin(fmax(m, -p.log_ratio_clamp), p.log_ratio_clamp);
          s_s[k] = exp(m);
          s_eps[k] = fmax(static_cast<double>(p.eps_min),
                          static_cast<double>(p.alpha) * hk / (static_cast<double>(ck)) * p.inv_logV);
          s_w[k] = static_cast<double>(ck);
        } else {
          s_s[k] = 0; s_eps[k] = 0; s_w[k] = 0;
        }
      }
    }
    if (threadIdx.x == 0) {
      for (int k = 0; k < K; ++k)
        s_w[k] = (s_w[k] > 0) ? (p.norm == ESPO_NORM_SEQ ? 1.0 / (nb * s_w[k]) : 1.0) : 0.0;
      ws.nb[i] = nb;
      for (int k = 1; k < K; ++k) ws.theta[int64_t(i) * (kMaxK - 1) + k - 1] = s_theta[k - 1];
    }
    __syncthreads();
  } else if (threadIdx.x == 0) {
    ws.nb[i] = static_cast<int>(n);
  }

  // ---- O5: per-token surrogate, clip decision, coefficient
  const double w_single = (p.norm == ESPO_NORM_SEQ) ? 1.0 / static_cast<double>(n) : 1.0;
  double Jl = 0.0, abslr = 0.0, hsum = 0.0, sqlr = 0.0, k3 = 0.0;
  double st_tok[kMaxK] = {0, 0, 0, 0}, st_clip[kMaxK] = {0, 0, 0, 0};
  double st_v[kMaxK] = {0, 0, 0, 0}, st_e[kMaxK] = {0, 0, 0, 0};
  for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) {
    if (!ws.flag[t]) continue;
    const double lp = ws.lp[t], old = ws.old[t];
    const float hf = ws.H[t];
    const double h = hf;
    int bk;
    double s, eps, w;
    if (single) {
      double m = lp - old;
      if (p.log_ratio_clamp > 0) m = fmin(fmax(m, -p.log_ratio_clamp), p.log_ratio_clamp);
      s = exp(m);
      eps = fmax(static_cast<double>(p.eps_min), static_cast<double>(p.alpha) * h * p.inv_logV);
      w = w_single;
      bk = 0;
    } else {
      bk = bucket_of(hf);
      s = s_s[bk]; eps = s_eps[bk]; w = s_w[bk];
    }
    const double v = (p.ratio_mode == ESPO_RATIO_GSPO_TOKEN) ? s : s * exp(lp - old);
    const double At = zs ? zscale * (h - hbar) : A;
    const double lo = 1.0 - eps, hi = 1.0 + eps;
    const double vc = fmin(fmax(v, lo), hi);
    const double ell = fmin(v * At, vc * At);
    const bool clipped = (At > 0 && v > hi) || (At < 0 && v < lo);
    Jl += w * ell;
    ws.coef[t] = clipped ? 0.f : static_cast<float>(At * v * w);
    const int sb = quant ? bk : 0;
    ws.bucket[t] = static_cast<uint8_t>(sb);
    ws.clip[t] = clipped ? 1 : 0;
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) {
      if (k == sb) {
        st_tok[k] += 1.0; st_clip[k] += clipped ? 1.0 : 0.0; st_v[k] += v; st_e[k] += eps;
      }
    }
    const double dlr = lp - old;
    abslr += fabs(dlr);
    sqlr += dlr * dlr;
    k3 += expm1(dlr) - dlr;   // KL(π_old ‖ π_θ) k3 estimator (train/inference mismatch)
    hsum += h;
  }
  const double J = block_sum<double>(Jl, shd);
  const double al = block_sum<double>(abslr, shd);
  const double hs = block_sum<double>(hsum, shd);
  const double sq = block_sum<double>(sqlr, shd);
  const double kk = block_sum<double>(k3, shd);
  double ncl = 0;
  for (int k = 0; k < kMaxK; ++k) {
    const double a = block_sum<double>(st_tok[k], shd);
    const double c = block_sum<double>(st_clip[k], shd);
    const double v = block_sum<double>(st_v[k], shd);
    const double ee = block_sum<double>(st_e[k], shd);
    put(8 + k, a); put(12 + k, c); put(16 + k, v); put(20 + k, ee);
    ncl += c;
  }
  if (threadIdx.x == 0) {
    ws.active[i] = 1;
    ws.J[i] = J;
  }
  put(0, J);
  put(1, 1.0);
  put(2, static_cast<double>(n));
  put(3, ws.ghead[i] == 2 ? 1.0 : 0.0);
  put(4, ws.ghead[i] ? 1.0 : 0.0);
  put(5, ncl);
  put(6, al);
  put(7, hs);
  put(24, sq);
  put(25, kk);
}

// ------------------------------------------------------------------ K0 (single-pass mode)
// The normaliser D of the loss (N active rollouts, or T_active tokens in TOKEN mode) depends
// only on the zero-variance filter and the mask (Q10, Q11), never on logits, so
// it can be fixed before the forward: then every chunk of complete rollouts can run
// forward → K3 → backward at once (espo_loss_fwd_bwd).
// K0a — one block per rollout: copies its mask rows, counts them, marks it active (writes
// the same red_r[1], red_r[2] terms K3 will write).
__global__ void __launch_bounds__(256) k_mask_counts(const uint8_t* mask, const Workspace ws, int R) {
  __shared__ long long sh[33];
  const int i = blockIdx.x;
  const int64_t b = ws.seq_off[i], e = ws.seq_off[i + 1];
  long long cnt = 0;
  for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) {
    const uint8_t m = mask ? (mask[t] != 0) : 1;
    ws.pmask[t] = m;
    cnt += m;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) sh[w] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long n = 0;
    for (int k = 0; k < int(blockDim.x >> 5); ++k) n += sh[k];
    const bool act = ws.cand[i] && n > 0;
    ws.red_r[1ll * R + i] = act ? 1.0 : 0.0;
    ws.red_r[2ll * R + i] = act ? static_cast<double>(n) : 0.0;
  }
}

// K0b — {N, T_active} in rollout order (deterministic).
__global__ void __launch_bounds__(256) k_mask_reduce(const Workspace ws, int R) {
  __shared__ double sh[2][256];
  double a = 0.0, n = 0.0;
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    a += ws.red_r[1ll * R + i];
    n += ws.red_r[2ll * R + i];
  }
  sh[0][threadIdx.x] = a;
  sh[1][threadIdx.x] = n;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + s];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ws.dpre[0] = sh[0][0];
    ws.dpre[1] = sh[1][0];
  }
}

// K0c — backward scale λ/D from the (all-reduced) counts; same expression as K4b.
__global__ void k_mask_scale(const Workspace ws, int norm, float logit_scale) {
  const double D = (norm == ESPO_NORM_SEQ) ? ws.dpre[0] : ws.dpre[1];
  *ws.bwd_scale = D > 0 ? static_cast<float>(static_cast<double>(logit_scale) / D) : 0.f;
}

// Single-pass chunk check: both ends of [lo, hi) must be rollout boundaries.
__global__ void k_check_chunk(const Workspace ws, int64_t lo, int64_t hi, int64_t T) {
  auto boundary = [&](int64_t r) { return r == T || ws.seq_off[ws.row_seq[r]] == r; };
  if (!boundary(lo) || !boundary(hi)) set_error(ws.err, ESPO_ERR_INVALID_ARGUMENT);
}

// K4 — rank-local deterministic reduction of the per-rollout terms (fixed order).
__global__ void __launch_bounds__(256) k_reduce_rollouts(const Workspace ws, int R) {
  __shared__ double sh[256];
  const int k = blockIdx.x;  // one block per reduced value
  double acc = 0.0;
  for (int i = threadIdx.x; i < R; i += blockDim.x) acc += ws.red_r[int64_t(k) * R + i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) ws.red[k] = sh[0];
}

// K4b — loss = −ΣJ_i/D (Q10, Q13), bwd scale λ/D, stats.
__global__ void k_finalize_scalar(const Workspace ws, int norm, float logit_scale, float* loss_out,
                                  espo_stats* stats) {
  const double* r = ws.red;
  const double D = (norm == ESPO_NORM_SEQ) ? r[1] : r[2];
  const bool bad = *ws.err != 0;
  double loss = D > 0 ? -r[0] / D : 0.0;
  if (bad) loss = __longlong_as_double(0x7ff8000000000000ll);
  *ws.bwd_scale = D > 0 ? static_cast<float>(static_cast<double>(logit_scale) / D) : 0.f;
  if (loss_out) *loss_out = static_cast<float>(loss);
  if (stats) {
    stats->loss = loss;
    stats->n_active_rollouts = r[1];
    stats->n_active_tokens = r[2];
    stats->n_zv_groups = r[3];
    stats->n_groups = r[4];
    stats->n_clipped_tokens = r[5];
    stats->mean_abs_logratio = r[2] > 0 ? r[6] / r[2] : 0.0;
    stats->mean_entropy = r[2] > 0 ? r[7] / r[2] : 0.0;
    for (int k = 0; k < kMaxK; ++k) {
      const double tk = r[8 + k];
      stats->clip_frac[k] = tk > 0 ? r[12 + k] / tk : 0.0;
      stats->mean_ratio[k] = tk > 0 ? r[16 + k] / tk : 0.0;
      stats->mean_eps[k] = tk > 0 ? r[20 + k] / tk : 0.0;
      stats->tokens_per_bucket[k] = tk;
    }
    stats->mean_sq_logratio = r[2] > 0 ? r[24] / r[2] : 0.0;
    stats->mean_k3 = r[2] > 0 ? r[25] / r[2] : 0.0;
  }
}

// Copies for the introspection API.
// espo_set_entropies: caller-supplied selection entropies into the context's copy (reading Q4's
// alternative). −0 becomes +0 (K3's radix select orders the fp32 bits of e ≥ 0);
// a negative value or NaN / ±inf sets the sticky error.
__global__ void k_set_entropies(const float* src, float* dst, int64_t n, int* err) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float x = src[i];
    if (!(fabsf(x) <= 3.4e38f)) set_error(err, ESPO_ERR_NONFINITE_INPUT);
    else if (x < 0.f) set_error(err, ESPO_ERR_INVALID_ARGUMENT);
    dst[i] = x + 0.f;
  }
}

__global__ void k_export_tokens(const Workspace ws, int64_t b, int64_t n, float* lse, float* lp,
                                float* H, float* q, float* coef, uint8_t* bucket, uint8_t* clip,
                                uint8_t* valid) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = b + k;
    const bool f = ws.flag[t] != 0;
    const float nan = __int_as_float(0x7fc00000);
    if (lse) lse[k] = f ? ws.lse[t] : nan;
    if (lp) lp[k] = f ? ws.lp[t] : nan;
    if (H) H[k] = f ? ws.H[t] : nan;
    if (q) q[k] = f ? ws.q[t] : nan;
    if (coef) coef[k] = f ? ws.coef[t] : 0.f;
    if (bucket) bucket[k] = f ? ws.bucket[t] : 255;
    if (clip) clip[k] = f ? ws.clip[t] : 255;
    if (valid) valid[k] = f ? 1 : 0;
  }
}

__global__ void k_export_rollouts(const Workspace ws, int R, double* adv, uint8_t* zv,
                                  uint8_t* active, double* J, int32_t* nb, float* theta) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < R; i += gridDim.x * blockDim.x) {
    if (adv) adv[i] = ws.adv[i];
    if (zv) zv[i] = (ws.cand[i] && ws.zsign[i] == 0) ? 0 : 1;
    if (active) active[i] = ws.active[i];
    if (J) J[i] = ws.J[i];
    if (nb) nb[i] = ws.nb[i];
    if (theta)
      for (int k = 0; k < kMaxK - 1; ++k) theta[int64_t(i) * (kMaxK - 1) + k] = ws.theta[int64_t(i) * (kMaxK - 1) + k];
  }
}

}  // namespace espo
