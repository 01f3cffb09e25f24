"""CPU oracle for the ESPO policy-loss pass — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg
and ``--impl reference`` arm) may import, call or execute anything under ``oracle/``.
The product path (``paper_2512_07710_b200`` + ``libespo.so``) never touches this file,
and this file imports nothing from the product path: the two share no code.

What it computes (all arithmetic in IEEE fp64, plain loops / numpy primitives, in the
order the paper states the method; citations are ``PAPER.md:<line> (<section/eq>)``):

  O1  group_advantages   PAPER.md:77-79 (§2.4.1 zero-variance prompts, masking) and
                         PAPER.md:105-107 (§2.4.2, "normalized token-level advantage" Â,
                         GRPO group normalisation; formula from SPEC.md:332-337)
  O2  row_stats          PAPER.md:111 (Eq. 1 numerator π_θ(y_t|·)) and PAPER.md:119-121
                         (Eq. 3 token entropy e_t, bounded by log|V|)
  O3  partition          PAPER.md:103,109 (§2.4.2 "tokens are grouped by their entropy
                         values"), 80/20 split from PAPER.md:95
  O4  bucket_ratio_clip  PAPER.md:115 (Eq. 2 length-normalised ratio s_τ) and
                         PAPER.md:119 (Eq. 3 entropy-adaptive ε_τ)
  O5  token_surrogate    PAPER.md:105 (J_ESPO min/clip surrogate) and PAPER.md:111-113
                         (Eq. 1 with stop-gradient)
  O3-5 rollout_objective one rollout's J_i and ∂J_i/∂lp: O3 → O4 per bucket → O5, with the
                         1/|τ|·1/|y_τ| normalisers
  O6  espo_loss          PAPER.md:105 (expectation, 1/G, 1/|τ|, 1/|y_τ| normalisers)
  O7  dlogits            chain rule through log-softmax of the Eq. 1 numerator; every
                         sg[·] term is constant
  O8  frozen_surrogate   the sg-frozen objective used by the finite-difference pins
  O9  lmhead_grads       (§8(f) row 1) dh = dz·W, dW = dzᵀ·h for logits z = h·Wᵀ
                         (Megatron log-prob recompute)

Readings where the paper is silent/garbled (IDs from SURVEY.md §8(c)-2; all listed in
DESIGN.md "Readings"): Q1 ratio reading R2 (GSPO-token sg[π_θ] denominator) is the
default, R1 (literal sg[π_old]) is a flag; Q2 outer 1/|τ| = number of non-empty buckets;
Q3 K=2 quantile split at 4/5, ties to the low bucket; Q5 α=0.4, ε_min=0.01; Q6 |V| = row
width; Q7 population std, adv_eps=1e-6; Q8 exact-equality ZV test; Q10 N = active
rollouts; Q11 mask=0 tokens excluded; Q12 clip tie passes gradient; Q13 loss = −J;
Q14 log-ratio clamp ±20; Q15 logit_scale λ; Q16 −inf legal, NaN/+inf error.

Every function here is pinned by tests/test_oracle_*.py against closed forms, hand
examples (tests/golden/), brute force (mpmath, 50 digits), invariants, reductions to
GSPO-token / token-level PPO, finite differences and torch autograd.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PARTITION_QUANTILE = 0
PARTITION_WHOLE = 1
PARTITION_SINGLETON = 2

RATIO_GSPO_TOKEN = 0  # reading R2 (default)
RATIO_LITERAL_OLD = 1  # reading R1

NORM_SEQ = 0  # paper: 1/N_rollouts · 1/#buckets · 1/|y_τ|
NORM_TOKEN = 1  # 1/T_active

ZV_MASK = 0   # zero-variance groups eliminated (north_star default)
ZV_RLZVP = 1  # ZVE stage 3: RL-ZVP entropy-guided advantages

MAX_STAT_BUCKETS = 4


class OracleInputError(ValueError):
    """Input the method cannot be evaluated on. ``code`` mirrors espo_status names."""

    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


@dataclass
class OracleConfig:
    vocab: int
    alpha: float = 0.4
    eps_min: float = 0.01
    split_num: int = 4
    split_den: int = 5
    n_buckets: int = 2
    partition: int = PARTITION_QUANTILE
    ratio_mode: int = RATIO_GSPO_TOKEN
    norm: int = NORM_SEQ
    std_unbiased: bool = False
    adv_eps: float = 1e-6
    zv_var_eps: float = 0.0
    logit_scale: float = 1.0
    log_ratio_clamp: float = 20.0
    zv_mode: int = ZV_MASK
    zvp_beta: float = 0.05
    zvp_threshold: float = 0.5


# ----------------------------------------------------------------------------------------
# O1 — prompt groups, zero-variance mask, GRPO advantages
# ----------------------------------------------------------------------------------------
def group_advantages(rewards, group_ids, cfg: OracleConfig) -> dict:
    """O1. PAPER.md:77 (§2.4.1): a group whose rollouts "all receive identical rewards"
    has zero variance and zero advantage; PAPER.md:79,91 + north_star: such groups are
    masked out. Â_i = (r_i − μ_g)/(σ_g + adv_eps) (population std).

    Sums run sequentially in rollout-index order with one rounding per IEEE operation
    (Python floats, no FMA), so the result is reproducible bit for bit.
    """
    r = [float(x) for x in np.asarray(rewards, dtype=np.float32)]
    gid = [int(x) for x in np.asarray(group_ids)]
    R = len(r)
    if len(gid) != R:
        raise OracleInputError("ESPO_ERR_INVALID_ARGUMENT", "rewards/group_ids length")
    for i in range(R):
        if not math.isfinite(r[i]):
            raise OracleInputError("ESPO_ERR_NONFINITE_INPUT", f"reward {i} = {r[i]}")
    for i in range(1, R):
        if gid[i] < gid[i - 1]:
            raise OracleInputError("ESPO_ERR_GROUPS_NOT_CONTIGUOUS", f"group_ids[{i}]")

    # groups = maximal runs of equal ids
    groups = []
    start = 0
    for i in range(1, R + 1):
        if i == R or gid[i] != gid[start]:
            groups.append((start, i))
            start = i

    adv = [0.0] * R
    zv = [False] * R
    group_of = [0] * R
    means, stds, zv_g = [], [], []
    for g, (s, e) in enumerate(groups):
        n = e - s
        mu = 0.0
        for j in range(s, e):
            mu = mu + r[j]
        mu = mu / n
        ss = 0.0
        for j in range(s, e):
            d = r[j] - mu
            ss = ss + d * d
        denom = (n - 1) if cfg.std_unbiased else n
        var = ss / denom if denom > 0 else 0.0
        sigma = math.sqrt(var)
        if n < 2:
            is_zv = True
        elif cfg.zv_var_eps > 0.0:
            is_zv = var <= cfg.zv_var_eps
        else:
            is_zv = all(r[j] == r[s] for j in range(s, e))  # exact equality, +0 == -0
        for j in range(s, e):
            group_of[j] = g
            zv[j] = is_zv
            adv[j] = 0.0 if is_zv else (r[j] - mu) / (sigma + cfg.adv_eps)
        means.append(mu)
        stds.append(sigma)
        zv_g.append(is_zv)
    return {
        "adv": np.array(adv, dtype=np.float64),
        "zv": np.array(zv, dtype=bool),
        "group_of": np.array(group_of, dtype=np.int64),
        "groups": groups,
        "mean": np.array(means),
        "std": np.array(stds),
        "zv_group": np.array(zv_g, dtype=bool),
        "n_groups": len(groups),
        "n_zv_groups": int(sum(zv_g)),
    }


def zvp_token_advantages(H, reward: float, cfg: OracleConfig):
    """O1' (RL-ZVP, ZVE stage 3 "Advantage reshaping"; instantiation of the cited
    method from SPEC.md:338-343): for a rollout of a zero-variance group with reward r,
    a_t = β·s·(e_t − ē)/log|V|, s = +1 if r < threshold (all fail: favour exploration) else −1,
    ē = the rollout's mean token entropy. |a_t| ≤ β and Σ_t a_t = 0."""
    H = np.asarray(H, dtype=np.float64)
    sgn = 1.0 if reward < cfg.zvp_threshold else -1.0
    hbar = float(sum(H.tolist())) / len(H)
    return np.array([cfg.zvp_beta * sgn * (h - hbar) / math.log(cfg.vocab) for h in H.tolist()])


def reshape_reward(base: float, response, max_len: int, buffer: int = 0, ngram: int = 4,
                   gamma_rep: float = 1.0, rep_thresh: float = 0.2):
    """ZVE stage 2 "Reward reshaping" (length and repetition penalties; concrete
    form SPEC.md:262-265). Length penalty: 0 if len ≤ max_len − buffer, else linear from 0 to
    −1 on [max_len − buffer, max_len] (buffer = ⌈max_len/8⌉ by default), −1 beyond.
    Repetition penalty: −γ·max(0, f − thresh), f = fraction of the len−n+1 positions whose
    n-gram occurred at an earlier position. Returns (final, length_penalty, rep_penalty)."""
    toks = [int(t) for t in response]
    n = len(toks)
    buf = buffer if buffer > 0 else -(-max_len // 8)
    start = max_len - buf
    if n <= start:
        lpen = 0.0
    elif n >= max_len:
        lpen = -1.0
    else:
        lpen = -(n - start) / buf
    seen = set()
    rep = 0
    for p in range(n - ngram + 1):
        g = tuple(toks[p:p + ngram])
        if g in seen:
            rep += 1
        seen.add(g)
    frac = rep / (n - ngram + 1) if n >= ngram else 0.0
    rpen = -gamma_rep * max(0.0, frac - rep_thresh)
    return base + lpen + rpen, lpen, rpen


# ----------------------------------------------------------------------------------------
# O2 — per-token log-softmax statistics
# ----------------------------------------------------------------------------------------
def row_stats(z_row, y: int, logit_scale: float = 1.0):
    """O2. For one logits row z (the distribution that produced token y):
    x = λ·z, p = softmax(x), lse = log Σ e^x, lp = log p_y (π_θ(y_t|·)),
    H = −Σ p log p with 0·log 0 := 0 (PAPER.md:119 e_t), q = Σ_{v≠y} p_v.
    Returns (lse, lp, H, q) in fp64.
    """
    x = float(logit_scale) * np.asarray(z_row, dtype=np.float64)
    if np.isnan(x).any() or np.isposinf(x).any():
        raise OracleInputError("ESPO_ERR_NONFINITE_INPUT", "NaN/+inf logit")
    if not (0 <= y < x.shape[0]):
        raise OracleInputError("ESPO_ERR_TOKEN_OUT_OF_RANGE", f"token {y}")
    if x[y] == -np.inf:
        # a token of probability 0 cannot have been sampled; lp would be −inf
        raise OracleInputError("ESPO_ERR_NONFINITE_INPUT", "target logit is -inf")
    M = x.max()
    e = np.exp(x - M)
    S = e.sum()
    lse = M + math.log(S)
    p = e / S
    lp = x[y] - lse
    nz = p > 0.0
    H = -float(np.sum(p[nz] * np.log(p[nz])))
    q = float(np.sum(p[:y]) + np.sum(p[y + 1:]))
    return float(lse), float(lp), H, q


# ----------------------------------------------------------------------------------------
# O3 — entropy partition of one sequence
# ----------------------------------------------------------------------------------------
def split_ranks(n: int, cfg: OracleConfig):
    """The 1-based order statistics that define the K−1 entropy thresholds (reading Q3):
    K=2: rank max(⌊split_num·n/split_den⌋, 1) (80/20); K>2: max(⌊k·n/K⌋, 1)."""
    K = cfg.n_buckets
    if K == 2:
        return [max((cfg.split_num * n) // cfg.split_den, 1)]
    return [max((k * n) // K, 1) for k in range(1, K)]


def partition(H, cfg: OracleConfig):
    """O3. PAPER.md:109: "Within each sequence, tokens are grouped by their entropy
    values". Returns (bucket index per token, number of non-empty buckets nb).
    Quantile mode: θ_k = the rank-th smallest H (full sort); bucket = #{k : H > θ_k},
    so ties go to the lower bucket and bucket ids keep their pre-drop index.
    WHOLE: every token in bucket 0 (GSPO-token). SINGLETON: each token its own bucket.
    """
    H = np.asarray(H, dtype=np.float64)
    n = H.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.int64), 0
    if cfg.partition == PARTITION_WHOLE or cfg.n_buckets == 1:
        return np.zeros(n, dtype=np.int64), 1
    if cfg.partition == PARTITION_SINGLETON:
        return np.arange(n, dtype=np.int64), n
    srt = sorted(H.tolist())
    thetas = [srt[rank - 1] for rank in split_ranks(n, cfg)]
    b = np.array([sum(1 for th in thetas if h > th) for h in H.tolist()], dtype=np.int64)
    nb = len(set(b.tolist()))
    return b, nb


# ----------------------------------------------------------------------------------------
# O4 — per-bucket ratio (Eq. 2) and entropy-adaptive clip (Eq. 3)
# ----------------------------------------------------------------------------------------
def bucket_ratio_clip(lp, old, H, cfg: OracleConfig):
    """O4 for the tokens of ONE bucket τ (arrays over its tokens, index order).
    Eq. 2: s_τ = (Π π_θ/π_old)^{1/|y_τ|} = exp(Σ(lp−old)/|y_τ|), with the
    log-ratio clamped to ±log_ratio_clamp (reading Q14; 0 = off).
    Eq. 3: ε_τ = (α/|y_τ|) Σ e_t / log|V|, floored at ε_min (reading Q5).
    """
    n = len(lp)
    delta = 0.0
    for a, b in zip(np.asarray(lp, dtype=np.float64).tolist(),
                    np.asarray(old, dtype=np.float64).tolist()):
        delta += a - b
    m = delta / n
    c = cfg.log_ratio_clamp
    if c > 0:
        m = min(max(m, -c), c)
    s = math.exp(m)
    hsum = float(sum(np.asarray(H, dtype=np.float64).tolist()))
    eps = max(cfg.eps_min, cfg.alpha * hsum / (n * math.log(cfg.vocab)))
    return s, eps


# ----------------------------------------------------------------------------------------
# O5 — token surrogate
# ----------------------------------------------------------------------------------------
def token_surrogate(v: float, A: float, eps: float):
    """O5. PAPER.md:105: ℓ = min(v·Â, clip(v, 1−ε, 1+ε)·Â). κ = 1 unless the clipped
    branch is strictly active (then ∂ℓ/∂v = 0); a tie at v = 1±ε passes (reading Q12)."""
    lo, hi = 1.0 - eps, 1.0 + eps
    vc = min(max(v, lo), hi)
    ell = min(v * A, vc * A)
    kappa = not ((A > 0 and v > hi) or (A < 0 and v < lo))
    return ell, kappa


# ----------------------------------------------------------------------------------------
# O3-O5 composed — one rollout's ESPO objective J_i
# ----------------------------------------------------------------------------------------
def rollout_objective(lp, old, H, A_t, cfg: OracleConfig, inject_bucket=None,
                      inject_kappa=None) -> dict:
    """One active rollout i with valid tokens t = 0..n−1 (index order), PAPER.md:105-121:

      J_i = (1/|τ|) Σ_τ (1/|y_τ|) Σ_{t∈y_τ} min(v_t·Â_t, clip(v_t, 1−ε_τ, 1+ε_τ)·Â_t)

    with the buckets τ of O3 (|τ| = nb, the number of non-empty buckets, reading Q2),
    s_τ from Eq. 2 and ε_τ from Eq. 3 evaluated over the bucket's own tokens (O4), and
    v_t = s_τ (reading R2: sg[s_τ]·π_θ/sg[π_θ]) or v_t = s_τ·π_θ/π_old
    (R1, the literal sg[π_old] denominator). NORM_TOKEN replaces 1/(nb·|y_τ|) by 1.

    ∂J_i/∂lp_t: every sg[·] is constant, so only the Eq. 1 numerator
    π_θ(y_t) varies and ∂v_t/∂lp_t = v_t; the min picks the clipped branch (slope 0) when
    it is strictly smaller (O5's κ): ∂J_i/∂lp_t = κ_t·Â_t·v_t·w_t, w_t = 1/(nb·|y_τ|).

    Inputs: lp, old, H, A_t — arrays over the rollout's valid tokens. ``inject_*`` replace
    the bucket / clip decisions (P11 decision-aware protocol). Returns per-token arrays
    (bucket, kappa, v, s, eps, w, ell, dJ_dlp) and J, nb, theta."""
    lp = np.asarray(lp, dtype=np.float64)
    old = np.asarray(old, dtype=np.float64)
    H = np.asarray(H, dtype=np.float64)
    A_t = np.asarray(A_t, dtype=np.float64)
    n = len(lp)
    b, nb = partition(H, cfg)
    theta = None
    if cfg.partition == PARTITION_QUANTILE and cfg.n_buckets > 1 and n > 0:
        srt = sorted(H.tolist())
        theta = [srt[rk - 1] for rk in split_ranks(n, cfg)]
    if inject_bucket is not None and cfg.partition == PARTITION_QUANTILE:
        b = np.asarray(inject_bucket).astype(np.int64)
        nb = len(set(b.tolist()))
    out = {k: np.zeros(n) for k in ("v", "s", "eps", "w", "ell", "dJ_dlp")}
    out["bucket"] = np.zeros(n, dtype=np.int64)
    out["kappa"] = np.zeros(n, dtype=bool)
    Ji = 0.0
    for k in sorted(set(b.tolist())):
        sel = np.nonzero(b == k)[0]
        size = len(sel)
        s, eps = bucket_ratio_clip(lp[sel], old[sel], H[sel], cfg)
        w = 1.0 / (nb * size) if cfg.norm == NORM_SEQ else 1.0
        for j in sel.tolist():
            if cfg.ratio_mode == RATIO_GSPO_TOKEN:
                v = s                     # sg[s_τ]·π_θ/sg[π_θ]: value s_τ
            else:
                v = s * math.exp(lp[j] - old[j])
            At = float(A_t[j])
            ell, kap = token_surrogate(v, At, eps)
            if inject_kappa is not None:
                kap = bool(np.asarray(inject_kappa)[j])
            Ji += w * ell
            out["dJ_dlp"][j] = At * v * w if kap else 0.0
            out["bucket"][j] = 0 if cfg.partition != PARTITION_QUANTILE else k
            out["kappa"][j] = kap
            out["v"][j], out["s"][j], out["eps"][j], out["w"][j], out["ell"][j] = v, s, eps, w, ell
    out.update(J=Ji, nb=nb, theta=theta)
    return out


# ----------------------------------------------------------------------------------------
# O6/O7 — the whole pass
# ----------------------------------------------------------------------------------------
@dataclass
class OracleResult:
    loss: float
    J_sum: float
    denom: float
    adv: np.ndarray
    zv: np.ndarray
    active: np.ndarray
    n_valid: np.ndarray
    J_i: np.ndarray
    nb: np.ndarray
    lse: np.ndarray
    lp: np.ndarray
    H: np.ndarray
    q: np.ndarray
    bucket: np.ndarray       # stats bucket per token (−1 if not evaluated)
    kappa: np.ndarray        # 1/0 per token (−1 if not evaluated)
    v: np.ndarray
    eps_tok: np.ndarray      # ε_τ of the token's bucket
    s_tok: np.ndarray        # s_τ of the token's bucket
    coef: np.ndarray         # c_t = ∂J_i/∂lp_t (before 1/D)
    adv_tok: np.ndarray      # advantage used for each token (NaN if not evaluated)
    w_tok: np.ndarray        # normaliser weight of the token inside J_i
    theta: dict = field(default_factory=dict)   # rollout -> thresholds (quantile mode)
    stats: dict = field(default_factory=dict)
    group: dict = field(default_factory=dict)


def espo_loss(logits, tokens, old_logp, mask, rewards, group_ids, seq_offsets,
              cfg: OracleConfig, row_key=None, inject_bucket=None, inject_kappa=None,
              stats_cache=None, entropy=None) -> OracleResult:
    """O6: J = (1/D) Σ_i J_i, loss = −J (reading Q13), where for active
    rollout i with non-empty buckets τ:  J_i = Σ_τ (1/(nb_i·|y_τ|)) Σ_{t∈τ} ℓ_t  and
    D = number of active rollouts (reading Q10; NORM_TOKEN: J_i = Σ_t ℓ_t, D = T_active).

    logits[t] must give row t (an array [T, V] or any indexable); rows of zero-variance
    or inactive rollouts and masked tokens are never read (P3). ``row_key(t)`` lets rows
    that are bit-identical share one O2 evaluation (memoised on (key, y)).
    ``inject_bucket``/``inject_kappa`` (per-token arrays) replace the oracle's own
    bucket / clip decisions (P11 decision-aware protocol).
    ``entropy`` (per-token array, optional): caller-supplied selection entropies — reading
    Q4's alternative (SPEC.md:460 takes the rollout policy's
    entropies) — used in place of the computed H_t wherever the method uses e_t: the
    partition (O3), ε_τ (O4, Eq. 3), RL-ZVP's token advantages
     and the mean-entropy statistic. lse, lp, q and H themselves still come
    from the logits (O2); the gradient is unchanged in form (entropies are detached).
    """
    tokens = np.asarray(tokens)
    old_logp = np.asarray(old_logp, dtype=np.float32).astype(np.float64)
    seq_offsets = np.asarray(seq_offsets, dtype=np.int64)
    T = int(seq_offsets[-1])
    R = len(seq_offsets) - 1
    mask = np.ones(T, dtype=bool) if mask is None else np.asarray(mask).astype(bool)
    grp = group_advantages(rewards, group_ids, cfg)
    if seq_offsets[0] != 0 or np.any(np.diff(seq_offsets) < 0):
        raise OracleInputError("ESPO_ERR_INVALID_ARGUMENT", "seq_offsets")
    V = cfg.vocab
    if stats_cache is None:
        stats_cache = {}

    nanT = lambda: np.full(T, np.nan)
    lse_a, lp_a, H_a, q_a = nanT(), nanT(), nanT(), nanT()
    v_a, eps_a, s_a, coef_a, w_a = nanT(), nanT(), nanT(), np.zeros(T), nanT()
    bucket_a = np.full(T, -1, dtype=np.int64)
    kappa_a = np.full(T, -1, dtype=np.int64)
    active = np.zeros(R, dtype=bool)
    n_valid = np.zeros(R, dtype=np.int64)
    J_i = np.zeros(R)
    nb_a = np.zeros(R, dtype=np.int64)
    theta = {}

    K = MAX_STAT_BUCKETS
    tok_k = np.zeros(K)
    clip_k = np.zeros(K)
    vsum_k = np.zeros(K)
    esum_k = np.zeros(K)
    sum_abs_lr = 0.0
    sum_sq_lr = 0.0
    sum_k3 = 0.0
    sum_H = 0.0
    n_clipped = 0

    rewards32 = np.asarray(rewards, dtype=np.float32)
    adv_tok = np.full(T, np.nan)
    for i in range(R):
        zvp = bool(grp["zv"][i]) and cfg.zv_mode == ZV_RLZVP
        if grp["zv"][i] and not zvp:
            continue                       # eliminated group: never read (P3)
        rows = np.arange(seq_offsets[i], seq_offsets[i + 1])
        valid = rows[mask[rows]]
        n = len(valid)
        n_valid[i] = n
        if n == 0:
            continue
        active[i] = True
        A = float(grp["adv"][i])
        lp = np.empty(n)
        H = np.empty(n)
        for j, t in enumerate(valid.tolist()):
            y = int(tokens[t])
            key = (row_key(t), y) if row_key is not None else None
            if key is not None and key in stats_cache:
                st = stats_cache[key]
            else:
                st = row_stats(logits[t], y, cfg.logit_scale)
                if key is not None:
                    stats_cache[key] = st
            lse_a[t], lp_a[t], H_a[t], q_a[t] = st
            lp[j], H[j] = st[1], st[2]
        old = old_logp[valid]
        if entropy is not None:      # caller-supplied selection entropies (reading Q4 alt.)
            H = np.asarray(entropy, dtype=np.float64)[valid]
        # per-token advantages: the group's Â broadcast, or RL-ZVP's a_t
        A_t = zvp_token_advantages(H, float(rewards32[i]), cfg) if zvp else np.full(n, A)
        adv_tok[valid] = A_t

        # O3-O5 for this rollout
        inj_b = None if inject_bucket is None else np.asarray(inject_bucket)[valid]
        inj_k = None if inject_kappa is None else np.asarray(inject_kappa)[valid]
        ro = rollout_objective(lp, old, H, A_t, cfg, inject_bucket=inj_b, inject_kappa=inj_k)
        if ro["theta"] is not None:
            theta[i] = ro["theta"]
        nb_a[i] = ro["nb"]
        for j, t in enumerate(valid.tolist()):
            kap = bool(ro["kappa"][j])
            sk = int(ro["bucket"][j])
            coef_a[t] = ro["dJ_dlp"][j]
            bucket_a[t] = sk
            kappa_a[t] = 1 if kap else 0
            v_a[t], eps_a[t], s_a[t], w_a[t] = ro["v"][j], ro["eps"][j], ro["s"][j], ro["w"][j]
            tok_k[sk] += 1
            clip_k[sk] += 0 if kap else 1
            vsum_k[sk] += ro["v"][j]
            esum_k[sk] += ro["eps"][j]
            n_clipped += 0 if kap else 1
            d_lr = lp[j] - old[j]
            sum_abs_lr += abs(d_lr)
            sum_sq_lr += d_lr * d_lr
            # k3 estimator of KL(π_old ‖ π_θ) from samples y ~ π_old: r − 1 − log r,
            # r = π_θ(y)/π_old(y) (train/inference mismatch)
            sum_k3 += math.expm1(d_lr) - d_lr
            sum_H += H[j]
        J_i[i] = ro["J"]

    n_active = int(active.sum())
    t_active = int(n_valid[active].sum())
    denom = float(n_active if cfg.norm == NORM_SEQ else t_active)
    J_sum = float(J_i.sum())
    J = J_sum / denom if denom > 0 else 0.0
    loss = -J if denom > 0 else 0.0
    stats = {
        "loss": loss,
        "n_active_rollouts": n_active,
        "n_active_tokens": t_active,
        "n_zv_groups": grp["n_zv_groups"],
        "n_groups": grp["n_groups"],
        "n_clipped_tokens": n_clipped,
        "mean_abs_logratio": sum_abs_lr / t_active if t_active else 0.0,
        "mean_entropy": sum_H / t_active if t_active else 0.0,
        "clip_frac": [clip_k[k] / tok_k[k] if tok_k[k] else 0.0 for k in range(K)],
        "mean_ratio": [vsum_k[k] / tok_k[k] if tok_k[k] else 0.0 for k in range(K)],
        "mean_eps": [esum_k[k] / tok_k[k] if tok_k[k] else 0.0 for k in range(K)],
        "tokens_per_bucket": tok_k.tolist(),
        "mean_sq_logratio": sum_sq_lr / t_active if t_active else 0.0,
        "mean_k3": sum_k3 / t_active if t_active else 0.0,
    }
    return OracleResult(loss=loss, J_sum=J_sum, denom=denom, adv=grp["adv"], zv=grp["zv"],
                        active=active, n_valid=n_valid, J_i=J_i, nb=nb_a, lse=lse_a,
                        lp=lp_a, H=H_a, q=q_a, bucket=bucket_a, kappa=kappa_a, v=v_a,
                        eps_tok=eps_a, s_tok=s_a, coef=coef_a, adv_tok=adv_tok, w_tok=w_a,
                        theta=theta,
                        stats=stats,
                        group=grp)


def dlogits_row(res: OracleResult, t: int, z_row, y: int, cfg: OracleConfig,
                grad_loss: float = 1.0) -> np.ndarray:
    """O7. d loss/d z_{t,v} = λ·g_t·(1[v = y] − p_v), g_t = −grad_loss·c_t/D, because only
    the Eq. 1 numerator log π_θ(y_t) carries gradient (sg) and
    ∂ log softmax(λz)_y/∂z_v = λ(1[v=y] − p_v). The target entry uses q_t = Σ_{v≠y} p_v.
    Rows of inactive rollouts / masked tokens / eliminated groups are 0."""
    V = len(z_row)
    if np.isnan(res.lp[t]) or res.denom == 0:
        return np.zeros(V)
    lam = cfg.logit_scale
    g = -grad_loss * res.coef[t] / res.denom
    x = lam * np.asarray(z_row, dtype=np.float64)
    p = np.exp(x - res.lse[t])
    dz = lam * g * (-p)
    dz[y] = lam * g * res.q[t]
    return dz


def frozen_surrogate_loss(logits_eval, res: OracleResult, tokens, old_logp, seq_offsets,
                          cfg: OracleConfig, grad_loss: float = 1.0) -> float:
    """Frozen-sg surrogate F(z; z0) used for finite differences: every
    sg[·] (s_τ, the R2 denominator lp_t), ε_τ, the partition, Â and D are taken from
    ``res`` (evaluated at z0); only the Eq. 1 numerator lp_t(z) varies with z."""
    old_logp = np.asarray(old_logp, dtype=np.float32).astype(np.float64)
    J = 0.0
    R = len(seq_offsets) - 1
    for i in range(R):
        if not res.active[i]:
            continue
        for t in range(int(seq_offsets[i]), int(seq_offsets[i + 1])):
            if res.kappa[t] < 0:
                continue
            A = float(res.adv_tok[t])
            _, lp_z, _, _ = row_stats(logits_eval[t], int(tokens[t]), cfg.logit_scale)
            if cfg.ratio_mode == RATIO_GSPO_TOKEN:
                v = res.s_tok[t] * math.exp(lp_z - res.lp[t])
            else:
                v = res.s_tok[t] * math.exp(lp_z - old_logp[t])
            ell, _ = token_surrogate(v, A, res.eps_tok[t])
            J += res.w_tok[t] * ell
    return -grad_loss * J / res.denom if res.denom > 0 else 0.0


def lmhead_grads(res: OracleResult, hidden, weight, tokens, cfg: OracleConfig,
                 grad_loss: float = 1.0):
    """O9 (the LM head in front of the path; Megatron log-prob recompute,
    PAPER.md:129-131). With logits z = h·Wᵀ (row t: z_t = W h_t), the chain rule through
    O7 gives dL/dh_t = Σ_v dz_{t,v} W_v and dL/dW_v = Σ_t dz_{t,v} h_t, i.e.
    dh = dz·W and dW = dzᵀ·h, where dz is O7's matrix on z = h·Wᵀ in fp64.
    Returns (dz, dh, dW), all fp64."""
    h = np.asarray(hidden, dtype=np.float64)
    W = np.asarray(weight, dtype=np.float64)
    z = h @ W.T
    dz = np.stack([dlogits_row(res, t, z[t], int(tokens[t]), cfg, grad_loss)
                   for t in range(h.shape[0])])
    return dz, dz @ W, dz.T @ h
