"""Seeded synthetic inputs for the ESPO loss pass (shared by tests, smoke and bench).

This module holds NONE of the method's arithmetic: no softmax, log-softmax, entropy,
advantage, partition or ratio. It only draws random numbers in the shapes and with the
structure of the paper's workloads (BASELINE.json configs C0–C4, recipe in DESIGN.md
"Input recipe"):

- prompt groups of G rollouts ("{y_i}_{i=1}^G ~ π_old"), binary rewards
  Bernoulli(p_g), p_g ~ U(0,1) (verifier/GenRM rewards are {0,1}: PAPER.md:195,207),
  with forced uniform-reward (zero-variance) groups where the config asks for them;
- packed rollouts (cu_seqlens), fixed or lognormal lengths (long tail);
- logits rows shaped like LLM next-token distributions with an 80/20 entropy mix
  (PAPER.md:95): background N(0,1) − (ln V + 2.07); 20% of rows "high entropy"
  (k ~ U{2..8} candidates ~ N(0,1)), 80% with one dominant id ~ U(2, 8);
- sampled tokens by the Gumbel-max trick (argmax(z + Gumbel) — exact sampling without
  evaluating a softmax);
- rollout-engine log-probs as a drift added to a CALLER-SUPPLIED lp (the caller gets lp
  from the oracle in tests, from torch.log_softmax in bench setup).

All randomness: numpy Philox keyed by (seed, stream...) — `rng_for`; torch variants use a
torch.Generator seeded from the same 64-bit seed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MASTER_SEED = 20251207
MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def config_seed(index: int) -> int:
    return splitmix64(MASTER_SEED ^ index)


def rng_for(seed: int, *stream: int) -> np.random.Generator:
    ss = np.random.SeedSequence([seed & MASK64, *[s & MASK64 for s in stream]])
    return np.random.Generator(np.random.Philox(ss))


@dataclass(frozen=True)
class Workload:
    name: str
    index: int
    n_prompts: int
    G: int
    L: int                  # tokens per rollout (max if var_len)
    V: int
    dtype: str              # "f32" | "bf16"
    forced_zv: int = 0      # number of groups forced to uniform rewards
    var_len: bool = False   # lognormal lengths clamp(round(lognormal(ln 3000, 0.8)), 64, L)
    mask_tail: int = 0      # mask=0 on the last u ~ U{0..mask_tail} rows of each rollout

    @property
    def R(self) -> int:
        return self.n_prompts * self.G


WORKLOADS = {
    "C0": Workload("C0", 0, 4, 4, 64, 1024, "f32", forced_zv=1, mask_tail=16),
    "C1": Workload("C1", 1, 64, 8, 4096, 151936, "bf16"),
    "C2": Workload("C2", 2, 32, 16, 32768, 151936, "bf16"),
    "C3": Workload("C3", 3, 256, 16, 8192, 151936, "bf16", forced_zv=154, var_len=True),
    "C4": Workload("C4", 4, 512, 16, 16384, 151936, "bf16"),
}


def make_layout(w: Workload, seed: int):
    """group_ids int32[R] (contiguous, non-decreasing), seq_offsets int64[R+1]."""
    group_ids = np.repeat(np.arange(w.n_prompts, dtype=np.int32), w.G)
    if w.var_len:
        rng = rng_for(seed, 1)
        L = np.round(rng.lognormal(np.log(3000.0), 0.8, size=w.R))
        lengths = np.clip(L, 64, w.L).astype(np.int64)
    else:
        lengths = np.full(w.R, w.L, dtype=np.int64)
    seq_offsets = np.zeros(w.R + 1, dtype=np.int64)
    np.cumsum(lengths, out=seq_offsets[1:])
    return group_ids, seq_offsets


def make_rewards(w: Workload, seed: int, forced_groups=None) -> np.ndarray:
    """Binary rewards. Forced groups get uniform rewards (alternating all-1 / all-0);
    C0 forces group 2 to all-1 and resamples the others until mixed."""
    rng = rng_for(seed, 2)
    r = np.zeros((w.n_prompts, w.G), dtype=np.float32)
    if forced_groups is None:
        if w.name == "C0":
            forced_groups = [2]
        else:
            forced_groups = sorted(rng.choice(w.n_prompts, size=w.forced_zv,
                                              replace=False).tolist()) if w.forced_zv else []
    forced = set(forced_groups)
    for g in range(w.n_prompts):
        if g in forced:
            r[g, :] = 1.0 if (g % 2 == 0) else 0.0
            continue
        while True:
            p = rng.uniform()
            r[g] = (rng.uniform(size=w.G) < p).astype(np.float32)
            if not w.forced_zv or w.G < 2 or r[g].min() != r[g].max():
                break
    return r.reshape(-1)


def make_mask(w: Workload, seq_offsets: np.ndarray, seed: int) -> np.ndarray:
    T = int(seq_offsets[-1])
    m = np.ones(T, dtype=np.uint8)
    if w.mask_tail:
        rng = rng_for(seed, 3)
        for i in range(len(seq_offsets) - 1):
            u = int(rng.integers(0, w.mask_tail + 1))
            if u:
                m[seq_offsets[i + 1] - u: seq_offsets[i + 1]] = 0
    return m


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 → bfloat16 (round-to-nearest-even); returned widened as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32)
    b = (u >> 16) & np.uint32(1)
    b += np.uint32(0x7FFF)
    b += u                                   # uint32 wrap only for NaN payloads (fixed below)
    b &= np.uint32(0xFFFF0000)
    out = b.view(np.float32).reshape(a.shape)
    nan = np.isnan(a)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out


def bf16_bits(a_bf16_valued: np.ndarray) -> np.ndarray:
    """uint16 storage of float32 values that are exactly bf16-representable."""
    return (np.ascontiguousarray(a_bf16_valued, dtype=np.float32).view(np.uint32) >> 16
            ).astype(np.uint16)


def make_logit_rows(n_rows: int, V: int, seed: int, stream: int = 4,
                    dtype: str = "f32") -> np.ndarray:
    """Structured logits rows [n_rows, V] (float32; bf16-valued if dtype == 'bf16')."""
    rng = rng_for(seed, stream)
    B = np.log(V) + 2.07
    z = rng.standard_normal((n_rows, V), dtype=np.float32) - np.float32(B)
    high = rng.uniform(size=n_rows) < 0.2
    for r in range(n_rows):
        if high[r]:
            k = int(rng.integers(2, 9))
            ids = np.unique(rng.integers(0, V, size=k))   # distinct candidate ids
            z[r, ids] = rng.standard_normal(len(ids)).astype(np.float32)
        else:
            z[r, int(rng.integers(0, V))] = np.float32(rng.uniform(2.0, 8.0))
    if dtype == "bf16":
        z = round_to_bf16(z)
    return z


def sample_tokens_gumbel(rows: np.ndarray, seed: int, stream: int = 5,
                         logit_scale: float = 1.0) -> np.ndarray:
    """y_t ~ softmax(λ z_t) by the Gumbel-max trick: argmax_v (λ z_v + G_v)."""
    rng = rng_for(seed, stream)
    out = np.empty(rows.shape[0], dtype=np.int32)
    for r in range(rows.shape[0]):
        u = rng.uniform(np.finfo(np.float64).tiny, 1.0, size=rows.shape[1])
        g = -np.log(-np.log(u))
        out[r] = int(np.argmax(logit_scale * rows[r].astype(np.float64) + g))
    return out


def drift_old_logp(lp: np.ndarray, seq_offsets: np.ndarray, seed: int,
                   sigma_seq: float = 0.04, sigma_tok: float = 0.02) -> np.ndarray:
    """Rollout-engine log-probs: old_t = lp_t + b_i + σ_tok·n_t, b_i ~ N(0, σ_seq) per
    rollout (train/infer mismatch). ``lp`` is supplied by the caller."""
    rng = rng_for(seed, 6)
    R = len(seq_offsets) - 1
    lengths = np.diff(seq_offsets)
    b = np.repeat(rng.normal(0.0, sigma_seq, size=R), lengths)
    n = rng.standard_normal(int(seq_offsets[-1]))
    old = np.asarray(lp, dtype=np.float64) + b + sigma_tok * n
    return old.astype(np.float32)


# ---------------------------------------------------------------------------------------
# torch variants (device-side generation of large buffers; bench + full-size GPU tests)
# ---------------------------------------------------------------------------------------
def make_logit_rows_torch(n_rows: int, V: int, seed: int, device, dtype,
                          rows_per_call: int = 2048):
    """Same recipe as make_logit_rows, drawn on `device` with torch.Generator (values are
    NOT bit-identical to the numpy variant; parity tests copy the buffer to the host)."""
    import torch
    out = torch.empty((n_rows, V), dtype=dtype, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed & ((1 << 63) - 1))
    B = float(np.log(V) + 2.07)
    for r0 in range(0, n_rows, rows_per_call):
        n = min(rows_per_call, n_rows - r0)
        z = torch.randn((n, V), generator=g, device=device, dtype=torch.float32) - B
        high = torch.rand((n,), generator=g, device=device) < 0.2
        k = torch.randint(2, 9, (n,), generator=g, device=device)
        ids = torch.randint(0, V, (n, 8), generator=g, device=device)
        vals_high = torch.randn((n, 8), generator=g, device=device)
        vals_low = torch.rand((n, 1), generator=g, device=device) * 6.0 + 2.0
        j = torch.arange(8, device=device).unsqueeze(0)
        use = torch.where(high.unsqueeze(1), j < k.unsqueeze(1), j == 0)
        vals = torch.where(high.unsqueeze(1), vals_high, vals_low.expand(n, 8))
        cur = torch.gather(z, 1, ids)
        z.scatter_(1, ids, torch.where(use, vals, cur))
        out[r0:r0 + n].copy_(z.to(dtype))
    return out


def sample_tokens_gumbel_torch(rows, seed: int, logit_scale: float = 1.0,
                               rows_per_call: int = 2048):
    import torch
    g = torch.Generator(device=rows.device)
    g.manual_seed((seed ^ 0x5bd1e995) & ((1 << 63) - 1))
    out = torch.empty(rows.shape[0], dtype=torch.int32, device=rows.device)
    for r0 in range(0, rows.shape[0], rows_per_call):
        n = min(rows_per_call, rows.shape[0] - r0)
        u = torch.rand((n, rows.shape[1]), generator=g, device=rows.device,
                       dtype=torch.float64).clamp_min(1e-300)
        gum = -torch.log(-torch.log(u))
        out[r0:r0 + n] = torch.argmax(logit_scale * rows[r0:r0 + n].double() + gum,
                                      dim=1).to(torch.int32)
    return out
