"""Small seeded ESPO instances for tests (inputs only; expected values come from oracle/)."""
from __future__ import annotations

import numpy as np

import espo_synth as S
from oracle import espo_oracle as O


class Instance:
    def __init__(self, logits, tokens, old_logp, mask, rewards, group_ids, seq_offsets, V,
                 dtype="f32"):
        self.logits = logits
        self.tokens = tokens
        self.old_logp = old_logp
        self.mask = mask
        self.rewards = rewards
        self.group_ids = group_ids
        self.seq_offsets = seq_offsets
        self.V = V
        self.dtype = dtype

    @property
    def T(self):
        return int(self.seq_offsets[-1])

    @property
    def R(self):
        return len(self.seq_offsets) - 1

    def run(self, cfg, **kw):
        return O.espo_loss(self.logits, self.tokens, self.old_logp, self.mask, self.rewards,
                           self.group_ids, self.seq_offsets, cfg, **kw)


def exact_lp(logits, tokens, logit_scale=1.0):
    """lp of every row via the oracle (used only to build realistic old_logp inputs)."""
    return np.array([O.row_stats(logits[t], int(tokens[t]), logit_scale)[1]
                     for t in range(logits.shape[0])])


def tiny_instance(seed, V=7, group_sizes=(3, 3), lengths=None, L=5, sigma_seq=0.1,
                  sigma_tok=0.05, rewards=None, mask_tail=0, logit_scale=1.0, dtype="f32"):
    """Random tiny batch: explicit group sizes, per-rollout lengths, drifted old_logp."""
    rng = S.rng_for(seed, 100)
    R = int(sum(group_sizes))
    group_ids = np.repeat(np.arange(len(group_sizes), dtype=np.int32), group_sizes)
    if lengths is None:
        lengths = [L] * R
    seq_offsets = np.zeros(R + 1, dtype=np.int64)
    np.cumsum(lengths, out=seq_offsets[1:])
    T = int(seq_offsets[-1])
    logits = S.make_logit_rows(T, V, seed, dtype=dtype) if V >= 64 else \
        (rng.standard_normal((T, V)) * 2.0).astype(np.float32)
    if dtype == "bf16":
        logits = S.round_to_bf16(logits)
    tokens = S.sample_tokens_gumbel(logits, seed, logit_scale=logit_scale)
    if rewards is None:
        rewards = np.zeros(R, dtype=np.float32)
        i = 0
        for g in group_sizes:
            while True:
                r = (rng.uniform(size=g) < 0.5).astype(np.float32)
                if g < 2 or r.min() != r.max():
                    break
            rewards[i:i + g] = r
            i += g
    mask = np.ones(T, dtype=np.uint8)
    if mask_tail:
        for i in range(R):
            u = int(rng.integers(0, mask_tail + 1))
            if u:
                mask[seq_offsets[i + 1] - u: seq_offsets[i + 1]] = 0
    lp = exact_lp(logits, tokens, logit_scale)
    old = S.drift_old_logp(lp, seq_offsets, seed, sigma_seq=sigma_seq, sigma_tok=sigma_tok)
    return Instance(logits, tokens, old, mask, np.asarray(rewards, np.float32), group_ids,
                    seq_offsets, V, dtype)


def workload_instance(name, seed=None, n_prompts=None, L=None, V=None):
    """A (possibly shrunk) instance of a BASELINE workload recipe, generated on the CPU."""
    w = S.WORKLOADS[name]
    kw = {}
    if n_prompts is not None:
        kw["n_prompts"] = n_prompts
        kw["forced_zv"] = min(w.forced_zv, n_prompts)
    if L is not None:
        kw["L"] = L
    if V is not None:
        kw["V"] = V
    if kw:
        from dataclasses import replace
        w = replace(w, **kw)
    seed = S.config_seed(w.index) if seed is None else seed
    group_ids, seq_offsets = S.make_layout(w, seed)
    rewards = S.make_rewards(w, seed)
    mask = S.make_mask(w, seq_offsets, seed)
    T = int(seq_offsets[-1])
    logits = S.make_logit_rows(T, w.V, seed, dtype=w.dtype)
    tokens = S.sample_tokens_gumbel(logits, seed)
    lp = exact_lp(logits, tokens)
    old = S.drift_old_logp(lp, seq_offsets, seed)
    return Instance(logits, tokens, old, mask, rewards, group_ids, seq_offsets, w.V, w.dtype)
