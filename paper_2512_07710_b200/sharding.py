"""Host-side sharding of a global ESPO batch over data-parallel ranks.

Every coupling of the ESPO loss is inside a rollout (entropy buckets, s_τ, ε_τ) or inside a
prompt group (μ, σ, zero-variance test), so whole prompt groups go to ranks and no logits,
log-probs or entropies ever cross GPUs; the only exchange is the all-reduce of the
normaliser and loss terms inside espo_loss_finalize. Groups are assigned by LPT
(longest-processing-time first) on their expected sweep cost — the paper's own
length-balanced scheduling idea (§3.1.1) applied to the loss pass — or in
contiguous blocks. Plain numpy; identical on every rank given the same inputs.
"""
from __future__ import annotations

import heapq

import numpy as np

# relative per-token cost: an active row is read twice and written once (6V bytes), a row
# of an eliminated group is only zero-filled (2V bytes)
COST_ACTIVE, COST_ELIMINATED = 3.0, 1.0


def group_spans(group_ids):
    """[(first_rollout, end_rollout)] for each maximal run of equal ids (must be sorted)."""
    g = np.asarray(group_ids)
    if g.size and np.any(np.diff(g) < 0):
        raise ValueError("group_ids must be non-decreasing (contiguous prompt groups)")
    starts = np.flatnonzero(np.r_[True, g[1:] != g[:-1]]) if g.size else np.zeros(0, int)
    ends = np.r_[starts[1:], g.size].astype(int)
    return list(zip(starts.tolist(), ends.tolist()))


def group_costs(group_ids, seq_offsets, rewards=None):
    """Expected sweep cost per group: tokens × (3 if the group can be active else 1)."""
    so = np.asarray(seq_offsets, dtype=np.int64)
    costs = []
    for s, e in group_spans(group_ids):
        tokens = float(so[e] - so[s])
        active = True
        if rewards is not None:
            r = np.asarray(rewards, dtype=np.float32)[s:e]
            active = (e - s) >= 2 and r.min() != r.max()
        costs.append(tokens * (COST_ACTIVE if active else COST_ELIMINATED))
    return np.array(costs)


def plan_shards(group_ids, seq_offsets, world, rewards=None, method="lpt"):
    """Returns a list (one per rank) of sorted group indices covering every group once."""
    spans = group_spans(group_ids)
    B = len(spans)
    if method == "block":
        cuts = np.linspace(0, B, world + 1).round().astype(int)
        return [list(range(cuts[r], cuts[r + 1])) for r in range(world)]
    if method != "lpt":
        raise ValueError(method)
    cost = group_costs(group_ids, seq_offsets, rewards)
    order = sorted(range(B), key=lambda g: (-cost[g], g))       # deterministic tie-break
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for g in order:
        load, r = heapq.heappop(heap)
        out[r].append(g)
        heapq.heappush(heap, (load + cost[g], r))
    return [sorted(x) for x in out]


def shard_batch(plan_rank, group_ids, seq_offsets):
    """Rank-local layout for the groups in plan_rank: (rollout indices, token indices,
    local group_ids, local seq_offsets). Token indices gather the rank's rows of the global
    per-token arrays (tokens, old_logp, mask) and logits."""
    spans = group_spans(group_ids)
    so = np.asarray(seq_offsets, dtype=np.int64)
    rollouts = np.concatenate([np.arange(*spans[g]) for g in plan_rank]) if plan_rank else \
        np.zeros(0, np.int64)
    lengths = so[rollouts + 1] - so[rollouts]
    local_so = np.zeros(len(rollouts) + 1, dtype=np.int64)
    np.cumsum(lengths, out=local_so[1:])
    tokens = np.concatenate([np.arange(so[i], so[i + 1]) for i in rollouts]) if len(rollouts) \
        else np.zeros(0, np.int64)
    local_gid = np.asarray(group_ids)[rollouts].astype(np.int32)
    return rollouts, tokens, local_gid, local_so


def imbalance(plan, group_ids, seq_offsets, rewards=None):
    """max/mean of the per-rank cost (1.0 = perfect balance)."""
    cost = group_costs(group_ids, seq_offsets, rewards)
    loads = np.array([cost[p].sum() for p in plan])
    return float(loads.max() / loads.mean()) if loads.mean() > 0 else 1.0
