"""Property pins of the oracle's whole objective (hypothesis-generated tiny batches):
symmetries the paper's definitions imply, so that a mis-indexed or mis-normalised term in
O1–O7 breaks one of them.
- permuting prompt groups (with their rollouts and tokens) leaves loss and per-row dlogits
  unchanged (the objective is a sum over groups);
- permuting rollouts inside a group permutes their J_i and leaves the loss unchanged (Â is
  permutation-equivariant);
- adding a constant to a row's logits changes nothing (softmax shift invariance: lp, H and
  p_v are functions of differences);
- scaling all rewards by c > 0 and shifting them by a constant leaves the loss unchanged
  (GRPO normalisation; adv_eps = 0 to make it exact)."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import espo_oracle as O
from tests._instances import Instance, tiny_instance


def _inst(seed, sizes, L):
    return tiny_instance(seed, V=9, group_sizes=tuple(sizes), L=L, mask_tail=2, sigma_seq=0.1)


def _permute_groups(inst, order):
    sizes = np.bincount(inst.group_ids)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    rows, rolls, lengths = [], [], []
    for g in order:
        for i in range(starts[g], starts[g + 1]):
            rolls.append(i)
            rows.extend(range(inst.seq_offsets[i], inst.seq_offsets[i + 1]))
            lengths.append(inst.seq_offsets[i + 1] - inst.seq_offsets[i])
    rows, rolls = np.array(rows, int), np.array(rolls, int)
    gid = np.repeat(np.arange(len(order), dtype=np.int32), [sizes[g] for g in order])
    so = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    return Instance(inst.logits[rows], inst.tokens[rows], inst.old_logp[rows], inst.mask[rows],
                    inst.rewards[rolls], gid, so, inst.V), rows


@settings(max_examples=25, deadline=None)
@given(seed=st.integers(0, 10 ** 6), sizes=st.lists(st.integers(1, 4), min_size=2, max_size=4),
       L=st.integers(2, 6), data=st.data())
def test_group_permutation_invariance(seed, sizes, L, data):
    inst = _inst(seed, sizes, L)
    order = data.draw(st.permutations(list(range(len(sizes)))))
    cfg = O.OracleConfig(vocab=inst.V)
    a = inst.run(cfg)
    p, rows = _permute_groups(inst, order)
    b = p.run(cfg)
    assert b.loss == pytest.approx(a.loss, rel=1e-12, abs=1e-15)
    for t_new, t_old in enumerate(rows[:12]):
        da = O.dlogits_row(a, int(t_old), inst.logits[t_old], int(inst.tokens[t_old]), cfg)
        db = O.dlogits_row(b, t_new, p.logits[t_new], int(p.tokens[t_new]), cfg)
        np.testing.assert_allclose(db, da, rtol=1e-12, atol=1e-16)


@settings(max_examples=25, deadline=None)
@given(seed=st.integers(0, 10 ** 6), G=st.integers(2, 5), L=st.integers(2, 6), data=st.data())
def test_rollout_permutation_within_group(seed, G, L, data):
    inst = _inst(seed, [G], L)
    perm = data.draw(st.permutations(list(range(G))))
    rows = np.concatenate([np.arange(inst.seq_offsets[i], inst.seq_offsets[i + 1]) for i in perm])
    so = np.concatenate([[0], np.cumsum([inst.seq_offsets[i + 1] - inst.seq_offsets[i]
                                         for i in perm])]).astype(np.int64)
    p = Instance(inst.logits[rows], inst.tokens[rows], inst.old_logp[rows], inst.mask[rows],
                 inst.rewards[perm], inst.group_ids, so, inst.V)
    cfg = O.OracleConfig(vocab=inst.V)
    a, b = inst.run(cfg), p.run(cfg)
    assert b.loss == pytest.approx(a.loss, rel=1e-12, abs=1e-15)
    np.testing.assert_allclose(b.J_i, a.J_i[perm], rtol=1e-12, atol=1e-15)


@settings(max_examples=25, deadline=None)
@given(seed=st.integers(0, 10 ** 6), shift=st.floats(-20, 20), row=st.integers(0, 100))
def test_logit_shift_invariance(seed, shift, row):
    inst = _inst(seed, [3, 2], 4)
    t = row % inst.T
    cfg = O.OracleConfig(vocab=inst.V)
    a = inst.run(cfg)
    z = inst.logits.astype(np.float64).copy()
    z[t] += shift
    p = Instance(z, inst.tokens, inst.old_logp, inst.mask, inst.rewards, inst.group_ids,
                 inst.seq_offsets, inst.V)
    b = p.run(cfg)
    assert b.loss == pytest.approx(a.loss, rel=1e-9, abs=1e-12)
    if a.kappa[t] >= 0:
        assert b.lp[t] == pytest.approx(a.lp[t], abs=1e-11)
        assert b.H[t] == pytest.approx(a.H[t], abs=1e-11)
    np.testing.assert_allclose(O.dlogits_row(b, t, z[t], int(inst.tokens[t]), cfg),
                               O.dlogits_row(a, t, inst.logits[t], int(inst.tokens[t]), cfg),
                               rtol=1e-8, atol=1e-14)


@settings(max_examples=25, deadline=None)
@given(seed=st.integers(0, 10 ** 6), scale=st.sampled_from([0.25, 0.5, 2.0, 3.0, 6.0]),
       off=st.sampled_from([-2.0, -0.5, 0.0, 1.5, 3.0]))
def test_reward_affine_invariance(seed, scale, off):
    # dyadic scale / offset: the f32 rewards the oracle reads are exactly the affine image
    inst = _inst(seed, [3, 3, 2], 4)
    inst.rewards = np.array([1, 0, 0.5, 1, 1, 1, 0.25, 0.75], np.float32)
    cfg = O.OracleConfig(vocab=inst.V, adv_eps=0.0)
    a = inst.run(cfg)
    r2 = (inst.rewards.astype(np.float64) * scale + off)
    p = Instance(inst.logits, inst.tokens, inst.old_logp, inst.mask, r2, inst.group_ids,
                 inst.seq_offsets, inst.V)
    b = p.run(cfg)
    assert list(b.zv) == list(a.zv)
    assert b.loss == pytest.approx(a.loss, rel=1e-9, abs=1e-12)
