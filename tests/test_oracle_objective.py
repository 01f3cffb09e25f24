"""Pins for oracle O3–O7: partition, Eq. 2/3, surrogate, objective, gradient.

PAPER.md:103-121 (§2.4.2 ESPO, Eqs. 1-3). Pins: SPEC hand examples (tests/golden/),
order-statistic brute force, the on-policy invariant, all-ZV → 0, the P3 elimination
invariant, reductions to GSPO-token (WHOLE) and token-level PPO (SINGLETON) written here
from their textbook definitions with torch ops, torch autograd of the frozen-sg surrogate,
and fp64 central finite differences."""
import json
import math
import os

import mpmath
import numpy as np
import pytest
import torch

from oracle import espo_oracle as O
from tests._instances import tiny_instance, workload_instance

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def mp_eval(expr):
    return float(mpmath.mpf(eval(expr, {"log": mpmath.log, "exp": mpmath.exp})))


# ------------------------------------------------------------------------------- O3
@pytest.mark.parametrize("case", GOLD["partition"], ids=lambda c: c["cite"][-30:])
def test_spec_partition(case):
    cfg = O.OracleConfig(vocab=16, n_buckets=case["K"])
    b, nb = O.partition(np.array(case["H"]), cfg)
    assert nb == case["n_buckets"]
    assert int((b > 0).sum()) == case["n_high"]
    if "high_values" in case:
        assert sorted(np.array(case["H"])[b > 0].tolist()) == sorted(case["high_values"])


def test_partition_q3_edge_cases():
    cfg = O.OracleConfig(vocab=16)
    b, nb = O.partition(np.array([0.2, 0.1]), cfg)     # n_low = ⌊8/5⌋ = 1 → θ = 0.1
    assert list(b) == [1, 0] and nb == 2
    b, nb = O.partition(np.array([1, 1, 1, 2, 2.0]), cfg)  # θ = 4th smallest = 2
    assert list(b) == [0] * 5 and nb == 1
    b, nb = O.partition(np.array([0.5]), cfg)
    assert list(b) == [0] and nb == 1
    b, nb = O.partition(np.array([0.5]), O.OracleConfig(vocab=16, partition=O.PARTITION_SINGLETON))
    assert nb == 1


def test_partition_order_statistic_brute_force():
    """θ is the rank-th order statistic: #{H ≤ θ} ≥ rank > #{H < θ}; bucket membership
    depends only on the value (permutation invariant); high = strictly above θ."""
    rng = np.random.default_rng(2)
    for K in (2, 3, 4):
        cfg = O.OracleConfig(vocab=16, n_buckets=K)
        for _ in range(40):
            n = int(rng.integers(1, 40))
            H = rng.choice(rng.uniform(0, 3, size=max(1, n // 2)), size=n)  # many ties
            b, nb = O.partition(H, cfg)
            ranks = O.split_ranks(n, cfg)
            for k, rank in enumerate(ranks, start=1):
                th = np.sort(H)[rank - 1]
                assert (H <= th).sum() >= rank > (H < th).sum()
                assert np.array_equal(b >= k, H > th)
            perm = rng.permutation(n)
            b2, nb2 = O.partition(H[perm], cfg)
            assert np.array_equal(b2, b[perm]) and nb2 == nb
            assert nb == len(set(b.tolist()))
    # K=2 split counts: ⌊4n/5⌋ lowest (distinct values) stay low
    cfg = O.OracleConfig(vocab=16)
    for n in range(1, 30):
        H = rng.permutation(n).astype(float)
        b, _ = O.partition(H, cfg)
        assert (b == 0).sum() == max((4 * n) // 5, 1)


# ------------------------------------------------------------------------------- O4
@pytest.mark.parametrize("case", GOLD["eps"], ids=lambda c: c["cite"][-28:])
def test_spec_eps(case):
    cfg = O.OracleConfig(vocab=case["V"], alpha=case["alpha"], eps_min=case["eps_min"])
    H = [mp_eval(e) for e in case["H_expr"]]
    n = len(H)
    _, eps = O.bucket_ratio_clip(np.zeros(n), np.zeros(n), np.array(H), cfg)
    assert eps == pytest.approx(mp_eval(case["expected_expr"]), rel=1e-14)


@pytest.mark.parametrize("case", GOLD["seq_ratio"], ids=lambda c: c["cite"][-28:])
def test_spec_seq_ratio(case):
    lr = case.get("log_ratios") or [mp_eval(e) for e in case["log_ratios_expr"]]
    n = len(lr)
    old = np.linspace(-3, -1, n)
    s, _ = O.bucket_ratio_clip(old + np.array(lr), old, np.zeros(n), O.OracleConfig(vocab=16))
    assert s == pytest.approx(mp_eval(case["expected_expr"]), rel=1e-14)


def test_eps_monotone_bounded_and_clamp():
    cfg = O.OracleConfig(vocab=1000, alpha=0.4, eps_min=0.0)
    prev = -1
    for h in np.linspace(0, math.log(1000), 20):
        _, e = O.bucket_ratio_clip(np.zeros(3), np.zeros(3), np.full(3, h), cfg)
        assert prev <= e <= 0.4 + 1e-15
        prev = e
    s, _ = O.bucket_ratio_clip(np.array([100.0]), np.array([0.0]), np.zeros(1),
                               O.OracleConfig(vocab=16))
    assert s == pytest.approx(math.exp(20.0))       # reading Q14
    s, _ = O.bucket_ratio_clip(np.array([30.0]), np.array([0.0]), np.zeros(1),
                               O.OracleConfig(vocab=16, log_ratio_clamp=0))
    assert s == pytest.approx(math.exp(30.0))


# ------------------------------------------------------------------------------- O5
def test_surrogate_cases():
    e = 0.2
    assert O.token_surrogate(1.5, 1.0, e) == (pytest.approx(1.2), False)   # clipped above
    assert O.token_surrogate(0.5, 1.0, e) == (pytest.approx(0.5), True)    # A>0, low: pass
    assert O.token_surrogate(0.5, -1.0, e) == (pytest.approx(-0.8), False)  # A<0 clipped
    assert O.token_surrogate(1.5, -1.0, e) == (pytest.approx(-1.5), True)
    assert O.token_surrogate(1.2, 1.0, e)[1] is True                      # tie passes (Q12)
    assert O.token_surrogate(1.1, 0.0, e) == (0.0, True)
    rng = np.random.default_rng(0)
    for _ in range(200):
        v, A, eps = rng.uniform(0.3, 2), rng.normal(), rng.uniform(0.01, 0.5)
        ell, _ = O.token_surrogate(v, A, eps)
        assert ell == min(v * A, min(max(v, 1 - eps), 1 + eps) * A)
        if A > 0:
            assert ell <= (1 + eps) * A + 1e-15


@pytest.mark.parametrize("case", GOLD["token_ratio"], ids=lambda c: c["cite"][-20:])
def test_spec_token_ratio_literal(case):
    """SPEC.md:415 example under the literal reading R1: v = s_group·exp(lp − old)."""
    inst = tiny_instance(1, V=5, group_sizes=(2,), L=1)
    inst.logits[:] = 0.0
    inst.tokens[:] = 0
    lp0 = -math.log(5)
    inst.old_logp = np.array([lp0 - 0.3, lp0 - 0.3], np.float32)
    cfg = O.OracleConfig(vocab=5, ratio_mode=O.RATIO_LITERAL_OLD, partition=O.PARTITION_WHOLE,
                         log_ratio_clamp=0)
    res = inst.run(cfg)
    # s_group = exp(0.3 - rounding) for a one-token bucket; v = s·exp(lp − old) = exp(0.6)
    old = float(np.float32(lp0 - 0.3))
    assert res.v[0] == pytest.approx(math.exp(2 * (lp0 - old)), rel=1e-12)
    # with s_group pinned to 1 the value is exp(0.3)
    assert res.v[0] / res.s_tok[0] == pytest.approx(mp_eval(case["expected_expr"]), rel=1e-6)


# ------------------------------------------------------------------------------- O6
def _full_groups_instance(seed, **kw):
    return tiny_instance(seed, V=9, group_sizes=(4, 3, 2), L=6, **kw)


def test_on_policy_invariant():
    """old := lp ⇒ every v = 1 ⇒ J = Σ_active Â_i / N = 0 (advantages of each group sum
    to 0 when every rollout of a non-ZV group has ≥ 1 valid token). SPEC.md:421."""
    for seed in range(5):
        inst = _full_groups_instance(seed)
        res0 = inst.run(O.OracleConfig(vocab=inst.V))
        inst.old_logp = res0.lp.astype(np.float32)
        for mode in (O.RATIO_GSPO_TOKEN, O.RATIO_LITERAL_OLD):
            res = inst.run(O.OracleConfig(vocab=inst.V, ratio_mode=mode))
            assert abs(res.loss) < 1e-6          # old_logp is f32-rounded lp
            assert abs(res.J_sum - res.adv[res.active].sum()) < 1e-6


def test_on_policy_partial_groups():
    """With a fully-masked rollout the expectation is Σ_active Â_i / N, not 0."""
    inst = _full_groups_instance(3)
    inst.mask[inst.seq_offsets[1]:inst.seq_offsets[2]] = 0
    res0 = inst.run(O.OracleConfig(vocab=inst.V))
    inst.old_logp = res0.lp.astype(np.float32)
    res = inst.run(O.OracleConfig(vocab=inst.V))
    assert not res.active[1]
    assert res.J_sum == pytest.approx(res.adv[res.active].sum(), abs=1e-6)
    assert res.loss == pytest.approx(-res.adv[res.active].sum() / res.active.sum(), abs=1e-6)


def test_weights_sum_to_one_per_rollout():
    inst = workload_instance("C0")
    res = inst.run(O.OracleConfig(vocab=inst.V))
    for i in range(inst.R):
        if res.active[i]:
            w = res.w_tok[inst.seq_offsets[i]:inst.seq_offsets[i + 1]]
            assert np.nansum(w) == pytest.approx(1.0, rel=1e-12)
    assert res.stats["n_zv_groups"] >= 1


def test_all_zv_batch_is_exactly_zero():
    inst = tiny_instance(4, V=8, group_sizes=(3, 2, 1), rewards=[1, 1, 1, 0, 0, 0.5])
    res = inst.run(O.OracleConfig(vocab=8))
    assert res.loss == 0.0 and res.denom == 0 and not res.active.any()
    for t in range(inst.T):
        assert not np.any(O.dlogits_row(res, t, inst.logits[t], int(inst.tokens[t]),
                                        O.OracleConfig(vocab=8)))


def test_elimination_invariant_zv_rows_never_read():
    """P3: overwrite zero-variance rows and masked rows with NaN — nothing changes."""
    inst = workload_instance("C0")
    cfg = O.OracleConfig(vocab=inst.V)
    res = inst.run(cfg)
    bad = inst.logits.copy()
    for i in range(inst.R):
        if res.zv[i]:
            bad[inst.seq_offsets[i]:inst.seq_offsets[i + 1]] = np.nan
    bad[inst.mask == 0] = np.nan
    inst2 = inst
    inst2.logits = bad
    res2 = inst2.run(cfg)
    assert res2.loss == res.loss
    assert np.array_equal(res2.coef, res.coef)


def _gspo_token_reference(inst, eps0):
    """GSPO-token (one ratio for every token of a sequence), written from
    its definition with torch: s_i = exp(mean_t(lp − old)), ℓ_i = min(sÂ, clip(s)Â)."""
    J, N = 0.0, 0
    res = inst.run(O.OracleConfig(vocab=inst.V))      # only for lp, Â, active
    for i in range(inst.R):
        if not res.active[i]:
            continue
        rows = [t for t in range(inst.seq_offsets[i], inst.seq_offsets[i + 1]) if inst.mask[t]]
        lr = torch.tensor(res.lp[rows] - inst.old_logp[rows].astype(np.float64))
        s = torch.exp(lr.mean().clamp(-20, 20))
        A = float(res.adv[i])
        ell = torch.minimum(s * A, torch.clamp(s, 1 - eps0, 1 + eps0) * A)
        J += float(ell)
        N += 1
    return -J / N


def _token_ppo_reference(inst, eps0):
    """Token-level PPO/GRPO with a per-sequence token mean, textbook."""
    res = inst.run(O.OracleConfig(vocab=inst.V))
    J, N = 0.0, 0
    for i in range(inst.R):
        if not res.active[i]:
            continue
        rows = [t for t in range(inst.seq_offsets[i], inst.seq_offsets[i + 1]) if inst.mask[t]]
        r = torch.exp(torch.tensor(res.lp[rows] - inst.old_logp[rows].astype(np.float64)))
        A = float(res.adv[i])
        J += float(torch.minimum(r * A, torch.clamp(r, 1 - eps0, 1 + eps0) * A).mean())
        N += 1
    return -J / N


@pytest.mark.parametrize("seed", range(4))
def test_reduction_whole_is_gspo_token(seed):
    inst = tiny_instance(seed, V=11, group_sizes=(4, 4), L=7, sigma_seq=0.15, mask_tail=2)
    eps0 = 0.05
    cfg = O.OracleConfig(vocab=11, partition=O.PARTITION_WHOLE, alpha=0.0, eps_min=eps0)
    assert inst.run(cfg).loss == pytest.approx(_gspo_token_reference(inst, eps0), abs=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_reduction_singleton_is_token_ppo(seed):
    inst = tiny_instance(seed, V=11, group_sizes=(4, 4), L=7, sigma_seq=0.15, mask_tail=2)
    eps0 = 0.05
    cfg = O.OracleConfig(vocab=11, partition=O.PARTITION_SINGLETON, alpha=0.0, eps_min=eps0)
    assert inst.run(cfg).loss == pytest.approx(_token_ppo_reference(inst, eps0), abs=1e-12)
    # negative test: the literal reading R1 squares the token ratio, so it is NOT PPO
    cfg1 = O.OracleConfig(vocab=11, partition=O.PARTITION_SINGLETON, alpha=0.0, eps_min=eps0,
                          ratio_mode=O.RATIO_LITERAL_OLD)
    assert abs(inst.run(cfg1).loss - _token_ppo_reference(inst, eps0)) > 1e-6


def test_token_norm_identity():
    """WHOLE partition + equal lengths, no masking: 1/(N·n) weights == 1/T_active."""
    inst = tiny_instance(9, V=7, group_sizes=(3, 3), L=5)
    a = inst.run(O.OracleConfig(vocab=7, partition=O.PARTITION_WHOLE))
    b = inst.run(O.OracleConfig(vocab=7, partition=O.PARTITION_WHOLE, norm=O.NORM_TOKEN))
    assert a.loss == pytest.approx(b.loss, rel=1e-13)


# ------------------------------------------------------------------------------- O7
CONFIGS = [
    dict(),
    dict(ratio_mode=O.RATIO_LITERAL_OLD),
    dict(norm=O.NORM_TOKEN),
    dict(partition=O.PARTITION_SINGLETON),
    dict(partition=O.PARTITION_WHOLE, logit_scale=0.8),
    dict(n_buckets=3, logit_scale=1.3),
]


def _torch_frozen_loss(z, inst, res, cfg, grad_loss):
    """Frozen-sg surrogate in torch (textbook log_softmax + clamp/minimum); autograd gives
    ∂/∂z independently of the oracle's closed-form O7."""
    lp = torch.log_softmax(cfg.logit_scale * z, dim=-1)
    J = torch.zeros((), dtype=torch.float64)
    for i in range(inst.R):
        if not res.active[i]:
            continue
        for t in range(inst.seq_offsets[i], inst.seq_offsets[i + 1]):
            if res.kappa[t] < 0:
                continue
            A = float(res.adv_tok[t])
            lpt = lp[t, int(inst.tokens[t])]
            base = res.lp[t] if cfg.ratio_mode == O.RATIO_GSPO_TOKEN else float(inst.old_logp[t])
            v = res.s_tok[t] * torch.exp(lpt - base)
            e = res.eps_tok[t]
            J = J + res.w_tok[t] * torch.minimum(v * A, torch.clamp(v, 1 - e, 1 + e) * A)
    return -grad_loss * J / res.denom


@pytest.mark.parametrize("kw", CONFIGS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "default")
def test_gradient_matches_torch_autograd(kw):
    for seed in range(3):
        inst = tiny_instance(seed + 10, V=13, group_sizes=(4, 3), L=8, mask_tail=2,
                             sigma_seq=0.1, logit_scale=kw.get("logit_scale", 1.0))
        cfg = O.OracleConfig(vocab=13, **kw)
        res = inst.run(cfg)
        z = torch.tensor(inst.logits.astype(np.float64), requires_grad=True)
        loss = _torch_frozen_loss(z, inst, res, cfg, grad_loss=0.7)
        assert float(loss) == pytest.approx(res.loss * 0.7, rel=1e-12, abs=1e-15)
        loss.backward()
        for t in range(inst.T):
            dz = O.dlogits_row(res, t, inst.logits[t], int(inst.tokens[t]), cfg, grad_loss=0.7)
            np.testing.assert_allclose(dz, z.grad[t].numpy(), rtol=1e-10, atol=1e-14)
            assert abs(dz.sum()) < 1e-14          # softmax-gradient identity


def test_gradient_matches_finite_differences():
    """fp64 central FD (h = 1e-6) of the frozen-sg surrogate, ≥ 20 random configurations,
    skipping tokens whose ratio is within 10h of a clip kink."""
    h = 1e-6
    checked = 0
    for seed in range(24):
        rng = np.random.default_rng(seed)
        kw = CONFIGS[seed % len(CONFIGS)]
        inst = tiny_instance(seed + 50, V=6, group_sizes=(3, 2), L=4, sigma_seq=0.1,
                             logit_scale=kw.get("logit_scale", 1.0))
        cfg = O.OracleConfig(vocab=6, **kw)
        res = inst.run(cfg)
        if res.denom == 0:
            continue
        for _ in range(4):
            t = int(rng.integers(0, inst.T))
            if res.kappa[t] < 0:
                continue
            vv, e = res.v[t], res.eps_tok[t]
            if min(abs(vv - (1 + e)), abs(vv - (1 - e))) < 10 * h * max(1, vv) * 10:
                continue
            col = int(rng.integers(0, inst.V))
            zp = inst.logits.astype(np.float64).copy()
            zm = zp.copy()
            zp[t, col] += h
            zm[t, col] -= h
            fp = O.frozen_surrogate_loss(zp, res, inst.tokens, inst.old_logp, inst.seq_offsets, cfg)
            fm = O.frozen_surrogate_loss(zm, res, inst.tokens, inst.old_logp, inst.seq_offsets, cfg)
            fd = (fp - fm) / (2 * h)
            dz = O.dlogits_row(res, t, inst.logits[t], int(inst.tokens[t]), cfg)[col]
            assert fd == pytest.approx(dz, rel=1e-6, abs=1e-9)
            checked += 1
    assert checked >= 20


def test_gradient_sign():
    """Raising the sampled token's logit raises π_θ(y): with Â > 0 in the unclipped region
    the loss must fall (dz_y < 0); with Â < 0 it must rise."""
    inst = tiny_instance(21, V=7, group_sizes=(2,), L=3, sigma_seq=0.0, sigma_tok=0.0,
                         rewards=[1, 0])
    cfg = O.OracleConfig(vocab=7)
    res = inst.run(cfg)
    for t in range(inst.T):
        y = int(inst.tokens[t])
        dz = O.dlogits_row(res, t, inst.logits[t], y, cfg)
        A = res.adv[0] if t < inst.seq_offsets[1] else res.adv[1]
        assert np.sign(dz[y]) == -np.sign(A)


# ------------------------------------------------------------------- RL-ZVP (ZVE stage 3)
def test_zvp_spec_examples():
    """SPEC.md:342 examples and SPEC.md:354 invariants for the RL-ZVP instantiation of the
    cited method."""
    cfg = O.OracleConfig(vocab=1000)
    a = O.zvp_token_advantages(np.full(7, 1.3), 0.0, cfg)          # all entropies equal
    assert np.all(a == 0.0)
    H = np.array([0.01, 0.02, 3.5, 0.01])                         # one high-entropy token
    a = O.zvp_token_advantages(H, 0.0, cfg)                       # all-fail group (r < 0.5)
    assert a[2] > 0 and np.all(a[[0, 1, 3]] < 0)
    a1 = O.zvp_token_advantages(H, 1.0, cfg)                      # all-pass: sign flips
    np.testing.assert_allclose(a1, -a, rtol=0, atol=0)
    rng = np.random.default_rng(4)
    for _ in range(100):
        H = rng.uniform(0, np.log(1000), size=int(rng.integers(1, 50)))
        a = O.zvp_token_advantages(H, float(rng.uniform()), cfg)
        assert np.all(np.abs(a) <= cfg.zvp_beta + 1e-15)
        assert abs(a.mean()) < 1e-9


def test_zvp_without_zv_groups_equals_mask_mode():
    inst = tiny_instance(12, V=64, group_sizes=(4, 3), L=6, sigma_seq=0.1)
    a = inst.run(O.OracleConfig(vocab=64))
    b = inst.run(O.OracleConfig(vocab=64, zv_mode=O.ZV_RLZVP))
    assert a.loss == b.loss and np.array_equal(a.coef, b.coef)


def test_zvp_reads_zv_rows_and_bounds_advantages():
    inst = tiny_instance(13, V=64, group_sizes=(4, 3, 2, 1), L=7, mask_tail=2,
                         rewards=[1, 0, 1, 0, 1, 1, 1, 0, 0, 0.3])
    m = inst.run(O.OracleConfig(vocab=64))
    z = inst.run(O.OracleConfig(vocab=64, zv_mode=O.ZV_RLZVP))
    assert m.active.sum() == 4 and z.active.sum() == inst.R
    zv_rows = np.concatenate([np.arange(inst.seq_offsets[i], inst.seq_offsets[i + 1])
                              for i in range(inst.R) if z.zv[i]])
    v = z.kappa[zv_rows] >= 0
    assert np.all(np.abs(z.adv_tok[zv_rows][v]) <= 0.05 + 1e-15)
    # non-ZV rollouts keep their GRPO advantage and bucket machinery; N grows
    assert z.denom == inst.R and m.denom == 4
    np.testing.assert_allclose(z.J_i[:4], m.J_i[:4], rtol=1e-14)


def test_zvp_gradient_matches_torch_autograd():
    for seed in range(3):
        inst = tiny_instance(seed + 40, V=13, group_sizes=(3, 3, 2), L=8, mask_tail=2,
                             sigma_seq=0.1, rewards=[1, 0, 1, 1, 1, 1, 0, 0])
        cfg = O.OracleConfig(vocab=13, zv_mode=O.ZV_RLZVP, zvp_beta=0.3)
        res = inst.run(cfg)
        z = torch.tensor(inst.logits.astype(np.float64), requires_grad=True)
        loss = _torch_frozen_loss(z, inst, res, cfg, grad_loss=1.0)
        assert float(loss) == pytest.approx(res.loss, rel=1e-12, abs=1e-15)
        loss.backward()
        for t in range(inst.T):
            dz = O.dlogits_row(res, t, inst.logits[t], int(inst.tokens[t]), cfg)
            np.testing.assert_allclose(dz, z.grad[t].numpy(), rtol=1e-10, atol=1e-14)


# --------------------------------------------------- O9: LM-head gradients (§8(f) row 1)
def _lmhead_instance(seed, V=11, d=5, kw=None):
    rng = np.random.default_rng(seed)
    base = tiny_instance(seed + 300, V=V, group_sizes=(3, 2), L=6, mask_tail=2, sigma_seq=0.1,
                         logit_scale=(kw or {}).get("logit_scale", 1.0))
    h = rng.standard_normal((base.T, d))
    W = rng.standard_normal((V, d))
    z = h @ W.T
    lp = np.array([O.row_stats(z[t], int(base.tokens[t]), (kw or {}).get("logit_scale", 1.0))[1]
                   for t in range(base.T)])
    old = (lp + rng.normal(0, 0.05, size=base.T)).astype(np.float32)
    inst = type(base)(z, base.tokens, old, base.mask, base.rewards, base.group_ids,
                      base.seq_offsets, V)
    return inst, h, W


@pytest.mark.parametrize("kw", CONFIGS[:3] + [dict(logit_scale=0.7)],
                         ids=["default", "literal", "token_norm", "lambda0.7"])
def test_lmhead_grads_match_torch_autograd(kw):
    """O9 against autograd of the torch frozen surrogate through z = h·Wᵀ (a transposed or
    swapped operand in O9 fails: h and W have different shapes)."""
    inst, h, W = _lmhead_instance(3, kw=kw)
    cfg = O.OracleConfig(vocab=inst.V, **kw)
    res = inst.run(cfg)
    ht = torch.tensor(h, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    loss = _torch_frozen_loss(ht @ Wt.T, inst, res, cfg, grad_loss=1.3)
    loss.backward()
    dz, dh, dW = O.lmhead_grads(res, h, W, inst.tokens, cfg, grad_loss=1.3)
    assert dz.shape == (inst.T, inst.V) and dh.shape == h.shape and dW.shape == W.shape
    np.testing.assert_allclose(dh, ht.grad.numpy(), rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(dW, Wt.grad.numpy(), rtol=1e-10, atol=1e-14)
    assert np.abs(dh).max() > 0 and np.abs(dW).max() > 0


def test_lmhead_grads_match_finite_differences():
    """fp64 central differences of the frozen surrogate F(h·Wᵀ) in single h and W entries."""
    inst, h, W = _lmhead_instance(8)
    cfg = O.OracleConfig(vocab=inst.V)
    res = inst.run(cfg)
    _, dh, dW = O.lmhead_grads(res, h, W, inst.tokens, cfg)
    F = lambda hh, WW: O.frozen_surrogate_loss(hh @ WW.T, res, inst.tokens, inst.old_logp,
                                               inst.seq_offsets, cfg)
    eps = 1e-6
    rng = np.random.default_rng(0)
    for _ in range(12):
        t, j = int(rng.integers(0, h.shape[0])), int(rng.integers(0, h.shape[1]))
        hp, hm = h.copy(), h.copy()
        hp[t, j] += eps
        hm[t, j] -= eps
        assert (F(hp, W) - F(hm, W)) / (2 * eps) == pytest.approx(dh[t, j], rel=1e-5, abs=1e-9)
        v = int(rng.integers(0, W.shape[0]))
        Wp, Wm = W.copy(), W.copy()
        Wp[v, j] += eps
        Wm[v, j] -= eps
        assert (F(h, Wp) - F(h, Wm)) / (2 * eps) == pytest.approx(dW[v, j], rel=1e-5, abs=1e-9)


def test_mismatch_statistics_closed_forms():
    """Train/inference mismatch stats: with old = lp − c on every token,
    mean|Δ| = |c|, mean Δ² = c² and the k3 KL estimate = e^c − 1 − c (up to the f32 rounding
    of old_logp); on-policy all three vanish; k3 ≥ 0 always."""
    inst = _full_groups_instance(2)
    res0 = inst.run(O.OracleConfig(vocab=inst.V))
    for c in (0.0, 0.03, -0.2, 0.7):
        inst.old_logp = (res0.lp - c).astype(np.float32)
        st = inst.run(O.OracleConfig(vocab=inst.V)).stats
        assert st["mean_abs_logratio"] == pytest.approx(abs(c), abs=2e-6)
        assert st["mean_sq_logratio"] == pytest.approx(c * c, abs=4e-6)
        assert st["mean_k3"] == pytest.approx(math.expm1(c) - c, abs=4e-6)
    rng = np.random.default_rng(0)
    inst.old_logp = (res0.lp + rng.normal(0, 0.5, size=len(res0.lp))).astype(np.float32)
    st = inst.run(O.OracleConfig(vocab=inst.V)).stats
    assert st["mean_k3"] > 0 and st["mean_sq_logratio"] >= st["mean_abs_logratio"] ** 2
