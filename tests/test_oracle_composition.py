"""Pins for ESPO's defining composition (§2.4.2, Eqs. 1-3): Eq. 2 and Eq. 3
evaluated PER ENTROPY BUCKET, and the 1/|τ|·1/|y_τ| normaliser of J_ESPO.

The single-function pins (test_oracle_objective.py) check O3, O4 and O5 in isolation and the
objective at degenerate extremes (α = 0 reductions, the on-policy invariant v = 1, Σw = 1).
These pins fix the composed values on inputs where the buckets get different s_τ and ε_τ:

  - W3 (SURVEY.md:323-337): one sequence, K = 2 quantile split, α = 0.4 — J_i and every
    ∂J_i/∂lp_t under readings R2 and R1 and both advantage signs, through
    ``rollout_objective``;
  - W4 (SURVEY.md:339-350): ``espo_loss`` + ``dlogits_row`` end to end (loss and both
    dlogits rows), one group of two, singleton buckets;
  - a K = 2 quantile case worked by hand here (closed forms in the docstring), through
    ``espo_loss`` + ``dlogits_row`` end to end, built from rows that put equal logits on a
    support of m tokens (the rest −inf): such a row has p = 1/m on the support, H = ln m and
    lp = −ln m exactly, so every s_τ and ε_τ has a closed form.

Each of these fails under the three mutations that survived round 1 (ε_τ from the whole
sequence's mean entropy; s_τ from the whole sequence (GSPO); w = 1/n instead of
1/(nb·|y_τ|)); tools/mutation_check.py applies them to a scratch copy and runs the pins.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest

from oracle import espo_oracle as O

W = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_worked.json")))


# ------------------------------------------------------------------------------- W3
@pytest.mark.parametrize("case", W["W3"]["cases"], ids=lambda c: f"A{c['A']:+g}-{c['reading']}")
def test_w3_rollout_objective(case):
    w3 = W["W3"]
    tol = w3["tol"]
    cfg = O.OracleConfig(vocab=w3["V"], alpha=w3["alpha"], eps_min=w3["eps_min"],
                         n_buckets=w3["K"], split_num=w3["split"][0], split_den=w3["split"][1],
                         ratio_mode=O.RATIO_GSPO_TOKEN if case["reading"] == "R2"
                         else O.RATIO_LITERAL_OLD)
    n = len(w3["H"])
    # lp itself only enters through lp − old (both readings); any base works
    lp = np.full(n, -1.25)
    old = lp - np.array(w3["log_ratio"])
    ro = O.rollout_objective(lp, old, np.array(w3["H"]), np.full(n, case["A"]), cfg)
    assert ro["bucket"].tolist() == w3["bucket"]
    assert ro["nb"] == 2
    assert ro["theta"] == [w3["theta"]]
    for t in range(n):
        k = w3["bucket"][t]
        assert ro["s"][t] == pytest.approx(w3["s"][k], abs=tol)
        assert ro["eps"][t] == pytest.approx(w3["eps"][k], abs=tol)
    assert ro["J"] == pytest.approx(case["J"], abs=tol)
    np.testing.assert_allclose(ro["dJ_dlp"], case["dJ_dlp"], rtol=0, atol=tol)


def test_w3_scaled_advantage():
    """W3's sequence with the Â of a [1, 0] group (Â = ±½/(½ + 1e-6)): no v crosses 1 ± ε,
    so J_i and every ∂J_i/∂lp_t scale by |Â| exactly (ℓ and c are linear in Â)."""
    w3 = W["W3"]
    cfg = O.OracleConfig(vocab=w3["V"], alpha=w3["alpha"], eps_min=w3["eps_min"])
    n = len(w3["H"])
    Ahat = 0.5 / (0.5 + 1e-6)
    for A, case in ((1.0, w3["cases"][0]), (-1.0, w3["cases"][2])):
        ro = O.rollout_objective(np.zeros(n), -np.array(w3["log_ratio"]), np.array(w3["H"]),
                                 np.full(n, A * Ahat), cfg)
        assert ro["J"] == pytest.approx(Ahat * case["J"], abs=1e-11)
        np.testing.assert_allclose(ro["dJ_dlp"], Ahat * np.array(case["dJ_dlp"]), atol=1e-11)


# ------------------------------------------------------------------------------- W4
def test_w4_end_to_end():
    w4 = W["W4"]
    cfg = O.OracleConfig(vocab=w4["V"], alpha=w4["alpha"], partition=O.PARTITION_SINGLETON)
    logits = np.array(w4["logits"])
    tokens = np.array(w4["tokens"], dtype=np.int32)
    lp = [float(logits[t][tokens[t]] - np.log(np.exp(logits[t]).sum())) for t in range(2)]
    # old = lp + shift (old = [lp0 − 0.1, lp1 + 0.05]); held in fp32 like the
    # ABI's old_logp: |Δold| ≤ 2^-25·|old| ≈ 1.6e-8 moves s (and v, ℓ, g, loss, dz) by
    # ≤ 1.1·1.6e-8 → tolerance 5e-8 (W4 itself is quoted to 1e-10..1e-12)
    old = np.array([lp[0] + w4["old_shift"][0], lp[1] + w4["old_shift"][1]], dtype=np.float32)
    res = O.espo_loss(logits, tokens, old, None, np.array(w4["rewards"], dtype=np.float32),
                      np.array([0, 0]), np.array([0, 1, 2]), cfg)
    tol = 5e-8
    assert res.loss == pytest.approx(w4["loss"], abs=tol)
    for t, row in enumerate(w4["rows"]):
        assert res.s_tok[t] == pytest.approx(row["s"], abs=tol)
        if "eps" in row:
            assert res.eps_tok[t] == pytest.approx(row["eps"], abs=1e-9)
        g = -res.coef[t] / res.denom
        assert g == pytest.approx(row["g"], abs=tol)
        dz = O.dlogits_row(res, t, logits[t], int(tokens[t]), cfg)
        np.testing.assert_allclose(dz, row["dlogits"], rtol=0, atol=tol)


# ------------------------------------------------------------------------- hand-worked K=2
def _support_row(V, support, y):
    z = np.full(V, -np.inf)
    z[list(support)] = 0.0
    assert y in support
    return z


def _hand_instance():
    """Worked by hand (V = 16, α = 0.4, ε_min = 0.01, K = 2 at 4/5, reading R2, NORM_SEQ).

    Group 0 = rollouts 0, 1 with rewards [1, 0]: μ = ½, σ = ½, Â = ±½/(½ + 1e-6) = ±a.
    Group 1 = rollouts 2, 3 with rewards [1, 1]: zero variance, eliminated (rows are NaN).

    Rollout 0, support sizes m = [1, 2, 1, 16, 1] (+ one masked NaN row):
      H = [0, ln2, 0, ln16, 0]; sorted, rank ⌊4·5/5⌋ = 4 → θ = ln2; high = {t3}.
      low = {0,1,2,4}: mean H = ln2/4 → ε = 0.4·(ln2/4)/ln16 = 0.025;
                       δ = lp − old = [1/64, −1/32, 1/16, ·, 0] → s = e^{0.046875/4} = e^{0.01171875}
                       v = s ∈ (0.975, 1.025) → unclipped, w = 1/(2·4) = 1/8.
      high = {3}: ε = 0.4·ln16/ln16 = 0.4; δ = ½ → s = e^{½} > 1.4 and Â > 0 → clipped,
                  ℓ = 1.4·a, w = ½, ∂/∂lp = 0.
      J_0 = a·(4·⅛·e^{0.01171875} + ½·1.4) = a·(½e^{0.01171875} + 0.7).
    Rollout 1, m = [2, 2, 4, 4, 8]:
      H = ln2·[1, 1, 2, 2, 3]; rank 4 → θ = 2ln2; high = {t4}.
      low: mean H = 1.5·ln2 → ε = 0.4·1.5/4 = 0.15; δ = [−¼, 0, −⅛, −⅛] → s = e^{−⅛} ∈ (0.85, 1.15)
           → unclipped (Â < 0), w = ⅛.
      high: ε = 0.4·3/4 = 0.3; δ = −½ → s = e^{−½} < 0.7 and Â < 0 → clipped, ℓ = 0.7·(−a).
      J_1 = −a·(½e^{−⅛} + 0.35).
    N = 2 active rollouts; loss = −(J_0 + J_1)/2.
    dlogits row t: g_t = −c_t/N, c_t = Â·s·w (0 when clipped), dz = g·(onehot_y − 1/m on
    the support), 0 off the support and on masked / eliminated rows.
    """
    V = 16
    rows, tokens, old, mask = [], [], [], []
    rng = np.random.default_rng(7)

    def add(m, delta, ok=True):
        sup = sorted(rng.choice(V, size=m, replace=False).tolist())
        y = sup[int(rng.integers(m))]
        rows.append(_support_row(V, sup, y) if ok else np.full(V, np.nan))
        tokens.append(y)
        old.append(-math.log(m) - delta if ok else 0.0)
        mask.append(ok)

    for m, d in zip([1, 2, 1, 16, 1], [1 / 64, -1 / 32, 1 / 16, 0.5, 0.0]):
        add(m, d)
    add(1, 0.0, ok=False)                                  # masked row (never read)
    for m, d in zip([2, 2, 4, 4, 8], [-0.25, 0.0, -0.125, -0.125, -0.5]):
        add(m, d)
    for _ in range(6):                                      # eliminated group: NaN rows
        rows.append(np.full(V, np.nan))
        tokens.append(0)
        old.append(0.0)
        mask.append(True)
    seq_offsets = np.array([0, 6, 11, 14, 17])
    return dict(logits=np.array(rows), tokens=np.array(tokens, dtype=np.int32),
                old=np.array(old, dtype=np.float32), mask=np.array(mask),
                rewards=np.array([1, 0, 1, 1], dtype=np.float32),
                group_ids=np.array([0, 0, 1, 1]), seq_offsets=seq_offsets)


def test_hand_worked_k2_quantile_end_to_end():
    inst = _hand_instance()
    cfg = O.OracleConfig(vocab=16)
    res = O.espo_loss(inst["logits"], inst["tokens"], inst["old"], inst["mask"], inst["rewards"],
                      inst["group_ids"], inst["seq_offsets"], cfg)
    mp = mpmath.mp
    mp.dps = 30
    a = mpmath.mpf("0.5") / (mpmath.mpf("0.5") + mpmath.mpf("1e-6"))
    s0, s1 = mpmath.exp(mpmath.mpf("0.01171875")), mpmath.exp(mpmath.mpf("-0.125"))
    J0 = a * (s0 / 2 + mpmath.mpf("0.7"))
    J1 = -a * (s1 / 2 + mpmath.mpf("0.35"))
    # old log-probs go through fp32 (the ABI's dtype): |Δδ| ≤ 2.4e-7 → tolerance 1e-6
    tol = 1e-6
    assert res.denom == 2 and res.active.tolist() == [True, True, False, False]
    assert res.nb.tolist() == [2, 2, 0, 0]
    assert res.J_i[0] == pytest.approx(float(J0), abs=tol)
    assert res.J_i[1] == pytest.approx(float(J1), abs=tol)
    assert res.loss == pytest.approx(float(-(J0 + J1) / 2), abs=tol)
    # buckets, ratios and clips per token
    exp_bucket = [0, 0, 0, 1, 0, -1, 0, 0, 0, 0, 1] + [-1] * 6
    assert res.bucket.tolist() == exp_bucket
    exp_eps = [0.025] * 3 + [0.4, 0.025] + [None] + [0.15] * 4 + [0.3]
    exp_s = [float(s0)] * 3 + [math.exp(0.5), float(s0)] + [None] + [float(s1)] * 4 + [math.exp(-0.5)]
    for t in range(11):
        if exp_eps[t] is None:
            assert res.kappa[t] == -1
            continue
        assert res.eps_tok[t] == pytest.approx(exp_eps[t], abs=1e-12)
        assert res.s_tok[t] == pytest.approx(exp_s[t], abs=tol)
    assert res.kappa[:11].tolist() == [1, 1, 1, 0, 1, -1, 1, 1, 1, 1, 0]
    # gradient rows
    for t in range(17):
        dz = O.dlogits_row(res, t, inst["logits"][t], int(inst["tokens"][t]), cfg)
        if t in (3, 5, 10) or t >= 11:
            assert not np.any(dz), t                        # clipped / masked / eliminated
            continue
        c = (float(a * s0) if t < 5 else float(-a * s1)) / 8
        g = -c / 2
        z = inst["logits"][t]
        m = int(np.isfinite(z).sum())
        exp = np.where(np.isfinite(z), -g / m, 0.0)
        exp[int(inst["tokens"][t])] += g
        np.testing.assert_allclose(dz, exp, rtol=0, atol=tol)


# ------------------------------------------- caller-supplied selection entropies (Q4 alt.)
def test_supplied_entropies_reach_partition_and_clip():
    """Reading Q4's alternative (the rollout policy's entropies): entropies
    given by the caller replace e_t in the partition and in Eq. 3's ε_τ
    (PAPER.md:119), nowhere else. Worked by hand: two rollouts of one group, rewards (1, 0)
    ⇒ Â = ±0.5/(0.5 + 1e-6); every row uniform over V = 4 (lp = −ln 4, H = ln 4 exactly) and
    old = lp in fp32 (v = 1 to 4e-9: old is −ln 4 rounded to fp32). Computed entropies are all equal ⇒ one bucket, ∂J_i/∂lp_t = Â/5.
    Supplied e = (5, 4, 3, 2, 1): n_low = ⌊4·5/5⌋ = 4, θ = 4 (4th smallest) ⇒ high = {t0},
    low = {t1..t4}; ∂J_i/∂lp_t = Â/(2·1) for t0 and Â/(2·4) for the others;
    ε_high = 0.4·5/ln 4, ε_low = 0.4·(10/4)/ln 4; J_i = Â either way (v = 1)."""
    cfg = O.OracleConfig(vocab=4)
    z = np.zeros((10, 4))
    tok = np.array([0, 1, 2, 3, 0, 1, 2, 3, 0, 1])
    old = np.full(10, -math.log(4.0), dtype=np.float32)
    so = np.array([0, 5, 10])
    rew = np.array([1.0, 0.0], dtype=np.float32)
    gid = np.array([0, 0], dtype=np.int32)
    base = O.espo_loss(z, tok, old, None, rew, gid, so, cfg)
    A = 0.5 / (0.5 + 1e-6)
    np.testing.assert_allclose(base.coef[:5], A / 5, rtol=1e-7)
    same = O.espo_loss(z, tok, old, None, rew, gid, so, cfg, entropy=base.H)
    assert same.loss == base.loss and np.array_equal(same.coef, base.coef)
    e = np.array([5, 4, 3, 2, 1, 5, 4, 3, 2, 1], dtype=np.float32)
    got = O.espo_loss(z, tok, old, None, rew, gid, so, cfg, entropy=e)
    assert got.bucket[:5].tolist() == [1, 0, 0, 0, 0] and got.nb[0] == 2
    np.testing.assert_allclose(got.coef[:5], [A / 2] + [A / 8] * 4, rtol=1e-7)
    np.testing.assert_allclose(got.coef[5:], [-A / 2] + [-A / 8] * 4, rtol=1e-7)
    lnV = math.log(4.0)
    np.testing.assert_allclose(got.eps_tok[:5], [0.4 * 5 / lnV] + [0.4 * 2.5 / lnV] * 4,
                               rtol=1e-12)
    np.testing.assert_allclose(got.J_i, [A, -A], rtol=1e-7)
    np.testing.assert_allclose(got.H, base.H, rtol=0, atol=0)       # O2 untouched
    np.testing.assert_allclose(got.stats["mean_entropy"], 3.0, rtol=1e-12)
