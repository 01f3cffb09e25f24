"""Pins for oracle O1 (group_advantages): SPEC hand examples, closed forms, invariants.

O1 follows PAPER.md:77-79 (§2.4.1 zero-variance prompts; masking per north_star) and
PAPER.md:105-107 (GRPO-normalised advantage Â; formula SPEC.md:332-337)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import espo_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def cfg(**kw):
    return O.OracleConfig(vocab=16, **kw)


@pytest.mark.parametrize("case", GOLD["group_stats"], ids=lambda c: str(c["rewards"]))
def test_spec_group_stats(case):
    r = np.array(case["rewards"], np.float32)
    g = O.group_advantages(r, np.zeros(len(r), np.int32), cfg())
    assert bool(g["zv_group"][0]) == case["zero_variance"]
    assert g["std"][0] ** 2 == pytest.approx(case["variance"], abs=1e-15)
    if case["zero_variance"]:
        assert np.all(g["adv"] == 0.0)


@pytest.mark.parametrize("case", GOLD["advantages"], ids=lambda c: str(c["rewards"]))
def test_spec_advantages(case):
    r = np.array(case["rewards"], np.float32)
    g = O.group_advantages(r, np.zeros(len(r), np.int32), cfg())
    np.testing.assert_allclose(g["adv"], case["expected"], atol=case["abs_tol"], rtol=0)


def test_closed_forms_population_and_unbiased():
    # [1,0,0,0]: μ = 1/4, σ = sqrt(3/16) → Â_1 = (3/4)/(√3/4 + 1e-6)
    g = O.group_advantages(np.array([1, 0, 0, 0], np.float32), np.zeros(4, np.int32), cfg())
    assert g["adv"][0] == pytest.approx(0.75 / (math.sqrt(3) / 4 + 1e-6), rel=1e-15)
    assert g["adv"][1] == pytest.approx(-0.25 / (math.sqrt(3) / 4 + 1e-6), rel=1e-15)
    # unbiased: [1,0] → σ = sqrt(0.5), Â = ±0.5/(√0.5 + 1e-6)
    g = O.group_advantages(np.array([1, 0], np.float32), np.zeros(2, np.int32),
                           cfg(std_unbiased=True))
    assert g["adv"][0] == pytest.approx(0.5 / (math.sqrt(0.5) + 1e-6), rel=1e-15)
    assert g["adv"][1] == pytest.approx(-g["adv"][0], rel=1e-15)


def test_q8_float_trap_uses_exact_equality():
    """Eight rewards of 0.1f: the naive fp32 formula gives a spurious nonzero advantage;
    the exact-equality ZV test (reading Q8, "identical rewards") gives 0."""
    r = np.full(8, 0.1, np.float32)
    mean32 = np.float32(0)
    for x in r:
        mean32 = np.float32(mean32 + x)
    mean32 = np.float32(mean32 / np.float32(8))
    assert mean32 != r[0]          # the trap is real in fp32
    g = O.group_advantages(r, np.zeros(8, np.int32), cfg())
    assert g["zv_group"][0] and np.all(g["adv"] == 0.0)
    # +0 and −0 rewards are identical rewards
    g = O.group_advantages(np.array([0.0, -0.0, 0.0], np.float32), np.zeros(3, np.int32),
                           cfg())
    assert g["zv_group"][0]


def test_group_sums_to_zero_and_shift_scale_invariance():
    rng = np.random.default_rng(5)
    for _ in range(50):
        G = int(rng.integers(2, 17))
        r = (rng.integers(0, 11, size=G) / 8.0).astype(np.float32)
        if r.min() == r.max():
            continue
        gid = np.zeros(G, np.int32)
        a = O.group_advantages(r, gid, cfg(adv_eps=0.0))["adv"]
        assert abs(a.sum()) < 1e-12
        assert np.sum(a * a) == pytest.approx(G, rel=1e-12)       # unit population variance
        b = O.group_advantages((r + 3.0).astype(np.float32), gid, cfg(adv_eps=0.0))["adv"]
        np.testing.assert_allclose(b, a, rtol=1e-12, atol=1e-12)
        c = O.group_advantages((r * 4.0).astype(np.float32), gid, cfg(adv_eps=0.0))["adv"]
        np.testing.assert_allclose(c, a, rtol=1e-12, atol=1e-12)


def test_segmentation_and_counts():
    r = np.array([1, 0, 1, 1, 1, 0.3, 0.3, 0.3, 0.5], np.float32)
    gid = np.array([0, 0, 0, 4, 4, 7, 7, 7, 9], np.int32)
    g = O.group_advantages(r, gid, cfg())
    assert g["groups"] == [(0, 3), (3, 5), (5, 8), (8, 9)]
    assert g["n_groups"] == 4 and g["n_zv_groups"] == 3
    assert list(g["zv"]) == [False] * 3 + [True] * 6


def test_zv_var_eps_mode():
    r = np.array([1.0, 1.0 + 2 ** -20], np.float32)
    gid = np.zeros(2, np.int32)
    assert not O.group_advantages(r, gid, cfg())["zv_group"][0]
    assert O.group_advantages(r, gid, cfg(zv_var_eps=1e-12))["zv_group"][0]


def test_errors():
    with pytest.raises(O.OracleInputError) as e:
        O.group_advantages(np.zeros(3, np.float32), np.array([0, 1, 0], np.int32), cfg())
    assert e.value.code == "ESPO_ERR_GROUPS_NOT_CONTIGUOUS"
    with pytest.raises(O.OracleInputError) as e:
        O.group_advantages(np.array([0, np.nan], np.float32), np.zeros(2, np.int32), cfg())
    assert e.value.code == "ESPO_ERR_NONFINITE_INPUT"


# --------------------------------------------------- ZVE stage 2: reward reshaping
def test_reshape_reward_spec_examples():
    """short non-repetitive → no penalty; len = max_len → −1; a fully
    periodic "ab ab ab …" response → rep fraction from an independent scan."""
    final, lp_, rp = O.reshape_reward(0.7, list(range(20)), max_len=64)
    assert (final, lp_, rp) == (0.7, 0.0, 0.0)
    _, lp_, _ = O.reshape_reward(1.0, list(range(64)), max_len=64)
    assert lp_ == -1.0
    periodic = [1, 2] * 32                                   # 64 tokens
    _, _, rp = O.reshape_reward(1.0, periodic, max_len=1000)
    # 4-grams: positions 0 and 1 are new, the other 59 of 61 repeat → −(59/61 − 0.2)
    assert rp == pytest.approx(-(59 / 61 - 0.2), rel=1e-15)


def test_reshape_reward_length_ramp_and_brute_force_repetition():
    # buffer = ceil(100/8) = 13: ramp on [87, 100]
    for n, want in ((87, 0.0), (88, -1 / 13), (93, -6 / 13), (100, -1.0), (150, -1.0)):
        assert O.reshape_reward(0.0, list(range(n)), 100)[1] == pytest.approx(want)
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.integers(0, 40))
        toks = rng.integers(0, 3, size=n).tolist()
        _, _, rp = O.reshape_reward(0.0, toks, 10 ** 6, gamma_rep=2.0, rep_thresh=0.1)
        m = n - 3
        rep = sum(1 for p in range(max(m, 0))
                  if any(toks[q:q + 4] == toks[p:p + 4] for q in range(p)))
        frac = rep / m if m > 0 else 0.0
        assert rp == pytest.approx(-2.0 * max(0.0, frac - 0.1), abs=1e-15)


def test_reshaping_breaks_zero_variance_ties():
    """with penalties an all-correct group of different lengths is no longer
    zero-variance (reshaping "leverages negative samples")."""
    lengths = [30, 60, 95, 120]
    base = np.ones(4, np.float32)
    assert O.group_advantages(base, np.zeros(4, np.int32), cfg())["zv_group"][0]
    shaped = np.array([O.reshape_reward(1.0, list(range(n)), 100)[0] for n in lengths],
                      np.float32)
    assert not O.group_advantages(shaped, np.zeros(4, np.int32), cfg())["zv_group"][0]
