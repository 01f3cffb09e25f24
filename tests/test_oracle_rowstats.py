"""Pins for oracle O2 (row_stats): closed forms, SPEC hand examples, mpmath brute force.

O2 follows PAPER.md:111 (π_θ(y_t|·), Eq. 1 numerator) and PAPER.md:119-121 (entropy e_t
with upper bound log|V|, Eq. 3)."""
import json
import math
import os

import mpmath
import numpy as np
import pytest

from oracle import espo_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
mpmath.mp.dps = 50


def mp_eval(expr):
    return mpmath.mpf(eval(expr, {"log": mpmath.log, "exp": mpmath.exp, "sqrt": mpmath.sqrt}))


def brute(z, y, lam=1.0):
    """50-digit softmax statistics by direct definition (independent arithmetic)."""
    x = [mpmath.mpf(lam) * mpmath.mpf(float(v)) if not math.isinf(v) else None for v in z]
    e = [mpmath.e ** xi if xi is not None else mpmath.mpf(0) for xi in x]
    S = mpmath.fsum(e)
    p = [ei / S for ei in e]
    lse = mpmath.log(S)
    lp = mpmath.log(p[y])
    H = -mpmath.fsum(pi * mpmath.log(pi) for pi in p if pi > 0)
    q = mpmath.fsum(p[v] for v in range(len(p)) if v != y)
    return lse, lp, H, q


@pytest.mark.parametrize("case", GOLD["softmax"], ids=lambda c: c["cite"][:40])
def test_spec_softmax_examples(case):
    z = case["logits"] if "logits" in case else [float(mp_eval(e)) for e in case["logits_expr"]]
    lse, lp, H, q = O.row_stats(np.array(z, dtype=np.float64), case["y"])
    assert lp == pytest.approx(float(mp_eval(case["lp_expr"])), rel=1e-13, abs=1e-15)
    assert H == pytest.approx(float(mp_eval(case["H_expr"])), rel=1e-13, abs=1e-15)
    assert q == pytest.approx(float(mp_eval(case["q_expr"])), rel=1e-13)


@pytest.mark.parametrize("V", [2, 3, 16, 1024, 151936])
def test_uniform_closed_form(V):
    z = np.full(V, -3.25)
    lse, lp, H, q = O.row_stats(z, V // 3)
    assert lp == pytest.approx(-math.log(V), rel=1e-12)
    assert H == pytest.approx(math.log(V), rel=1e-12)
    assert q == pytest.approx((V - 1) / V, rel=1e-12)
    assert lse == pytest.approx(-3.25 + math.log(V), rel=1e-12)


@pytest.mark.parametrize("V", [5, 1024])
def test_spike_closed_form(V):
    """One logit +60 above V−1 equal ones: p_y = 1/(1+δ), δ = (V−1)e^{−60}."""
    z = np.zeros(V)
    z[2] = 60.0
    d = mpmath.mpf(V - 1) * mpmath.e ** -60
    lse, lp, H, q = O.row_stats(z, 2)
    assert q == pytest.approx(float(d / (1 + d)), rel=1e-12)
    assert lp == pytest.approx(float(-mpmath.log1p(d)), rel=1e-9)
    # exact: H = log(1+δ) + δ·60/(1+δ)   (p_y = 1/(1+δ); each other p = e^{-60}/(1+δ))
    H_exact = mpmath.log1p(d) + d * 60 / (1 + d)
    assert H == pytest.approx(float(H_exact), rel=1e-9)
    assert H < 1e-20
    # non-target token: lp = −60 − log(1+δ)
    _, lp0, _, q0 = O.row_stats(z, 0)
    assert lp0 == pytest.approx(-60.0 - float(mpmath.log1p(d)), rel=1e-14)
    assert 1.0 - q0 == pytest.approx(math.exp(-60.0) / (1 + float(d)), rel=1e-9)


def test_brute_force_random_rows():
    rng = np.random.default_rng(7)
    for trial in range(60):
        V = int(rng.integers(2, 17))
        z = rng.standard_normal(V) * rng.choice([0.1, 1.0, 5.0, 20.0])
        if trial % 5 == 0:
            z[rng.integers(0, V)] += 40.0        # peaked
        y = int(rng.integers(0, V))
        if trial % 7 == 0 and V > 2:
            k = (y + 1) % V
            z[k] = -np.inf                        # legal −inf entry
        lam = float(rng.choice([1.0, 0.7, 1.5]))
        got = O.row_stats(z, y, lam)
        ref = brute(z.tolist(), y, lam)
        lse, lp, H, q = (float(v) for v in ref)
        assert got[0] == pytest.approx(lse, rel=1e-13, abs=1e-13)
        assert got[1] == pytest.approx(lp, rel=1e-9, abs=1e-14)
        assert got[2] == pytest.approx(H, rel=1e-9, abs=1e-15)
        assert got[3] == pytest.approx(q, rel=1e-12, abs=1e-300)


def test_shift_invariance_and_scale():
    rng = np.random.default_rng(3)
    z = rng.standard_normal(300)
    a = O.row_stats(z, 17)
    b = O.row_stats(z + 123.5, 17)
    assert b[1] == pytest.approx(a[1], rel=1e-12)
    assert b[2] == pytest.approx(a[2], rel=1e-10)
    assert b[0] == pytest.approx(a[0] + 123.5, rel=1e-12)
    c = O.row_stats(z, 17, logit_scale=0.5)
    d = O.row_stats(0.5 * z, 17)
    assert c == pytest.approx(d, rel=1e-15)


def test_entropy_bounds():
    rng = np.random.default_rng(11)
    for V in (2, 10, 1000):
        for _ in range(20):
            z = rng.standard_normal(V) * rng.uniform(0, 10)
            _, lp, H, q = O.row_stats(z, int(rng.integers(0, V)))
            assert -1e-15 <= H <= math.log(V) + 1e-9
            assert lp <= 0.0
            assert 0.0 <= q <= 1.0


@pytest.mark.parametrize("bad,code", [(np.nan, "ESPO_ERR_NONFINITE_INPUT"),
                                      (np.inf, "ESPO_ERR_NONFINITE_INPUT")])
def test_nonfinite_errors(bad, code):
    z = np.zeros(8)
    z[5] = bad
    with pytest.raises(O.OracleInputError) as e:
        O.row_stats(z, 1)
    assert e.value.code == code


def test_token_range_and_target_minus_inf():
    with pytest.raises(O.OracleInputError) as e:
        O.row_stats(np.zeros(4), 4)
    assert e.value.code == "ESPO_ERR_TOKEN_OUT_OF_RANGE"
    z = np.zeros(4)
    z[1] = -np.inf
    with pytest.raises(O.OracleInputError):
        O.row_stats(z, 1)
