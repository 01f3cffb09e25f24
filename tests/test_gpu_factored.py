"""GPU parity of the factored-gradient mode (espo_loss_fwd_factored + espo_loss_row_scale):
one sweep per row writes G_t = onehot(y_t) − softmax(λ z_t) next to the row statistics, and
scale_t · G_t must be the oracle's d loss/d z_t (tolerances as the
two-sweep path: 1e-5 relative with fp32 G, the bf16 bound with bf16 G). Also: statistics,
loss and exact fields as the two-sweep path, chunk-order independence, in-place, compact
mode, the slow path (−inf logits, lp < −69), errors and call-order checks."""
import numpy as np
import pytest
import torch

from oracle import espo_oracle as O
from paper_2512_07710_b200.espo import Espo, EspoError
from tests._instances import exact_lp, tiny_instance, workload_instance
from tests.gpu_common import (check_dlogits_bf16, check_dlogits_f32, check_exact_fields,
                              check_loss, check_token_stats, decision_aware_reference,
                              oracle_cfg, oracle_dlogits, require_cuda, run_gpu, to_dev)
from tests.test_gpu_parity import VARIANTS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return require_cuda()


@pytest.fixture(scope="module")
def c0():
    return workload_instance("C0")


def full_check(g, inst, cfg, rtol=1e-5, grad="f32", grad_loss=1.0):
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, flips = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, rtol)
    want = oracle_dlogits(ref2, inst, cfg, np.arange(inst.T), grad_loss)
    if grad == "f32":
        check_dlogits_f32(g["dlogits"], want, rtol)
    else:
        check_dlogits_bf16(g["dlogits"], want)
    return ref2


IMPLS = pytest.mark.parametrize("impl", [0, 1, 3, 6], ids=["ring20w", "cta1024", "ring20w_tmem", "roll20w"])


@IMPLS
def test_c0_factored_parity(dev, c0, impl):
    g = run_gpu(c0, dev, factored=True, factored_impl=impl)
    ref = full_check(g, c0, oracle_cfg(c0.V))
    assert g["stats"]["n_zv_groups"] == 1
    assert g["stats"]["n_clipped_tokens"] == ref.stats["n_clipped_tokens"]
    # G rows of valid tokens: onehot − p sums to 0 (up to fp32 rounding of V terms)
    v = ref.kappa >= 0
    assert np.all(np.abs(g["G"][v].sum(axis=1)) < 1e-5)
    assert not np.any(g["G"][~v])            # rows without gradient are zero-filled


def test_factored_agrees_with_two_sweep(dev, c0):
    a = run_gpu(c0, dev)
    b = run_gpu(c0, dev, factored=True)
    assert b["loss"] == pytest.approx(a["loss"], rel=1e-6)
    assert a["stats"]["n_active_tokens"] == b["stats"]["n_active_tokens"]
    np.testing.assert_allclose(b["dlogits"], a["dlogits"], rtol=2e-6,
                               atol=1e-6 * np.abs(a["dlogits"]).max())


@pytest.mark.parametrize("kw", VARIANTS[:5], ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()))
def test_factored_config_variants(dev, kw):
    inst = tiny_instance(5, V=1024, group_sizes=(4, 4, 3, 2, 1), L=40, mask_tail=8,
                         sigma_seq=0.08, logit_scale=kw.get("logit_scale", 1.0))
    g = run_gpu(inst, dev, cfgkw=kw, factored=True)
    full_check(g, inst, oracle_cfg(inst.V, **kw))


def test_factored_grad_loss_and_temperature(dev):
    inst = tiny_instance(9, V=1536, group_sizes=(4, 4), L=24, mask_tail=3, logit_scale=0.8)
    g = run_gpu(inst, dev, cfgkw=dict(logit_scale=0.8), grad_loss=-2.5, factored=True)
    full_check(g, inst, oracle_cfg(inst.V, logit_scale=0.8), grad_loss=-2.5)


@IMPLS
def test_factored_bf16_logits_bf16_G(dev, impl):
    inst = tiny_instance(8, V=4096, group_sizes=(8, 8), L=48, dtype="bf16", mask_tail=5)
    g = run_gpu(inst, dev, logits_dtype=torch.bfloat16, factored=True, factored_impl=impl)
    full_check(g, inst, oracle_cfg(inst.V), rtol=2e-3, grad="bf16")


def test_factored_bf16_logits_f32_G_exact_grade(dev):
    inst = workload_instance("C0", seed=77)
    inst.logits = __import__("espo_synth").round_to_bf16(inst.logits)
    inst.dtype = "bf16"
    g = run_gpu(inst, dev, logits_dtype=torch.bfloat16, grad_dtype=torch.float32, factored=True)
    full_check(g, inst, oracle_cfg(inst.V))


def test_factored_chunks_any_order_bitwise(dev, c0):
    a = run_gpu(c0, dev, factored=True)
    b = run_gpu(c0, dev, factored=True, chunks=[(700, c0.T), (0, 130), (130, 700)])
    assert a["loss"] == b["loss"] and a["stats"] == b["stats"]
    assert np.array_equal(a["G"], b["G"]) and np.array_equal(a["scale"], b["scale"])
    for k in a["tok"]:
        assert np.array_equal(a["tok"][k], b["tok"][k], equal_nan=True), k


@IMPLS
def test_factored_in_place_ragged_vocab(dev, impl):
    inst = tiny_instance(3, V=1002, group_sizes=(4, 4), L=33, mask_tail=4)   # V % 4 != 0
    a = run_gpu(inst, dev, ld_pad=6, factored=True, factored_impl=impl)
    full_check(a, inst, oracle_cfg(inst.V))
    b = run_gpu(inst, dev, ld_pad=6, in_place=True, factored=True, factored_impl=impl)
    assert np.array_equal(a["G"], b["G"]) and a["loss"] == b["loss"]


@IMPLS
def test_factored_bf16_ragged_vocab(dev, impl):
    inst = tiny_instance(4, V=2051, group_sizes=(4, 4), L=20, dtype="bf16")
    g = run_gpu(inst, dev, logits_dtype=torch.bfloat16, grad_dtype=torch.float32, ld_pad=5,
                factored=True, factored_impl=impl)
    full_check(g, inst, oracle_cfg(inst.V))


@IMPLS
def test_factored_compact_leaves_rows_untouched(dev, c0, impl):
    g = run_gpu(c0, dev, cfgkw=dict(zero_fill_inactive_rows=0), factored=True, factored_impl=impl)
    ref = full_check(g, c0, oracle_cfg(c0.V))
    v = ref.kappa >= 0
    assert np.all(np.isnan(g["G"][~v]))      # never written
    assert not np.any(np.isnan(g["G"][v]))


@IMPLS
def test_factored_minus_inf_logits_and_slow_path(dev, impl):
    inst = tiny_instance(3, V=1024, group_sizes=(4, 4), L=16)
    rng = np.random.default_rng(0)
    inst.logits[:, 1000:] = -np.inf
    for t in range(inst.T):
        cols = rng.choice(1000, size=20, replace=False)
        inst.logits[t, cols[cols != inst.tokens[t]]] = -np.inf
    inst.tokens = np.minimum(inst.tokens, 999)
    inst.logits[np.arange(inst.T), inst.tokens] = np.maximum(
        inst.logits[np.arange(inst.T), inst.tokens], -5.0)
    for t in range(1, inst.T, 5):              # lp ≈ −90: u_y-referenced sums overflow
        inst.logits[t, inst.tokens[t]] = np.max(inst.logits[t]) - 90.0
    import espo_synth as S
    inst.old_logp = S.drift_old_logp(exact_lp(inst.logits, inst.tokens), inst.seq_offsets, 3)
    g = run_gpu(inst, dev, factored=True, factored_impl=impl)
    ref = full_check(g, inst, oracle_cfg(inst.V))
    assert np.nanmin(ref.lp) < -85
    v = ref.kappa >= 0
    assert np.all(g["G"][v][:, 1000:] == 0)


def test_factored_nan_rows_never_read(dev, c0):
    a = run_gpu(c0, dev, factored=True)
    ref = c0.run(oracle_cfg(c0.V))
    bad = c0.logits.copy()
    for i in range(c0.R):
        if ref.zv[i]:
            bad[c0.seq_offsets[i]:c0.seq_offsets[i + 1]] = np.nan
    bad[c0.mask == 0] = np.nan
    import copy
    inst = copy.copy(c0)
    inst.logits = bad
    b = run_gpu(inst, dev, factored=True)    # get_error raises if a NaN row was read
    assert a["loss"] == b["loss"] and np.array_equal(a["G"], b["G"])


def test_factored_errors_and_call_order(dev):
    inst = tiny_instance(5, V=512, group_sizes=(4,), L=6)
    inst.logits[3, 7 if inst.tokens[3] != 7 else 8] = np.nan
    ctx = Espo(inst.V, logits_dtype=torch.float32, device=dev.index)
    z = to_dev(inst.logits, torch.float32, dev)
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    with pytest.raises(EspoError):                 # before prepare
        ctx.loss_fwd_factored(z, tok, old)
    ctx.prepare(*args, n_tokens=inst.T)
    with pytest.raises(EspoError):                 # row scale before finalize
        ctx.loss_row_scale()
    with pytest.raises(EspoError):                 # misaligned G pitch
        ctx.loss_fwd_factored(z, tok, old, grad=torch.empty((inst.T, 513), device=dev)[:, :512])
    G = ctx.loss_fwd_factored(z, tok, old)
    with pytest.raises(EspoError):                 # rows covered twice
        ctx.loss_fwd_factored(z, tok, old, grad=G)
    loss, _ = ctx.loss_finalize()
    with pytest.raises(EspoError) as e:
        ctx.get_error()
    assert e.value.code == "ESPO_ERR_NONFINITE_INPUT"
    assert np.isnan(loss.item())
    ctx.close()
    # single-pass mode admits only espo_loss_fwd_bwd
    inst = tiny_instance(5, V=512, group_sizes=(4,), L=6)
    ctx = Espo(inst.V, logits_dtype=torch.float32, device=dev.index)
    ctx.prepare(*args, n_tokens=inst.T)
    ctx.set_mask(None)
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd_factored(to_dev(inst.logits, torch.float32, dev), tok, old)
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    ctx.close()


@pytest.mark.parametrize("dt", ["bf16_f32", "f32_f32", "bf16_bf16"])
@pytest.mark.parametrize("impl", [0, 1, 3, 4, 6], ids=["ring20w", "cta1024", "ring20w_tmem", "ring10w_2cta", "roll20w"])
def test_factored_full_vocab_low_probability_targets(dev, impl, dt):
    """V = 151,936 with targets ~14 nats below the row maximum: H = ln S − ln2·W/S cancels
    ~40×, so the row sums must be accurate to ~1e-7 (fp32 per chunk, fp64 across chunks).
    Full-width rows also exercise the TMEM stash (geometry 3: pass 2 forms p from pass 1's
    2^(u − u_y) for the first chunks of a row) and, with lp ≈ −90 rows, its slow-path
    fallback; geometry 4 runs two CTAs per SM."""
    inst = tiny_instance(21, V=151936, group_sizes=(4, 4), L=6, dtype="f32" if dt == "f32_f32" else "bf16")
    rng = np.random.default_rng(5)
    for t in range(inst.T):
        if t % 2 == 0:          # a background column: z ≈ −14 against a dominant entry
            inst.tokens[t] = int(rng.integers(0, inst.V))
    for t in (3, 17, 30):       # lp ≈ −90: the u_y-referenced sums overflow
        inst.logits[t, inst.tokens[t]] = np.max(inst.logits[t]) - 90.0
    import espo_synth as S
    if dt != "f32_f32":
        inst.logits = S.round_to_bf16(inst.logits)
    lp = exact_lp(inst.logits, inst.tokens)
    assert lp.min() < -85
    inst.old_logp = S.drift_old_logp(lp, inst.seq_offsets, 21)
    ldt = torch.float32 if dt == "f32_f32" else torch.bfloat16
    gdt = torch.bfloat16 if dt == "bf16_bf16" else torch.float32
    g = run_gpu(inst, dev, logits_dtype=ldt, grad_dtype=gdt, factored=True, factored_impl=impl)
    if dt == "bf16_bf16":
        full_check(g, inst, oracle_cfg(inst.V), rtol=2e-3, grad="bf16")
    else:
        full_check(g, inst, oracle_cfg(inst.V))


def test_factored_rlzvp_mode(dev):
    """RL-ZVP: zero-variance rollouts are read by the factored sweep too; their
    token advantages are entropy differences (absolute fp32 error ≈ β·1e-6/log V), so their
    gradient rows are compared at that scale, the rest at 1e-5 (as test_rlzvp_mode)."""
    from tests.gpu_common import check_exact_fields, check_token_stats
    inst = workload_instance("C0")
    kw = dict(zv_mode=O.ZV_RLZVP, zvp_beta=0.2)
    g = run_gpu(inst, dev, cfgkw=kw, factored=True)
    cfg = oracle_cfg(inst.V, **kw)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    zv_rows = np.zeros(inst.T, bool)
    for i in range(inst.R):
        if ref.zv[i]:
            zv_rows[inst.seq_offsets[i]:inst.seq_offsets[i + 1]] = True
    assert zv_rows.any()
    want = oracle_dlogits(ref2, inst, cfg, np.arange(inst.T))
    check_dlogits_f32(g["dlogits"][~zv_rows], want[~zv_rows])
    assert np.abs(g["dlogits"][zv_rows] - want[zv_rows]).max() <= 1e-4 * np.abs(want[zv_rows]).max()


@pytest.mark.parametrize("impl", [0, 1], ids=["ring20w", "cta1024"])
def test_factored_f32_logits_bf16_G(dev, c0, impl):
    """fp32 logits, bf16 G (4 inputs → one 8-byte store per vector): the bf16 bound."""
    g = run_gpu(c0, dev, grad_dtype=torch.bfloat16, factored=True, factored_impl=impl)
    full_check(g, c0, oracle_cfg(c0.V), rtol=2e-3, grad="bf16")


def test_factored_few_rows(dev):
    """Fewer rows than CTAs (most CTAs claim nothing) and a chunk of one row."""
    inst = tiny_instance(31, V=3000, group_sizes=(2, 2), L=3, mask_tail=1)
    g = run_gpu(inst, dev, factored=True, chunks=[(0, 1), (1, inst.T)])
    full_check(g, inst, oracle_cfg(inst.V))
