"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded
inputs — C0 in full, config variants, bf16 logits, chunking, both kernel variants.
Tolerances (north_star): bit-exact masks / membership / counts / advantages; 1e-5 relative
(fp32 logits) and 2e-3 (bf16 logits) on loss and gradients, P11 decision-aware protocol."""
import numpy as np
import pytest
import torch

from oracle import espo_oracle as O
from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import (check_dlogits_bf16, check_dlogits_f32, check_exact_fields,
                              check_loss, check_token_stats, decision_aware_reference,
                              oracle_cfg, oracle_dlogits, require_cuda, run_gpu)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return require_cuda()


@pytest.fixture(scope="module")
def c0():
    return workload_instance("C0")


def full_check(g, inst, cfg, rtol=1e-5, grad="f32", grad_loss=1.0, rows=None):
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, flips = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, rtol)
    rows = np.arange(inst.T) if rows is None else rows
    want = oracle_dlogits(ref2, inst, cfg, rows, grad_loss)
    if grad == "f32":
        check_dlogits_f32(g["dlogits"][rows], want, rtol)
    else:
        check_dlogits_bf16(g["dlogits"][rows], want)
    return ref2, flips


@pytest.mark.parametrize("fwd_impl,bwd_impl", [(0, 0), (1, 1)], ids=["tma", "ldg"])
def test_c0_full_parity(dev, c0, fwd_impl, bwd_impl):
    g = run_gpu(c0, dev, fwd_impl=fwd_impl, bwd_impl=bwd_impl)
    ref, _ = full_check(g, c0, oracle_cfg(c0.V))
    s = g["stats"]
    assert s["n_zv_groups"] == 1
    for k in ("mean_entropy", "mean_abs_logratio"):
        assert s[k] == pytest.approx(ref.stats[k], rel=1e-5)
    # Δ = lp − old carries lp's fp32 error (≤ 2e-6·max(1,|lp|)): bound the means by it
    lim = 2e-6 * max(1.0, float(np.nanmax(np.abs(ref.lp))))
    assert abs(s["mean_sq_logratio"] - ref.stats["mean_sq_logratio"]) <= 2 * lim * (
        ref.stats["mean_abs_logratio"] + lim) + 1e-12
    assert abs(s["mean_k3"] - ref.stats["mean_k3"]) <= 2 * lim * (
        ref.stats["mean_abs_logratio"] + lim) + 1e-12
    assert s["n_clipped_tokens"] == ref.stats["n_clipped_tokens"]
    for k in range(4):
        assert s["clip_frac"][k] == pytest.approx(ref.stats["clip_frac"][k], abs=1e-12)
        assert s["mean_ratio"][k] == pytest.approx(ref.stats["mean_ratio"][k], rel=1e-5)
        assert s["mean_eps"][k] == pytest.approx(ref.stats["mean_eps"][k], rel=1e-5)
    # advantages exported as f32 and zero for the eliminated group
    assert np.array_equal(g["adv_out"], ref.adv.astype(np.float32))


VARIANTS = [
    dict(ratio_mode=O.RATIO_LITERAL_OLD),
    dict(norm=O.NORM_TOKEN),
    dict(partition=O.PARTITION_SINGLETON),
    dict(partition=O.PARTITION_WHOLE),
    dict(n_buckets=3),
    dict(n_buckets=4, logit_scale=0.8),
    dict(std_unbiased=1, eps_min=0.0, alpha=0.9),
    dict(log_ratio_clamp=0.0, adv_eps=1e-3),
]


@pytest.mark.parametrize("kw", VARIANTS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()))
def test_config_variants(dev, kw):
    inst = tiny_instance(5, V=1024, group_sizes=(4, 4, 3, 2, 1), L=40, mask_tail=8,
                         sigma_seq=0.08, logit_scale=kw.get("logit_scale", 1.0))
    g = run_gpu(inst, dev, cfgkw=kw)
    full_check(g, inst, oracle_cfg(inst.V, **kw))


def test_grad_loss_scale(dev, c0):
    g = run_gpu(c0, dev, grad_loss=-2.5)
    full_check(g, c0, oracle_cfg(c0.V), grad_loss=-2.5)


@pytest.mark.parametrize("impl", [0, 1], ids=["tma", "ldg"])
def test_bf16_logits_f32_grads_exact_grade(dev, impl):
    """The bf16-input kernels must be exact-grade (1e-5) when they emit fp32 gradients."""
    inst = workload_instance("C0", seed=77)
    inst.logits = __import__("espo_synth").round_to_bf16(inst.logits)
    inst.dtype = "bf16"
    g = run_gpu(inst, dev, logits_dtype=torch.bfloat16, grad_dtype=torch.float32,
                fwd_impl=impl, bwd_impl=impl)
    full_check(g, inst, oracle_cfg(inst.V))


@pytest.mark.parametrize("impl", [0, 1], ids=["tma", "ldg"])
def test_bf16_logits_bf16_grads(dev, impl):
    inst = tiny_instance(8, V=4096, group_sizes=(8, 8), L=48, dtype="bf16", mask_tail=5)
    g = run_gpu(inst, dev, logits_dtype=torch.bfloat16, fwd_impl=impl, bwd_impl=impl)
    full_check(g, inst, oracle_cfg(inst.V), rtol=2e-3, grad="bf16")


def test_chunks_any_order_bitwise(dev, c0):
    a = run_gpu(c0, dev)
    T = c0.T
    cuts = [(700, T), (0, 130), (130, 700)]   # splits sequences, out of order
    b = run_gpu(c0, dev, chunks=cuts)
    assert a["loss"] == b["loss"]
    assert np.array_equal(a["dlogits"], b["dlogits"])
    assert a["stats"] == b["stats"]


def test_variants_agree(dev, c0):
    """TMA-ring and LDG variants: same per-element arithmetic, different batching of the
    fp32 partial sums — equal within fp32 summation error; the bwd sweep is elementwise and
    bitwise identical given identical row statistics."""
    a = run_gpu(c0, dev, fwd_impl=0, bwd_impl=0)
    b = run_gpu(c0, dev, fwd_impl=1, bwd_impl=1)
    assert b["loss"] == pytest.approx(a["loss"], rel=1e-6)
    np.testing.assert_allclose(b["dlogits"], a["dlogits"], rtol=2e-6,
                               atol=1e-6 * np.abs(a["dlogits"]).max())
    c = run_gpu(c0, dev, fwd_impl=0, bwd_impl=1)
    assert np.array_equal(a["dlogits"], c["dlogits"])


def test_determinism(dev, c0):
    a = run_gpu(c0, dev)
    b = run_gpu(c0, dev)
    assert a["loss"] == b["loss"] and a["stats"] == b["stats"]
    assert np.array_equal(a["dlogits"], b["dlogits"])
    for k in a["tok"]:
        assert np.array_equal(a["tok"][k], b["tok"][k], equal_nan=True), k


def test_in_place_and_padded_ld(dev):
    inst = tiny_instance(3, V=1002, group_sizes=(4, 4), L=33, mask_tail=4)   # ragged V
    a = run_gpu(inst, dev, ld_pad=6)
    full_check(a, inst, oracle_cfg(inst.V))
    b = run_gpu(inst, dev, ld_pad=6, in_place=True)
    assert np.array_equal(a["dlogits"], b["dlogits"])
    c = run_gpu(inst, dev, ld_pad=6, fwd_impl=1, bwd_impl=1, in_place=True)
    d = run_gpu(inst, dev, ld_pad=6, fwd_impl=1, bwd_impl=1)
    assert np.array_equal(c["dlogits"], d["dlogits"])


@pytest.mark.parametrize("impl", [0, 1], ids=["tma", "ldg"])
def test_bf16_ragged_vocab(dev, impl):
    inst = tiny_instance(4, V=2051, group_sizes=(4, 4), L=20, dtype="bf16")
    g = run_gpu(inst, dev, logits_dtype=torch.bfloat16, grad_dtype=torch.float32, ld_pad=5,
                fwd_impl=impl, bwd_impl=impl)
    full_check(g, inst, oracle_cfg(inst.V))


def test_rlzvp_mode(dev):
    """ZVE stage 3 as RL-ZVP: zero-variance groups are read and get entropy-
    guided token advantages. The token advantage β·s·(e_t − ē)/log V is a difference of
    entropies, so its fp32-vs-fp64 error is absolute (≈ β·1e-6/log V): coefficients and
    gradient rows of ZV rollouts are compared at that absolute scale."""
    inst = workload_instance("C0")
    kw = dict(zv_mode=O.ZV_RLZVP, zvp_beta=0.2)
    g = run_gpu(inst, dev, cfgkw=kw)
    cfg = oracle_cfg(inst.V, **kw)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    assert g["stats"]["n_zv_groups"] == 1 and ref.active.all()
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    zv_rows = np.zeros(inst.T, bool)
    for i in range(inst.R):
        if ref.zv[i]:
            zv_rows[inst.seq_offsets[i]:inst.seq_offsets[i + 1]] = True
    v = ref2.kappa >= 0
    atol_c = cfg.zvp_beta / np.log(inst.V) * 2e-5 * np.nanmax(ref2.w_tok) * 1.1
    dc = np.abs(g["tok"]["coef"].astype(np.float64) - ref2.coef)
    assert np.all(dc[v & ~zv_rows] <= 1e-5 * np.abs(ref2.coef[v & ~zv_rows]) + 1e-12)
    assert np.all(dc[v & zv_rows] <= 1e-5 * np.abs(ref2.coef[v & zv_rows]) + atol_c)
    rows = np.arange(inst.T)
    want = oracle_dlogits(ref2, inst, cfg, rows)
    check_dlogits_f32(g["dlogits"][~zv_rows], want[~zv_rows])
    # ZV rows: dz_v = −λ·(c_t/N)·(1[v=y] − p_v). The coefficient carries the absolute error
    # atol_c of the entropy difference (asserted above), p_v the usual relative 1e-5, so
    # |Δdz_v| ≤ λ·(atol_c/N)·|1[v=y] − p_v| + 2e-5·|dz_v| — element by element, per row
    lam = cfg.logit_scale
    zr = np.flatnonzero(zv_rows & v)
    x = lam * inst.logits[zr].astype(np.float64)
    p = np.exp(x - ref2.lse[zr][:, None])
    oh = np.zeros_like(p)
    oh[np.arange(len(zr)), inst.tokens[zr]] = 1.0
    lim = lam * (atol_c / ref2.denom) * np.abs(oh - p) + 2e-5 * np.abs(want[zr]) + 1e-30
    diff = np.abs(g["dlogits"][zr].astype(np.float64) - want[zr])
    assert np.all(diff <= lim), np.max(diff / lim)
    assert not np.any(g["dlogits"][zv_rows & ~v])
    # with every group mixed, RL-ZVP and masking coincide bitwise
    inst2 = tiny_instance(21, V=1024, group_sizes=(4, 4), L=24, sigma_seq=0.08)
    a = run_gpu(inst2, dev)
    b = run_gpu(inst2, dev, cfgkw=kw)
    assert a["loss"] == b["loss"] and np.array_equal(a["dlogits"], b["dlogits"])


def test_packed_f32x2_variant_is_bitwise_default(dev, c0):
    """The default fwd issues the fast-path chains as sm_100 FFMA2/FADD2 pairs; variant 8 is
    the same kernel in scalar FP32 (likewise K5's tiles: packed default, scalar bwd variant
    8): the per-lane arithmetic is unchanged, so every statistic and gradient is bitwise
    equal."""
    inst = tiny_instance(33, V=4104, group_sizes=(4, 4), L=40, dtype="bf16", mask_tail=5)
    for case, kw in ((c0, {}), (inst, {"logits_dtype": torch.bfloat16})):
        a = run_gpu(case, dev, fwd_impl=0, **kw)
        b = run_gpu(case, dev, fwd_impl=8, bwd_impl=8, **kw)
        assert a["loss"] == b["loss"] and a["stats"] == b["stats"]
        assert np.array_equal(a["dlogits"], b["dlogits"])
        for k in ("lse", "lp", "H", "q"):
            assert np.array_equal(a["tok"][k], b["tok"][k], equal_nan=True), k


@pytest.mark.parametrize("compact", [False, True], ids=["zero_fill", "compact"])
def test_tiled_list_bwd_variant_is_bitwise_default(dev, compact):
    """bwd variant 9 (tiles over the compact row lists) writes exactly the default's gradient
    (the per-element arithmetic is shared; only the work distribution differs); in compact
    mode rows without gradient stay untouched."""
    inst = tiny_instance(34, V=4104, group_sizes=(4, 4, 2), L=40, dtype="bf16", mask_tail=7,
                         rewards=[1, 0, 1, 1, 1, 1, 1, 1, 0, 1])
    kw = {"logits_dtype": torch.bfloat16, "cfgkw": {"zero_fill_inactive_rows": not compact}}
    a = run_gpu(inst, dev, **kw)
    b = run_gpu(inst, dev, bwd_impl=9, **kw)
    assert np.array_equal(a["dlogits"], b["dlogits"], equal_nan=True)
    if compact:
        untouched = ~(a["tok"]["coef"] != 0)
        assert np.isnan(b["dlogits"][untouched]).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_tiled_fwd_variant(dev, c0, dtype):
    """fwd variant 9: (row, 32 KB tile) blocks with per-tile partials merged by the combine
    kernel — a different summation order, so equal to the default within fp32 summation
    error, and to the oracle at the parity tolerances."""
    if dtype == "f32":
        inst, kw = c0, {}
    else:
        inst = tiny_instance(35, V=40000, group_sizes=(4, 4), L=24, dtype="bf16", mask_tail=5)
        kw = {"logits_dtype": torch.bfloat16, "grad_dtype": torch.float32}
    a = run_gpu(inst, dev, **kw)
    b = run_gpu(inst, dev, fwd_impl=9, **kw)
    assert b["loss"] == pytest.approx(a["loss"], rel=1e-6, abs=1e-9)
    v = a["tok"]["valid"].astype(bool)
    for k, tol in (("lse", 2e-6), ("lp", 2e-6), ("H", 1e-5)):
        x, y = a["tok"][k][v].astype(np.float64), b["tok"][k][v].astype(np.float64)
        assert np.all(np.abs(x - y) <= tol * np.maximum(1, np.abs(x))), k
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    check_exact_fields(b, ref)
    check_token_stats(b, ref)
    ref2, _ = decision_aware_reference(b, inst, ref, cfg)
    check_loss(b, ref2, 1e-5)
    check_dlogits_f32(b["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))


@pytest.mark.parametrize("impl", [0, 1, 2, 9], ids=["tile", "ldg", "tma", "tlist"])
def test_f32_logits_bf16_grads(dev, c0, impl):
    """fp32 logits with bf16 gradients (8-byte packed stores): every bwd variant within one
    bf16 rounding of the oracle, and equal to rounding the fp32-gradient run."""
    g = run_gpu(c0, dev, grad_dtype=torch.bfloat16, bwd_impl=impl)
    f = run_gpu(c0, dev, bwd_impl=impl)
    cfg = oracle_cfg(c0.V)
    ref = c0.run(cfg)
    ref2, _ = decision_aware_reference(g, c0, ref, cfg)
    check_dlogits_bf16(g["dlogits"], oracle_dlogits(ref2, c0, cfg, np.arange(c0.T)))
    want = torch.from_numpy(f["dlogits"]).to(torch.bfloat16).float().numpy()
    assert np.array_equal(g["dlogits"], want)


def test_group_permutation_invariance_gpu(dev, c0):
    """Reordering prompt groups (with their rollouts and token rows) permutes the gradient
    rows bit for bit and leaves the loss unchanged up to the fp64 order of the rollout sum —
    the per-row / per-rollout work is independent of where a group sits in the batch."""
    from tests.test_oracle_properties import _permute_groups
    a = run_gpu(c0, dev)
    p, rows = _permute_groups(c0, [3, 1, 0, 2])
    b = run_gpu(p, dev)
    assert b["loss"] == pytest.approx(a["loss"], rel=1e-12)
    assert np.array_equal(b["dlogits"], a["dlogits"][rows])


def test_compact_grid_bound_variable_lengths(dev):
    """Compact mode bounds the backward grid by the rows of non-eliminated rollouts, counted
    on the host from the layout copied at prepare: with variable lengths, empty rollouts, an
    eliminated group and chunks cutting rollouts, every row with gradient must still be
    written exactly as in full-size mode and every other row left untouched."""
    inst = tiny_instance(35, V=3000, group_sizes=(3, 4, 2, 3), dtype="bf16", mask_tail=3,
                         lengths=[17, 0, 40, 9, 9, 9, 9, 33, 1, 0, 25, 12],
                         rewards=[1, 0, 1, 1, 1, 1, 1, 0, 1, 1, 0, 0])
    chunks = [(0, 20), (20, 55), (55, 120), (120, inst.T)]
    kw = dict(logits_dtype=torch.bfloat16, chunks=chunks)
    full = run_gpu(inst, dev, **kw)
    # synchronised after prepare, so the grid bound (not the whole-chunk fallback) is used
    comp = run_gpu(inst, dev, cfgkw={"zero_fill_inactive_rows": 0}, sync_after_prepare=True, **kw)
    has_grad = full["tok"]["coef"] != 0
    assert has_grad.any() and (~has_grad).any()
    assert np.array_equal(comp["dlogits"][has_grad], full["dlogits"][has_grad])
    assert np.isnan(comp["dlogits"][~has_grad]).all()
    assert comp["loss"] == full["loss"]
