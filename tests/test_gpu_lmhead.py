"""Fused LM head + ESPO forward on tcgen05: the row statistics computed
from hidden states and the LM-head matrix without materialising logits must equal those of
the logits path on the same fp32 logits (h·Wᵀ with fp32 accumulation), and the oracle's on
fp64 logits within the fp32-accumulation error of the GEMM."""
import numpy as np
import pytest
import torch

import espo_synth as S
from oracle import espo_oracle as O
from paper_2512_07710_b200.espo import Espo, stats_to_dict
from tests.gpu_common import oracle_cfg, require_cuda, to_dev

pytestmark = pytest.mark.gpu


def make_case(seed, n_groups, G, L, V, d, zv_group=None, lam=1.0):
    rng = np.random.default_rng(seed)
    R = n_groups * G
    T = R * L
    h = (rng.standard_normal((T, d)) / np.sqrt(d) * 3).astype(np.float32)
    W = rng.standard_normal((V, d)).astype(np.float32)
    W[rng.integers(0, V, size=V // 50)] *= 3.0                  # a few strong tokens
    h, W = S.round_to_bf16(h), S.round_to_bf16(W)
    z64 = h.astype(np.float64) @ W.astype(np.float64).T
    tokens = S.sample_tokens_gumbel(z64.astype(np.float32), seed, logit_scale=lam)
    group_ids = np.repeat(np.arange(n_groups, dtype=np.int32), G)
    so = np.arange(R + 1, dtype=np.int64) * L
    rewards = (rng.uniform(size=R) < 0.5).astype(np.float32)
    for g in range(n_groups):
        rewards[g * G] = 1.0
        rewards[g * G + 1] = 0.0
    if zv_group is not None:
        rewards[zv_group * G:(zv_group + 1) * G] = 1.0
    lp = np.array([O.row_stats(z64[t], int(tokens[t]), lam)[1] for t in range(T)])
    old = S.drift_old_logp(lp, so, seed)
    mask = np.ones(T, np.uint8)
    mask[L - 5:L] = 0
    return dict(h=h, W=W, z64=z64, tokens=tokens, group_ids=group_ids, so=so, rewards=rewards,
                old=old, mask=mask, T=T, R=R)


# ESPO_OPT_LMHEAD_IMPL 0 (GEMM core; "gemm_mc": 4-CTA clusters with A multicast) / 1 with one
# CTA / pairs
KERNELS = ["gemm", "gemm_mc", "1cta", "2cta"]


def set_kernel(ctx, kern):
    from paper_2512_07710_b200.espo import OPT_LMHEAD_2CTA, OPT_LMHEAD_IMPL, OPT_LMHEAD_RASTER
    ctx.set_option(OPT_LMHEAD_IMPL, 0 if kern.startswith("gemm") else 1)
    ctx.set_option(OPT_LMHEAD_2CTA, int(kern == "2cta"))
    ctx.set_option(OPT_LMHEAD_RASTER, (1 << 25) if kern == "gemm_mc" else 0)


def run_path(case, dev, fused, V, kern="gemm"):
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
    set_kernel(ctx, kern)
    tok = to_dev(case["tokens"], torch.int32, dev)
    old = to_dev(case["old"], torch.float32, dev)
    mask = to_dev(case["mask"], torch.uint8, dev)
    ctx.prepare(to_dev(case["rewards"], torch.float32, dev), to_dev(case["group_ids"], torch.int32, dev),
                to_dev(case["so"], torch.int64, dev), n_tokens=case["T"])
    h = to_dev(case["h"], torch.bfloat16, dev)
    W = to_dev(case["W"], torch.bfloat16, dev)
    if fused:
        half = case["T"] // 2 + 37                   # two chunks, the first not a multiple of 128
        ctx.lmhead_fwd(h[:half], W, tok[:half], old[:half], mask[:half], row_begin=0)
        ctx.lmhead_fwd(h[half:], W, tok[half:], old[half:], mask[half:], row_begin=half)
    else:
        ld = (V + 3) // 4 * 4
        z = torch.zeros((case["T"], ld), dtype=torch.float32, device=dev)
        z[:, :V] = h.float() @ W.float().T
        ctx.loss_fwd(z, tok, old, mask)
    loss, stats = ctx.loss_finalize()
    ctx.get_error()
    out = dict(loss=float(loss.item()), stats=stats_to_dict(stats),
               tok={k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()})
    ctx.close()
    return out


@pytest.mark.parametrize("kern", KERNELS)
@pytest.mark.parametrize("shape", [(4, 4, 40, 1000, 200), (2, 8, 64, 4099, 512),
                                   (3, 8, 48, 5003, 256)],
                         ids=["V1000_d200", "V4099_d512", "V5003_d256_zv_block"])
def test_lmhead_fwd_matches_logits_path(shape, kern):
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = require_cuda()
    ng, G, L, V, d = shape
    case = make_case(5, ng, G, L, V, d, zv_group=1)
    f = run_path(case, dev, True, V, kern)
    u = run_path(case, dev, False, V)
    v = u["tok"]["valid"].astype(bool)
    assert np.array_equal(f["tok"]["valid"], u["tok"]["valid"])
    assert f["stats"]["n_active_tokens"] == u["stats"]["n_active_tokens"]
    # both paths accumulate h·Wᵀ in fp32 (different orders): per-row logit error bound
    hb = np.abs(case["h"].astype(np.float64)) @ np.abs(case["W"].astype(np.float64)).T
    bound = d * 2.0 ** -24 * hb.max(axis=1)[v]
    for k, tol, kb in (("lse", 2e-6, 2), ("lp", 2e-6, 4), ("H", 1e-5, 8)):
        a, b = f["tok"][k][v].astype(np.float64), u["tok"][k][v].astype(np.float64)
        lim = tol * np.maximum(1, np.abs(b)) + kb * bound
        assert np.all(np.abs(a - b) <= lim), (k, np.max(np.abs(a - b) / lim))
    assert f["loss"] == pytest.approx(u["loss"], rel=1e-3, abs=1e-6)
    # oracle on fp64 logits: within the fused GEMM's fp32-accumulation error
    cfg = oracle_cfg(V)
    ref = O.espo_loss(case["z64"], case["tokens"], case["old"], case["mask"], case["rewards"],
                      case["group_ids"], case["so"], cfg)
    assert np.array_equal(ref.kappa >= 0, v)
    for k, tol, kb in (("lse", 2e-6, 1), ("lp", 2e-6, 2), ("H", 1e-5, 4)):
        diff = np.abs(f["tok"][k][v].astype(np.float64) - getattr(ref, k)[v])
        lim = tol * np.maximum(1, np.abs(getattr(ref, k)[v])) + kb * bound
        assert np.all(diff <= lim), (k, np.max(diff / lim))
    assert f["stats"]["n_zv_groups"] == ref.stats["n_zv_groups"] == 1


@pytest.mark.parametrize("kern", KERNELS)
@pytest.mark.parametrize("shape,sub,dh_bf16,lam", [((4, 4, 40, 1000, 200), 0, False, 1.0),
                                                   ((2, 8, 64, 4099, 512), 256, True, 1.0),
                                                   ((3, 4, 32, 2000, 128), 128, False, 0.8)],
                         ids=["V1000_d200", "V4099_d512_sub256_bf16", "V2000_d128_lambda0.8"])
def test_lmhead_bwd_matches_oracle(shape, sub, dh_bf16, kern, lam):
    """espo_lmhead_bwd (tcgen05 recompute → bf16 dz → dh = dz·W, dW += dzᵀ·h) against O9 on
    fp64 logits, with the GPU's bucket / clip decisions injected where they flipped. Bound:
    dz is rounded to bf16 (2^-9) after an fp32 recompute whose logit error is ≤ the GEMM
    bound b_t; the contractions accumulate in fp32 over V (resp. n) terms."""
    from paper_2512_07710_b200.espo import OPT_LMHEAD_BWD_ROWS
    from tests._instances import Instance
    from tests.gpu_common import decision_aware_reference
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = require_cuda()
    ng, G, L, V, d = shape
    case = make_case(7, ng, G, L, V, d, zv_group=0, lam=lam)
    T = case["T"]
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index, logit_scale=lam)
    if sub:
        ctx.set_option(OPT_LMHEAD_BWD_ROWS, sub)
    set_kernel(ctx, kern)
    tok = to_dev(case["tokens"], torch.int32, dev)
    old = to_dev(case["old"], torch.float32, dev)
    mask = to_dev(case["mask"], torch.uint8, dev)
    ctx.prepare(to_dev(case["rewards"], torch.float32, dev), to_dev(case["group_ids"], torch.int32, dev),
                to_dev(case["so"], torch.int64, dev), n_tokens=T)
    h = to_dev(case["h"], torch.bfloat16, dev)
    W = to_dev(case["W"], torch.bfloat16, dev)
    ctx.lmhead_fwd(h, W, tok, old, mask)
    ctx.loss_finalize()
    gl = torch.tensor([0.75], dtype=torch.float32, device=dev)
    dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
    dh = torch.full((T, d), float("nan"), dtype=torch.bfloat16 if dh_bf16 else torch.float32,
                    device=dev)
    cut = T // 3 + 5                                   # two backward chunks, dW accumulates
    ctx.lmhead_bwd(h[:cut], W, dh[:cut], dW, row_begin=0, grad_loss=gl)
    ctx.lmhead_bwd(h[cut:], W, dh[cut:], dW, row_begin=cut, grad_loss=gl)
    ctx.get_error()
    g = dict(tok={k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()})
    ctx.close()
    inst = Instance(case["z64"], case["tokens"], case["old"], case["mask"], case["rewards"],
                    case["group_ids"], case["so"], V)
    cfg = oracle_cfg(V, logit_scale=lam)
    ref = inst.run(cfg)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    dz, dh_ref, dW_ref = O.lmhead_grads(ref2, case["h"], case["W"], case["tokens"], cfg, 0.75)
    hb = np.abs(case["h"].astype(np.float64)) @ np.abs(case["W"].astype(np.float64)).T
    b_t = d * 2.0 ** -24 * hb.max(axis=1)                    # per-row logit error bound
    adz = np.abs(dz) * (2.0 ** -9 + 4 * b_t[:, None] + 1e-6)  # per-element dz error bound
    Wa, ha = np.abs(case["W"].astype(np.float64)), np.abs(case["h"].astype(np.float64))
    lim_dh = adz @ Wa + V * 2.0 ** -24 * (np.abs(dz) @ Wa) + 1e-30
    lim_dW = adz.T @ ha + T * 2.0 ** -24 * (np.abs(dz).T @ ha) + 1e-30
    got_dh = dh.float().cpu().numpy().astype(np.float64)
    got_dW = dW.cpu().numpy().astype(np.float64)
    if dh_bf16:
        lim_dh = lim_dh + 2.0 ** -9 * np.abs(dh_ref) * 1.01
    assert np.all(np.abs(got_dh - dh_ref) <= lim_dh), np.max(np.abs(got_dh - dh_ref) / lim_dh)
    assert np.all(np.abs(got_dW - dW_ref) <= lim_dW), np.max(np.abs(got_dW - dW_ref) / lim_dW)
    # norm-wise: 2e-3 (the north_star bf16 tolerance); a bf16 dh adds its own output rounding
    for got, want, tol in ((got_dh, dh_ref, 2e-3 + (2.0 ** -9 if dh_bf16 else 0.0)),
                           (got_dW, dW_ref, 2e-3)):
        assert np.linalg.norm(got - want) <= tol * np.linalg.norm(want)
    # rows of the zero-variance group and masked rows carry no gradient
    zrows = ref2.kappa < 0
    assert zrows.any() and np.all(got_dh[zrows] == 0)


def test_lmhead_kernels_agree():
    """The GEMM-core kernels (pair 256 × 512 tiles, per-tile partials) and the dedicated
    one-CTA / CTA-pair kernels compute the same dot products in the same K order: statistics
    and the backward's dh/dW agree (within fp32 rounding of the partial merges)."""
    dev = require_cuda()
    V, d = 3000, 384
    case = make_case(9, 3, 4, 48, V, d, zv_group=2)
    outs = []
    for kern in KERNELS:
        ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
        set_kernel(ctx, kern)
        tok = to_dev(case["tokens"], torch.int32, dev)
        ctx.prepare(to_dev(case["rewards"], torch.float32, dev),
                    to_dev(case["group_ids"], torch.int32, dev), to_dev(case["so"], torch.int64, dev),
                    n_tokens=case["T"])
        h = to_dev(case["h"], torch.bfloat16, dev)
        W = to_dev(case["W"], torch.bfloat16, dev)
        ctx.lmhead_fwd(h, W, tok, to_dev(case["old"], torch.float32, dev),
                       to_dev(case["mask"], torch.uint8, dev))
        loss, _ = ctx.loss_finalize()
        dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
        dh, _ = ctx.lmhead_bwd(h, W, None, dW)
        ctx.get_error()
        t = {k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()}
        outs.append((float(loss.item()), t, dh.cpu().numpy(), dW.cpu().numpy()))
        ctx.close()
    (l0, t0, h0, w0) = outs[KERNELS.index("1cta")]
    for (l1, t1, h1, w1) in outs:
        v = t0["valid"].astype(bool)
        assert np.array_equal(v, t1["valid"].astype(bool))
        # each kernel is within the K2 bounds of the oracle (2e-6 / 2e-6 / 1e-5 relative to
        # max(1, |x|)); two of them therefore within twice that of each other
        for k, tol in (("lse", 4e-6), ("lp", 4e-6), ("H", 2e-5)):
            a, b = t1[k][v].astype(np.float64), t0[k][v].astype(np.float64)
            assert np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b))), k
        assert l1 == pytest.approx(l0, rel=1e-5, abs=1e-8)
        np.testing.assert_allclose(h1, h0, rtol=1e-3, atol=1e-6 * np.abs(h0).max())
        np.testing.assert_allclose(w1, w0, rtol=1e-3, atol=1e-6 * np.abs(w0).max())


def test_lmhead_errors_and_state():
    """espo_lmhead_bwd before finalize → BAD_STATE; fused LM head on a vocabulary-sharded
    context → UNSUPPORTED; misaligned hidden pitch → ALIGNMENT."""
    from paper_2512_07710_b200.espo import EspoError
    dev = require_cuda()
    V, d, T = 512, 64, 32
    h = torch.zeros((T, d), dtype=torch.bfloat16, device=dev)
    W = torch.zeros((V, d), dtype=torch.bfloat16, device=dev)
    tok = torch.zeros(T, dtype=torch.int32, device=dev)
    old = torch.zeros(T, dtype=torch.float32, device=dev)
    args = (torch.tensor([1.0, 0.0], device=dev), torch.zeros(2, dtype=torch.int32, device=dev),
            torch.tensor([0, 16, 32], dtype=torch.int64, device=dev))
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
    ctx.prepare(*args, n_tokens=T)
    with pytest.raises(EspoError) as e:
        ctx.lmhead_bwd(h, W)
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    hp = torch.zeros((T, d + 3), dtype=torch.bfloat16, device=dev)[:, :d]   # 134-byte pitch
    with pytest.raises(EspoError) as e:
        ctx.lmhead_fwd(hp, W, tok, old)
    assert e.value.code == "ESPO_ERR_ALIGNMENT"
    ctx.lmhead_fwd(h, W, tok, old)
    ctx.loss_finalize()
    dh, _ = ctx.lmhead_bwd(h, W)
    ctx.get_error()
    assert torch.isfinite(dh).all()
    ctx.close()
    sh = Espo(V, logits_dtype=torch.float32, device=dev.index, vocab_shard=(0, 256))
    sh.prepare(*args, n_tokens=T)
    with pytest.raises(EspoError) as e:
        sh.lmhead_fwd(h, W[:256], tok, old)
    assert e.value.code == "ESPO_ERR_UNSUPPORTED"
    sh.close()


@pytest.mark.parametrize("native", [0, 2, 3, 4, 5, 6, 7],
                         ids=["pair_default", "1cta", "pair256", "pair512", "mcast", "mcast_dh",
                              "dw256"])
@pytest.mark.parametrize("shape", [(3, 4, 50, 20000, 1000), (2, 4, 130, 5000, 2048)],
                         ids=["V20000_d1000_ntail", "V5000_d2048"])
def test_lmhead_bwd_native_gemm_equals_cublas(shape, native):
    """The library's tcgen05 GEMMs (dh: dz K-major × W MN-major; dW: dz MN-major × h MN-major)
    against cuBLAS on the same bf16 dz tile (ESPO_OPT_LMHEAD_BWD_GEMM 0 vs 1): both accumulate
    the same bf16 products in fp32, only the summation order differs — within
    K·2^-24·Σ|terms| elementwise. Covers N tails (d = 1000 is not a multiple of 256), row
    tails, several sub-chunks and dW accumulation across them."""
    from paper_2512_07710_b200.espo import (OPT_LMHEAD_BWD_GEMM, OPT_LMHEAD_BWD_ROWS,
                                            OPT_LMHEAD_COMPACT)
    dev = require_cuda()
    ng, G, L, V, d = shape
    case = make_case(13, ng, G, L, V, d, zv_group=0)
    T = case["T"]
    outs = []
    for impl in (native, 1):
        ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
        ctx.set_option(OPT_LMHEAD_BWD_GEMM, impl)
        ctx.set_option(OPT_LMHEAD_COMPACT, 0)     # same sub-chunks on both sides (cuBLAS: all rows)
        ctx.set_option(OPT_LMHEAD_BWD_ROWS, 256)
        tok = to_dev(case["tokens"], torch.int32, dev)
        ctx.prepare(to_dev(case["rewards"], torch.float32, dev),
                    to_dev(case["group_ids"], torch.int32, dev), to_dev(case["so"], torch.int64, dev),
                    n_tokens=T)
        h = to_dev(case["h"], torch.bfloat16, dev)
        W = to_dev(case["W"], torch.bfloat16, dev)
        ctx.lmhead_fwd(h, W, tok, to_dev(case["old"], torch.float32, dev),
                       to_dev(case["mask"], torch.uint8, dev))
        ctx.loss_finalize()
        dW = torch.full((V, d), 0.25, dtype=torch.float32, device=dev)   # accumulates onto 0.25
        dh = torch.full((T, d), float("nan"), dtype=torch.float32, device=dev)
        ctx.lmhead_bwd(h, W, dh, dW)
        ctx.get_error()
        outs.append((dh.cpu().numpy().astype(np.float64), dW.cpu().numpy().astype(np.float64)))
        ctx.close()
    (h0, w0), (h1, w1) = outs
    assert np.isfinite(h0).all() and np.isfinite(w0).all()
    Wa = np.abs(case["W"].astype(np.float64))
    ha = np.abs(case["h"].astype(np.float64))
    # |dz| ≤ the recomputed gradient's magnitude: bound from the cuBLAS result's own terms
    # is not available, so use |dz| ≤ max|dz| per row via dh ≈ Σ|dz||W|: take the loose
    # K·2^-23·(|dz|@|W|) with |dz| ≤ 1 (the coefficients are ≤ |Â|·v·w/N ≤ 1 here)
    lim_dh = V * 2.0 ** -23 * Wa.sum(0)[None, :] * 1.0 + 1e-30
    lim_dW = 0.25 * 2.0 ** -23 + T * 2.0 ** -23 * ha.sum(0)[None, :] + 1e-30
    assert np.all(np.abs(h0 - h1) <= lim_dh)
    assert np.all(np.abs(w0 - w1) <= lim_dW)
    assert np.linalg.norm(h0 - h1) <= 1e-4 * np.linalg.norm(h1)
    assert np.linalg.norm(w0 - w1 - 0) <= 1e-4 * np.linalg.norm(w1 - 0.25)


@pytest.mark.parametrize("gemm,sub", [(0, 0), (2, 128)], ids=["pair", "1cta_sub128"])
def test_lmhead_bwd_compaction_equals_all_rows(gemm, sub):
    """ESPO_OPT_LMHEAD_COMPACT: the backward over the gathered rows with gradient only equals
    the backward over all rows — dh bitwise (same per-row dot products in the same K order;
    rows without gradient exactly 0), dW within the fp32 accumulation-order bound (the same
    non-zero products summed in different K=16 groups)."""
    from paper_2512_07710_b200.espo import (OPT_LMHEAD_BWD_GEMM, OPT_LMHEAD_BWD_ROWS,
                                            OPT_LMHEAD_COMPACT)
    dev = require_cuda()
    V, d = 5003, 256
    case = make_case(21, 4, 4, 45, V, d, zv_group=1)      # ZV group + masked tail
    T = case["T"]
    case["old"] = case["old"] + np.where(np.arange(T) % 3 == 0, 0.5, 0.0).astype(np.float32)
    outs = []
    for compact in (1, 0):
        ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
        ctx.set_option(OPT_LMHEAD_BWD_GEMM, gemm)
        ctx.set_option(OPT_LMHEAD_COMPACT, compact)
        if sub:
            ctx.set_option(OPT_LMHEAD_BWD_ROWS, sub)
        tok = to_dev(case["tokens"], torch.int32, dev)
        ctx.prepare(to_dev(case["rewards"], torch.float32, dev),
                    to_dev(case["group_ids"], torch.int32, dev), to_dev(case["so"], torch.int64, dev),
                    n_tokens=T)
        h = to_dev(case["h"], torch.bfloat16, dev)
        W = to_dev(case["W"], torch.bfloat16, dev)
        ctx.lmhead_fwd(h, W, tok, to_dev(case["old"], torch.float32, dev),
                       to_dev(case["mask"], torch.uint8, dev))
        _, st = ctx.loss_finalize()
        dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
        dh = torch.full((T, d), float("nan"), dtype=torch.float32, device=dev)
        half = T // 2 + 3
        ctx.lmhead_bwd(h[:half], W, dh[:half], dW, row_begin=0)
        ctx.lmhead_bwd(h[half:], W, dh[half:], dW, row_begin=half)
        ctx.get_error()
        g = ctx.export_token_stats()
        outs.append((dh.cpu().numpy(), dW.cpu().numpy().astype(np.float64),
                     (g["coef"] != 0).cpu().numpy(), stats_to_dict(st)))
        ctx.close()
    (h1, w1, nz, st), (h0, w0, _, _) = outs
    assert 0 < nz.sum() < T and st["n_clipped_tokens"] > 0          # something to skip
    assert np.array_equal(h1, h0)                                   # bitwise, zeros included
    assert not np.any(h1[~nz])
    ha = np.abs(case["h"].astype(np.float64))
    lim = T * 2.0 ** -23 * (np.abs(w0).max() + 1e-30) + 2.0 ** -22 * np.abs(w0)
    assert np.all(np.abs(w1 - w0) <= lim + T * 2.0 ** -24 * ha.max())
    assert np.linalg.norm(w1 - w0) <= 1e-5 * np.linalg.norm(w0)


@pytest.mark.parametrize("kern", ["gemm", "1cta"])
def test_lmhead_degenerate_shapes(kern):
    """Edge cases of the GEMM-core LM head: every row of a zero-variance group (no live M-tile,
    no row with gradient: dh = 0, dW unchanged, loss 0), a single row, V smaller than one
    512-column tile, d = 8 (one K-step, mostly zero-filled by TMA), rows not a multiple of 256."""
    dev = require_cuda()
    # all rows eliminated
    V, d, G, L = 700, 64, 4, 33
    case = make_case(31, 1, G, L, V, d, zv_group=0)
    T = case["T"]
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
    set_kernel(ctx, kern)
    ctx.prepare(to_dev(case["rewards"], torch.float32, dev), to_dev(case["group_ids"], torch.int32, dev),
                to_dev(case["so"], torch.int64, dev), n_tokens=T)
    h = to_dev(case["h"], torch.bfloat16, dev)
    W = to_dev(case["W"], torch.bfloat16, dev)
    ctx.lmhead_fwd(h, W, to_dev(case["tokens"], torch.int32, dev), to_dev(case["old"], torch.float32, dev))
    loss, st = ctx.loss_finalize()
    dW = torch.full((V, d), 0.5, dtype=torch.float32, device=dev)
    dh, _ = ctx.lmhead_bwd(h, W, None, dW)
    ctx.get_error()
    assert float(loss.item()) == 0.0 and stats_to_dict(st)["n_active_rollouts"] == 0
    assert not torch.any(dh) and torch.all(dW == 0.5)
    ctx.close()
    # tiny shapes against the oracle: one 2-rollout group of 1-token rollouts at d = 8, and
    # 3 × 37 rows with V = 300 (< one tile)
    for (ng, G, L, V, d) in ((1, 2, 1, 300, 8), (1, 3, 37, 300, 40)):
        case = make_case(37, ng, G, L, V, d)
        case["mask"][:] = 1
        T = case["T"]
        ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
        set_kernel(ctx, kern)
        ctx.prepare(to_dev(case["rewards"], torch.float32, dev), to_dev(case["group_ids"], torch.int32, dev),
                    to_dev(case["so"], torch.int64, dev), n_tokens=T)
        h = to_dev(case["h"], torch.bfloat16, dev)
        W = to_dev(case["W"], torch.bfloat16, dev)
        ctx.lmhead_fwd(h, W, to_dev(case["tokens"], torch.int32, dev), to_dev(case["old"], torch.float32, dev),
                       to_dev(case["mask"], torch.uint8, dev))
        loss, _ = ctx.loss_finalize()
        dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
        dh, _ = ctx.lmhead_bwd(h, W, None, dW)
        ctx.get_error()
        ctx.close()
        cfg = oracle_cfg(V)
        ref = O.espo_loss(case["z64"], case["tokens"], case["old"], case["mask"], case["rewards"],
                          case["group_ids"], case["so"], cfg)
        assert float(loss.item()) == pytest.approx(ref.loss, rel=1e-4, abs=1e-6)
        _, dh_ref, dW_ref = O.lmhead_grads(ref, case["h"], case["W"], case["tokens"], cfg)
        got_h, got_w = dh.cpu().numpy().astype(np.float64), dW.cpu().numpy().astype(np.float64)
        assert np.linalg.norm(got_h - dh_ref) <= 5e-3 * np.linalg.norm(dh_ref) + 1e-12
        assert np.linalg.norm(got_w - dW_ref) <= 5e-3 * np.linalg.norm(dW_ref) + 1e-12


@pytest.mark.parametrize("kern", ["gemm", "1cta"])
def test_lmhead_rlzvp_mode_matches_logits_path(kern):
    """RL-ZVP (zero-variance groups read, entropy-guided advantages): the fused LM head reads
    the ZV rows too (their M-tiles are live) and gives the logits path's statistics, loss and
    gradients (dh, dW within the bf16-dz bound)."""
    from paper_2512_07710_b200.espo import ZV_RLZVP
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = require_cuda()
    V, d = 3004, 256            # fp32 logits rows of the unfused path: 16-byte pitch
    case = make_case(41, 3, 4, 40, V, d, zv_group=1)
    T = case["T"]
    outs = {}
    for fused in (True, False):
        ctx = Espo(V, logits_dtype=torch.float32, device=dev.index, zv_mode=ZV_RLZVP, zvp_beta=0.2)
        set_kernel(ctx, kern)
        tok = to_dev(case["tokens"], torch.int32, dev)
        old = to_dev(case["old"], torch.float32, dev)
        mask = to_dev(case["mask"], torch.uint8, dev)
        ctx.prepare(to_dev(case["rewards"], torch.float32, dev), to_dev(case["group_ids"], torch.int32, dev),
                    to_dev(case["so"], torch.int64, dev), n_tokens=T)
        h = to_dev(case["h"], torch.bfloat16, dev)
        W = to_dev(case["W"], torch.bfloat16, dev)
        if fused:
            ctx.lmhead_fwd(h, W, tok, old, mask)
            loss, st = ctx.loss_finalize()
            dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
            dh, _ = ctx.lmhead_bwd(h, W, None, dW)
        else:
            z = (h.float() @ W.float().T).contiguous()
            ctx.loss_fwd(z, tok, old, mask)
            loss, st = ctx.loss_finalize()
            dz = ctx.loss_bwd(z)
            dh = dz @ W.float()
            dW = dz.T @ h.float()
        ctx.get_error()
        outs[fused] = (float(loss.item()), stats_to_dict(st), dh.cpu().numpy().astype(np.float64),
                       dW.cpu().numpy().astype(np.float64),
                       {k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()})
        ctx.close()
    (lf, sf, hf, wf, tf), (lu, su, hu, wu, tu) = outs[True], outs[False]
    assert sf["n_zv_groups"] == 1 and sf["n_active_rollouts"] == su["n_active_rollouts"] == 12
    assert np.array_equal(tf["valid"], tu["valid"])
    assert lf == pytest.approx(lu, rel=2e-3, abs=1e-6)
    assert np.linalg.norm(hf - hu) <= 4e-3 * np.linalg.norm(hu)
    assert np.linalg.norm(wf - wu) <= 4e-3 * np.linalg.norm(wu)


@pytest.mark.parametrize("d", [256, 4160])
def test_dynamic_tile_scheduler_is_bitwise_the_static_one(d):
    """The CTA-pair GEMMs take their work items from an atomic counter (handed to the pair's
    roles through a shared-memory queue; the default) or a static round robin
    (ESPO_OPT_LMHEAD_RASTER bit 29). Each tile is still computed by one pair in the same K order and merged in
    the same fixed order, so the forward statistics, loss, dhidden and dweight must be bitwise
    those of the static schedule — with dead M-tiles skipped (a zero-variance group), the soft
    lockstep on, and (d = 4160) split-K dh and the dh / dW lockstep."""
    from paper_2512_07710_b200.espo import OPT_LMHEAD_RASTER, Espo, stats_to_dict
    dev = require_cuda()
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    G, L, V = 8, 64, 4104
    R = 3 * G
    n = R * L
    h = (torch.randn(n, d, device=dev, generator=g) / d ** 0.5 * 3).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev, generator=g).to(torch.bfloat16)
    tok = torch.randint(0, V, (n,), device=dev, dtype=torch.int32, generator=g)
    rew = torch.tensor([1.0, 0.0] * (G // 2) + [1.0] * G + [0.0, 1.0, 1.0, 0.0] * 2, device=dev)
    gid = torch.arange(3, dtype=torch.int32, device=dev).repeat_interleave(G)
    off = torch.arange(R + 1, device=dev, dtype=torch.int64) * L
    old = torch.full((n,), -8.0, device=dev)
    out = []
    for dyn in (0, 1):
        ctx = Espo(V, logits_dtype=torch.bfloat16, device=dev.index)
        ctx.set_option(OPT_LMHEAD_RASTER, dyn << 29)
        ctx.prepare(rew, gid, off, n_tokens=n)
        ctx.lmhead_fwd(h, W, tok, old)
        loss, stats = ctx.loss_finalize()
        dh = torch.empty((n, d), dtype=torch.float32, device=dev)
        dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
        ctx.lmhead_bwd(h, W, dh, dW)
        ctx.get_error()
        tk = ctx.export_token_stats()
        out.append((loss.clone(), stats.clone(), tk["lp"].clone(), tk["H"].clone(), dh, dW))
        ctx.close()
    assert stats_to_dict(out[0][1])["n_zv_groups"] == 1
    for a, b in zip(out[0], out[1]):
        assert torch.equal(torch.nan_to_num(a, nan=7.0), torch.nan_to_num(b, nan=7.0))
    assert float(out[0][4].abs().max()) > 0


@pytest.mark.parametrize("d", [1000, 4160])
def test_tma_reduce_dw_epilogue_is_bitwise(d):
    """The dW GEMM's epilogue adds each 32 × 32 fp32 block into dW with a TMA reduce
    (cp.reduce.async.bulk.tensor .add; the default) or an SM-side read-add-write
    (ESPO_OPT_LMHEAD_RASTER bit 30) — one fp32 add per element either way, so dW (accumulated
    over several sub-chunks onto a non-zero start, ragged vocabulary rows and d columns) is
    bitwise the same."""
    from paper_2512_07710_b200.espo import OPT_LMHEAD_BWD_ROWS, OPT_LMHEAD_RASTER, Espo
    dev = require_cuda()
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    G, L, V = 4, 96, 5003
    n = G * L
    h = (torch.randn(n, d, device=dev, generator=g) / d ** 0.5 * 3).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev, generator=g).to(torch.bfloat16)
    tok = torch.randint(0, V, (n,), device=dev, dtype=torch.int32, generator=g)
    rew = torch.tensor([1.0, 0.0, 1.0, 0.0], device=dev)
    gid = torch.zeros(G, dtype=torch.int32, device=dev)
    off = torch.arange(G + 1, device=dev, dtype=torch.int64) * L
    dW0 = torch.randn(V, d, device=dev, generator=g)
    out = []
    for red in (0, 1):
        ctx = Espo(V, logits_dtype=torch.bfloat16, device=dev.index)
        ctx.set_option(OPT_LMHEAD_RASTER, red << 30)
        ctx.set_option(OPT_LMHEAD_BWD_ROWS, 128)          # three sub-chunks accumulate into dW
        ctx.prepare(rew, gid, off, n_tokens=n)
        ctx.lmhead_fwd(h, W, tok, torch.full((n,), -8.0, device=dev))
        ctx.loss_finalize()
        dh = torch.empty((n, d), dtype=torch.float32, device=dev)
        dW = dW0.clone()
        ctx.lmhead_bwd(h, W, dh, dW)
        ctx.get_error()
        out.append((dh, dW))
        ctx.close()
    assert torch.equal(out[0][0], out[1][0])
    assert torch.equal(out[0][1], out[1][1])
    assert not torch.equal(out[0][1], dW0)
