"""Fused LM head at full size against the oracle: V = 151,936, d = 4,096,
n = 1,024 rows — espo_lmhead_fwd statistics and loss, and espo_lmhead_bwd's dh rows and dW
vocabulary rows (sampled) against O2-O7/O9 on fp64 logits z = h·Wᵀ of the same bf16 h, W.

Tolerances ("LM head"):
- per-token lse / lp / H: the K2 bounds (2e-6 / 2e-6 / 1e-5 relative) plus the fp32
  accumulation error of the logits GEMM, d·2^-24·max_v Σ_k |h_k W_vk| per row;
- loss: 2e-3 relative (north_star's bf16 tolerance; in practice ~1e-6);
- dh / dW: the kernel rounds dz to bf16 before the two contractions (RNE: ≤ 2^-8 relative per
  element), so (a) against the exact oracle, elementwise |Δ| ≤ (2^-8 + logit error)·|dz|·|W|
  summed over the contraction + fp32 accumulation, and (b) against the oracle's own dz
  rounded to bf16 the same way, the row-norm relative error ≤ 5e-4 (only rounding-boundary
  flips and fp32 accumulation order remain) — this pins the GEMM arithmetic itself."""
import numpy as np
import pytest
import torch

import espo_synth as S
from oracle import espo_oracle as O
from paper_2512_07710_b200.espo import Espo, stats_to_dict
from tests._instances import Instance
from tests.gpu_common import decision_aware_reference, oracle_cfg, require_cuda, to_dev

pytestmark = pytest.mark.gpu

V, D, G, L, NG = 151936, 4096, 8, 32, 4       # n = NG·G·L = 1024 rows


def _logits64(h, W, block=8192):
    h64 = h.astype(np.float64)
    z = np.empty((h.shape[0], W.shape[0]))
    for v0 in range(0, W.shape[0], block):
        z[:, v0:v0 + block] = h64 @ W[v0:v0 + block].astype(np.float64).T
    return z


def test_lmhead_full_size_vs_oracle():
    dev = require_cuda()
    rng = np.random.default_rng(2024)
    n = NG * G * L
    h = S.round_to_bf16((rng.standard_normal((n, D)) / np.sqrt(D) * 3).astype(np.float32))
    W = S.round_to_bf16(rng.standard_normal((V, D)).astype(np.float32))
    z64 = _logits64(h, W)
    tokens = S.sample_tokens_gumbel(z64.astype(np.float32), 99)
    gid = np.repeat(np.arange(NG, dtype=np.int32), G)
    so = np.arange(NG * G + 1, dtype=np.int64) * L
    rewards = (rng.uniform(size=NG * G) < 0.5).astype(np.float32)
    for g in range(NG):
        rewards[g * G], rewards[g * G + 1] = 1.0, 0.0
    rewards[2 * G:3 * G] = 1.0                              # one zero-variance group
    lp = np.array([O.row_stats(z64[t], int(tokens[t]))[1] for t in range(n)])
    old = S.drift_old_logp(lp, so, 99, sigma_seq=0.01, sigma_tok=0.02)
    mask = np.ones(n, np.uint8)
    mask[L - 4:L] = 0

    ctx = Espo(V, logits_dtype=torch.bfloat16, device=dev.index)
    tok = to_dev(tokens, torch.int32, dev)
    ctx.prepare(to_dev(rewards, torch.float32, dev), to_dev(gid, torch.int32, dev),
                to_dev(so, torch.int64, dev), n_tokens=n)
    hd, Wd = to_dev(h, torch.bfloat16, dev), to_dev(W, torch.bfloat16, dev)
    ctx.lmhead_fwd(hd, Wd, tok, to_dev(old, torch.float32, dev), to_dev(mask, torch.uint8, dev))
    loss, stats = ctx.loss_finalize()
    dW = torch.zeros((V, D), dtype=torch.float32, device=dev)
    dh = torch.full((n, D), float("nan"), dtype=torch.float32, device=dev)
    ctx.lmhead_bwd(hd, Wd, dh, dW)
    ctx.get_error()
    g = dict(tok={k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()})
    st = stats_to_dict(stats)
    ctx.close()

    inst = Instance(z64, tokens, old, mask, rewards, gid, so, V)
    cfg = oracle_cfg(V)
    ref = inst.run(cfg)
    v = ref.kappa >= 0
    assert np.array_equal(g["tok"]["valid"].astype(bool), v)
    # per-row logit error bound of the fp32-accumulating GEMM
    B = 16384
    blk = lambda a, v0: a[v0:v0 + B].astype(np.float64)       # W blocks in fp64, on the fly
    ha = np.abs(h).astype(np.float64)
    b_t = np.zeros(n)
    for v0 in range(0, V, B):
        b_t = np.maximum(b_t, (ha @ np.abs(blk(W, v0)).T).max(axis=1))
    b_t *= D * 2.0 ** -24
    for k, tol, kb in (("lse", 2e-6, 1), ("lp", 2e-6, 2), ("H", 1e-5, 4)):
        diff = np.abs(g["tok"][k][v].astype(np.float64) - getattr(ref, k)[v])
        lim = tol * np.maximum(1, np.abs(getattr(ref, k)[v])) + kb * b_t[v]
        assert np.all(diff <= lim), (k, np.max(diff / lim))
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    assert abs(st["loss"] - ref2.loss) <= 2e-3 * abs(ref2.loss) + 1e-9, (st["loss"], ref2.loss)

    # sampled rows of dh (incl. masked / eliminated rows) and vocabulary rows of dW (incl. the
    # sampled rows' targets, whose dz carries the +g·q term)
    rows = np.unique(np.concatenate([rng.choice(n, 24, replace=False), [L - 1, 2 * G * L + 3]]))
    dz = np.stack([O.dlogits_row(ref2, int(t), z64[t], int(tokens[t]), cfg) for t in range(n)])
    cols = np.unique(np.concatenate([rng.choice(V, 40, replace=False), tokens[rows[:24]]]))
    got_dh = dh[torch.from_numpy(rows).to(dev)].cpu().numpy().astype(np.float64)
    got_dW = dW[torch.from_numpy(cols).to(dev)].cpu().numpy().astype(np.float64)
    dh_ref = np.zeros((len(rows), D))
    for v0 in range(0, V, B):
        dh_ref += dz[rows, v0:v0 + B] @ blk(W, v0)
    dW_ref = dz[:, cols].T @ h.astype(np.float64)
    zrows = ~(ref2.coef[rows] != 0)
    assert np.all(got_dh[zrows] == 0)                      # no gradient: exactly zero
    # (a) exact oracle, elementwise: bf16 rounding of dz (2^-8) + logit error + fp32 sums
    adz = np.abs(dz) * (2.0 ** -8 + 4 * b_t[:, None] + 1e-6)
    lim_dh = np.zeros((len(rows), D))
    for v0 in range(0, V, B):
        lim_dh += (adz[rows, v0:v0 + B] + V * 2.0 ** -24 * np.abs(dz[rows, v0:v0 + B])) \
            @ np.abs(blk(W, v0))
    lim_dW = (adz[:, cols] + n * 2.0 ** -24 * np.abs(dz[:, cols])).T @ ha
    assert np.all(np.abs(got_dh - dh_ref) <= lim_dh + 1e-30), np.max(np.abs(got_dh - dh_ref) / (lim_dh + 1e-30))
    assert np.all(np.abs(got_dW - dW_ref) <= lim_dW + 1e-30), np.max(np.abs(got_dW - dW_ref) / (lim_dW + 1e-30))
    # (b) against the oracle's dz rounded to bf16 (RNE) the way the kernel rounds its own
    dzb = S.round_to_bf16(dz.astype(np.float32)).astype(np.float64)
    dhb = np.zeros((len(rows), D))
    for v0 in range(0, V, B):
        dhb += dzb[rows, v0:v0 + B] @ blk(W, v0)
    dWb = dzb[:, cols].T @ h.astype(np.float64)
    for r in range(len(rows)):
        nr = np.linalg.norm(dhb[r])
        if nr > 0:
            assert np.linalg.norm(got_dh[r] - dhb[r]) <= 5e-4 * nr, r
    for c in range(len(cols)):
        nc = np.linalg.norm(dWb[c])
        if nc > 0:
            assert np.linalg.norm(got_dW[c] - dWb[c]) <= 5e-4 * nc, c
