"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and compare with
the oracle by the P11 protocol of SURVEY.md §8(c) (exact fields bitwise, per-token stats
within fp32 bounds, decision-aware comparison of bucket / clip flips, loss and dlogits
within the north_star tolerances: 1e-5 relative for fp32 logits, 2e-3 for bf16)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import espo_oracle as O

GPU_TO_ORACLE = dict(alpha="alpha", eps_min="eps_min", n_buckets="n_buckets",
                     partition="partition", ratio_mode="ratio_mode", norm="norm",
                     std_unbiased="std_unbiased", adv_eps="adv_eps", zv_var_eps="zv_var_eps",
                     logit_scale="logit_scale", log_ratio_clamp="log_ratio_clamp")
F32_FIELDS = ("alpha", "eps_min", "logit_scale", "log_ratio_clamp", "zvp_beta", "zvp_threshold")


def require_cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    return torch.device("cuda", 0)


def oracle_cfg(V, **kw):
    """The oracle sees exactly the values the C config holds (float fields are f32)."""
    d = dict(alpha=0.4, eps_min=0.01, logit_scale=1.0, log_ratio_clamp=20.0, zvp_beta=0.05,
             zvp_threshold=0.5)
    d.update(kw)
    for k in F32_FIELDS:
        d[k] = float(np.float32(d[k]))
    return O.OracleConfig(vocab=V, **d)


def to_dev(a, dtype, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dtype)


def run_gpu(inst, dev, cfgkw=None, logits_dtype=torch.float32, grad_dtype=None, chunks=None,
            fwd_impl=0, bwd_impl=0, ld_pad=0, in_place=False, grad_loss=None, factored=False, factored_impl=0, sync_after_prepare=False,
            entropy=None, entropy_chunks=None):
    """Full pass on the GPU. chunks: list of (begin, end) for fwd (bwd uses the same).
    factored: espo_loss_fwd_factored per chunk + espo_loss_row_scale; "dlogits" is then
    scale_t · G_t formed in fp64 here (no second rounding), "G"/"scale" are returned too."""
    from paper_2512_07710_b200.espo import (Espo, OPT_BWD_IMPL, OPT_FACTORED_IMPL, OPT_FWD_IMPL,
                                            stats_to_dict)
    cfgkw = dict(cfgkw or {})
    V, T = inst.V, inst.T
    ctx = Espo(V, logits_dtype=logits_dtype, grad_dtype=grad_dtype, device=dev.index, **cfgkw)
    ctx.set_option(OPT_FWD_IMPL, fwd_impl)
    ctx.set_option(OPT_BWD_IMPL, bwd_impl)
    ctx.set_option(OPT_FACTORED_IMPL, factored_impl)
    ld = V + ld_pad
    zfull = torch.zeros((T, ld), dtype=logits_dtype, device=dev)
    zfull[:, :V] = to_dev(inst.logits, torch.float32, dev).to(logits_dtype)
    z = zfull
    tokens = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    mask = None if inst.mask is None else to_dev(inst.mask, torch.uint8, dev)
    adv_out = torch.empty(inst.R, dtype=torch.float32, device=dev)
    zv_out = torch.empty(inst.R, dtype=torch.uint8, device=dev)
    ctx.prepare(to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
                to_dev(inst.seq_offsets, torch.int64, dev), n_tokens=T, adv_out=adv_out,
                zv_out=zv_out)
    if sync_after_prepare:     # lets host-side copies taken at prepare land before the sweeps
        torch.cuda.synchronize(dev)
    if entropy is not None:    # caller-supplied selection entropies (espo_set_entropies)
        ent = torch.from_numpy(np.asarray(entropy, dtype=np.float32)).to(dev)
        for b, e in (entropy_chunks or [(0, T)]):
            ctx.set_entropies(ent[b:e], row_begin=b)
    chunks = chunks or [(0, T)]
    gl = None if grad_loss is None else torch.tensor([grad_loss], dtype=torch.float32, device=dev)
    if factored:
        G = z if in_place else torch.full((T, ld), float("nan"), dtype=ctx.grad_dtype, device=dev)
        for b, e in chunks:
            ctx.loss_fwd_factored(z[b:e], tokens[b:e], old[b:e],
                                  None if mask is None else mask[b:e], grad=G[b:e], row_begin=b)
        loss, stats = ctx.loss_finalize()
        scale = ctx.loss_row_scale(grad_loss=gl)
        ctx.get_error()
        Gn = G[:, :V].double().cpu().numpy()
        sc = scale.double().cpu().numpy()
        with np.errstate(invalid="ignore"):
            dl = sc[:, None] * Gn
        dl[sc == 0] = 0.0          # rows without gradient (G untouched in compact mode)
        tok = {k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()}
        rol = {k: v.cpu().numpy() for k, v in ctx.export_rollout_stats().items()}
        out = dict(loss=float(loss.item()), stats=stats_to_dict(stats), dlogits=dl, G=Gn,
                   scale=sc, tok=tok, rol=rol, adv_out=adv_out.cpu().numpy(),
                   zv_out=zv_out.cpu().numpy(), launches=ctx.launch_count)
        ctx.close()
        return out
    for b, e in chunks:
        ctx.loss_fwd(z[b:e], tokens[b:e], old[b:e], None if mask is None else mask[b:e],
                     row_begin=b)
    loss, stats = ctx.loss_finalize()
    if in_place:
        dz = z
    else:
        dz = torch.full((T, ld), float("nan"), dtype=ctx.grad_dtype, device=dev)
    for b, e in chunks:
        ctx.loss_bwd(z[b:e], dz[b:e], row_begin=b, grad_loss=gl)
    ctx.get_error()
    tok = {k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()}
    rol = {k: v.cpu().numpy() for k, v in ctx.export_rollout_stats().items()}
    out = dict(loss=float(loss.item()), stats=stats_to_dict(stats),
               dlogits=dz[:, :V].float().cpu().numpy(), tok=tok, rol=rol,
               adv_out=adv_out.cpu().numpy(), zv_out=zv_out.cpu().numpy(),
               launches=ctx.launch_count)
    ctx.close()
    return out


def check_exact_fields(g, ref):
    assert np.array_equal(g["rol"]["zv"].astype(bool), ref.zv)
    assert np.array_equal(g["zv_out"].astype(bool), ref.zv)
    assert np.array_equal(g["rol"]["active"].astype(bool), ref.active)
    # advantages: bit-exact (no-FMA fp64 in index order on both sides)
    assert np.array_equal(g["rol"]["adv"], ref.adv)
    s, rs = g["stats"], ref.stats
    for k in ("n_active_rollouts", "n_active_tokens", "n_zv_groups", "n_groups"):
        assert s[k] == rs[k], k
    valid = ref.kappa >= 0
    assert np.array_equal(g["tok"]["valid"].astype(bool), valid)


def check_token_stats(g, ref):
    v = ref.kappa >= 0
    t = g["tok"]
    for name, tol_abs_rel in (("lse", 2e-6), ("lp", 2e-6), ("H", 1e-5)):
        got, want = t[name][v].astype(np.float64), getattr(ref, name)[v]
        lim = tol_abs_rel * np.maximum(1.0, np.abs(want))
        bad = np.abs(got - want) > lim
        assert not bad.any(), (name, np.flatnonzero(bad)[:5], got[bad][:5], want[bad][:5])
    got, want = t["q"][v].astype(np.float64), ref.q[v]
    bad = np.abs(got - want) > 1e-5 * np.abs(want) + 1e-30
    assert not bad.any(), ("q", got[bad][:5], want[bad][:5])


def decision_aware_reference(g, inst, ref, cfg, flip_frac=1e-4, **run_kw):
    """P11.4: every bucket / clip disagreement must sit within δ of the oracle's kink; the
    oracle is then re-run with the GPU's decisions injected (run_kw: further arguments of
    the oracle run, e.g. supplied entropies)."""
    Hsel = np.asarray(run_kw["entropy"], dtype=np.float64) if run_kw.get("entropy") is not None else ref.H
    v = ref.kappa >= 0
    n_tok = int(v.sum())
    gb = g["tok"]["bucket"].astype(np.int64)
    gc = g["tok"]["clip"].astype(np.int64)
    flips = 0
    if cfg.partition == O.PARTITION_QUANTILE and cfg.n_buckets > 1:
        db = np.flatnonzero(v & (gb != ref.bucket))
        for t in db:
            i = int(np.searchsorted(inst.seq_offsets, t, side="right") - 1)
            margin = min(abs(Hsel[t] - th) for th in ref.theta[i])
            assert margin < 1e-5, ("bucket flip far from threshold", t, margin)
        flips += len(db)
    dc = np.flatnonzero(v & (gc != (1 - ref.kappa)))
    for t in dc:
        e = ref.eps_tok[t]
        margin = min(abs(ref.v[t] - (1 + e)), abs(ref.v[t] - (1 - e)))
        assert margin < 1e-5 * (1 + e) + 1e-6 * abs(ref.v[t]), ("clip flip far from kink", t, margin)
    flips += len(dc)
    assert flips <= max(flip_frac * n_tok, 3), flips
    if flips == 0:
        return ref, 0
    kap = np.where(v, 1 - gc, -1)
    ref2 = inst.run(cfg, inject_bucket=gb if cfg.partition == O.PARTITION_QUANTILE else None,
                    inject_kappa=kap, **run_kw)
    return ref2, flips


def check_loss(g, ref, rtol):
    floor = rtol * float(np.abs(ref.J_i).sum()) / max(ref.denom, 1.0)
    assert abs(g["loss"] - ref.loss) <= rtol * abs(ref.loss) + floor + 1e-12, (g["loss"], ref.loss)


def oracle_dlogits(ref, inst, cfg, rows, grad_loss=1.0):
    return np.stack([O.dlogits_row(ref, int(t), inst.logits[t], int(inst.tokens[t]), cfg,
                                   grad_loss) for t in rows])


def check_dlogits_f32(got, want, rtol=1e-5):
    for r in range(want.shape[0]):
        w, x = want[r], got[r].astype(np.float64)
        nrm = np.linalg.norm(w)
        if nrm == 0:
            assert not np.any(x), r
            continue
        assert np.linalg.norm(x - w) <= rtol * nrm, (r, np.linalg.norm(x - w) / nrm)
        lim = rtol * np.abs(w) + 1e-3 * rtol * np.abs(w).max()
        assert np.all(np.abs(x - w) <= lim), (r, np.max(np.abs(x - w) - lim))


def check_dlogits_bf16(got, want):
    x = got.astype(np.float64)
    tiny = 1e-8 * np.abs(want).max() if want.size else 0.0
    lim = (2.0 ** -8 + 1e-5) * np.abs(want) + tiny
    assert np.all(np.abs(x - want) <= lim), np.max(np.abs(x - want) - lim)
    nrm = np.linalg.norm(want)
    if nrm > 0:
        assert np.linalg.norm(x - want) / nrm <= 2e-3
