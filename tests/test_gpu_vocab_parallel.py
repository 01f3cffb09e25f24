"""Vocabulary-parallel ESPO: logits sharded by vocabulary columns as in
a Megatron vocab-parallel LM head. Each shard's sweep produces per-row partials
{R, S, W, u_y}; the partials of all shards are combined into the exact row statistics; the
backward writes each shard's columns. On one GPU the shards run as independent launches of
independent contexts and the all-gather is a device copy (no kernel waits on another);
results must match the oracle (and the unsharded run) at the usual tolerances."""
import numpy as np
import pytest
import torch

from paper_2512_07710_b200.espo import Espo
from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import (check_dlogits_bf16, check_dlogits_f32, check_exact_fields,
                              check_loss, check_token_stats, decision_aware_reference,
                              oracle_cfg, oracle_dlogits, require_cuda, run_gpu, to_dev)

pytestmark = pytest.mark.gpu


def run_sharded(inst, dev, shards, logits_dtype=torch.float32, grad_dtype=None, cfgkw=None,
                fwd_impl=0, bwd_impl=0):
    from paper_2512_07710_b200.espo import OPT_BWD_IMPL, OPT_FWD_IMPL, stats_to_dict
    cfgkw = dict(cfgkw or {})
    T, V = inst.T, inst.V
    align = 8 if logits_dtype == torch.bfloat16 else 4
    zfull = to_dev(inst.logits, torch.float32, dev)
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev)
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    ctxs, zs = [], []
    for v0, w in shards:
        ctx = Espo(V, logits_dtype=logits_dtype, grad_dtype=grad_dtype, device=dev.index,
                   vocab_shard=(v0, w), **cfgkw)
        ctx.set_option(OPT_FWD_IMPL, fwd_impl)
        ctx.set_option(OPT_BWD_IMPL, bwd_impl)
        ld = (w + align - 1) // align * align
        z = torch.zeros((T, ld), dtype=logits_dtype, device=dev)
        z[:, :w] = zfull[:, v0:v0 + w].to(logits_dtype)
        ctx.prepare(*args, n_tokens=T)
        ctxs.append(ctx)
        zs.append(z)
    parts = [c.loss_fwd_partial(z, tok, old, mask) for c, z in zip(ctxs, zs)]
    gathered = torch.stack(parts)                      # the TP all-gather, as a device copy
    out = []
    for (v0, w), c, z in zip(shards, ctxs, zs):
        c.loss_fwd_combine(gathered)
        loss, stats = c.loss_finalize()
        dz = c.loss_bwd(z)
        c.get_error()
        out.append((float(loss.item()), stats_to_dict(stats), dz[:, :w].float().cpu().numpy()))
    tokst = {k: v.cpu().numpy() for k, v in ctxs[0].export_token_stats().items()}
    rol = {k: v.cpu().numpy() for k, v in ctxs[0].export_rollout_stats().items()}
    for c in ctxs:
        c.close()
    dl = np.concatenate([o[2] for o in out], axis=1)
    return dict(loss=out[0][0], stats=out[0][1], losses=[o[0] for o in out], dlogits=dl,
                tok=tokst, rol=rol, zv_out=rol["zv"])


@pytest.mark.parametrize("impl", [0, 1], ids=["tma", "ldg"])
def test_vocab_parallel_fp32_three_shards(impl):
    dev = require_cuda()
    inst = workload_instance("C0")
    g = run_sharded(inst, dev, [(0, 300), (300, 400), (700, 324)], fwd_impl=impl, bwd_impl=impl)
    assert len(set(g["losses"])) == 1                 # every shard sees the same loss
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))
    u = run_gpu(inst, dev)                            # unsharded run: same result
    assert g["loss"] == pytest.approx(u["loss"], rel=1e-6)


def test_vocab_parallel_bf16_ragged_eight_shards():
    dev = require_cuda()
    inst = tiny_instance(17, V=4099, group_sizes=(8, 8), L=24, dtype="bf16", mask_tail=4)
    w = [512] * 7 + [4099 - 7 * 512]
    shards = [(sum(w[:k]), w[k]) for k in range(8)]
    g = run_sharded(inst, dev, shards, logits_dtype=torch.bfloat16, grad_dtype=torch.float32)
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))


def test_sharded_context_requires_partial_path():
    """A sharded context without a TP communicator cannot run the fused espo_loss_fwd."""
    from paper_2512_07710_b200.espo import EspoError
    dev = require_cuda()
    inst = tiny_instance(18, V=256, group_sizes=(2,), L=4)
    ctx = Espo(256, logits_dtype=torch.float32, device=dev.index, vocab_shard=(0, 128))
    ctx.prepare(to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
                to_dev(inst.seq_offsets, torch.int64, dev), n_tokens=inst.T)
    z = torch.zeros((inst.T, 128), dtype=torch.float32, device=dev)
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd(z, to_dev(inst.tokens, torch.int32, dev), to_dev(inst.old_logp, torch.float32, dev))
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    ctx.close()
