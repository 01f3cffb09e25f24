"""Context parallelism (SURVEY §8(f) row 3 sibling): rollouts split across CP ranks by token
blocks. On one GPU the ranks are separate contexts; espo_cp_gather_local stands in for the
NCCL all-gather of the 13 B/token the per-rollout reduction reads. Every CP rank must report
the unsharded loss bit for bit, and the gradient rows of its block must be bitwise those of
the unsharded run (and so match the oracle)."""
import numpy as np
import pytest
import torch

from oracle import espo_oracle as O
from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import (check_dlogits_f32, check_exact_fields, check_loss,
                              check_token_stats, decision_aware_reference, oracle_cfg,
                              oracle_dlogits, require_cuda, run_gpu, to_dev)

pytestmark = pytest.mark.gpu


def run_cp(inst, dev, cp, cfgkw=None, logits_dtype=torch.float32, sub_chunks=2, factored=False):
    """factored: each CP rank runs espo_loss_fwd_factored on its block (G into one buffer) and
    the gradient rows are espo_loss_row_scale · G (fp64 here)."""
    from paper_2512_07710_b200.espo import Espo, stats_to_dict
    T, V = inst.T, inst.V
    z = to_dev(inst.logits, torch.float32, dev).to(logits_dtype)
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev)
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    ctxs = []
    for k in range(cp):
        c = Espo(V, logits_dtype=logits_dtype, device=dev.index, **(cfgkw or {}))
        c.attach_cp(k, cp, local=True)
        c.prepare(*args, n_tokens=T)
        ctxs.append(c)
    G = torch.full((T, V), float("nan"), dtype=ctxs[0].grad_dtype, device=dev)
    for c in ctxs:                                   # each rank sweeps its own block
        lo, hi = c.cp_block()
        cuts = np.linspace(lo, hi, sub_chunks + 1).astype(int)
        for b, e in zip(cuts[:-1], cuts[1:]):
            if e > b:
                if factored:
                    c.loss_fwd_factored(z[b:e], tok[b:e], old[b:e], mask[b:e], grad=G[b:e],
                                        row_begin=int(b))
                else:
                    c.loss_fwd(z[b:e], tok[b:e], old[b:e], mask[b:e], row_begin=int(b))
    for c in ctxs:
        c.cp_gather_local(ctxs)
    dz = torch.full((T, V), float("nan"), dtype=ctxs[0].grad_dtype, device=dev)
    dzf = np.full((T, V), np.nan)
    out = []
    for c in ctxs:
        loss, stats = c.loss_finalize()
        lo, hi = c.cp_block()
        if hi > lo and factored:
            sc = c.loss_row_scale(lo, hi - lo).double().cpu().numpy()
            Gb = G[lo:hi].double().cpu().numpy()
            with np.errstate(invalid="ignore"):
                dzf[lo:hi] = sc[:, None] * Gb
            dzf[lo:hi][sc == 0] = 0.0
        elif hi > lo:
            c.loss_bwd(z[lo:hi], dz[lo:hi], row_begin=lo)
        c.get_error()
        out.append((float(loss.item()), stats_to_dict(stats)))
    res = dict(losses=[o[0] for o in out], loss=out[0][0], stats=out[0][1],
               dlogits=dzf if factored else dz.float().cpu().numpy(),
               tok={k: v.cpu().numpy() for k, v in ctxs[0].export_token_stats().items()},
               rol={k: v.cpu().numpy() for k, v in ctxs[0].export_rollout_stats().items()})
    res["zv_out"] = res["rol"]["zv"]
    for c in ctxs:
        c.close()
    return res


@pytest.mark.parametrize("cp", [2, 3, 5])
def test_context_parallel_equals_unsharded(cp):
    dev = require_cuda()
    inst = workload_instance("C0")                   # 16 rollouts × 64: blocks cut sequences
    g = run_cp(inst, dev, cp)
    u = run_gpu(inst, dev)
    assert all(l == u["loss"] for l in g["losses"])
    assert g["stats"] == u["stats"]
    assert np.array_equal(g["dlogits"], u["dlogits"])
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))


def test_context_parallel_bf16_rlzvp_variable_lengths():
    dev = require_cuda()
    inst = tiny_instance(81, V=2056, group_sizes=(4, 3, 4), lengths=[30, 7, 0, 44, 12, 9, 25,
                                                                      3, 40, 18, 22],
                         dtype="bf16", mask_tail=3, rewards=[1, 0, 1, 1, 1, 1, 1, 0, 0, 1, 0])
    kw = dict(cfgkw={"zv_mode": O.ZV_RLZVP}, logits_dtype=torch.bfloat16)
    g = run_cp(inst, dev, 4, **kw)
    u = run_gpu(inst, dev, **kw)
    assert all(l == u["loss"] for l in g["losses"])
    assert np.array_equal(g["dlogits"], u["dlogits"], equal_nan=True)


def test_context_parallel_rejects_rows_outside_block():
    from paper_2512_07710_b200.espo import Espo, EspoError
    dev = require_cuda()
    inst = workload_instance("C0")
    c = Espo(inst.V, logits_dtype=torch.float32, device=dev.index)
    c.attach_cp(1, 2, local=True)
    c.prepare(to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
              to_dev(inst.seq_offsets, torch.int64, dev), n_tokens=inst.T)
    z = to_dev(inst.logits, torch.float32, dev)
    with pytest.raises(EspoError) as e:
        c.loss_fwd(z[:10], to_dev(inst.tokens[:10], torch.int32, dev),
                   to_dev(inst.old_logp[:10], torch.float32, dev))
    assert e.value.code == "ESPO_ERR_INVALID_ARGUMENT"
    lo, hi = c.cp_block()
    c.loss_fwd(z[lo:hi], to_dev(inst.tokens[lo:hi], torch.int32, dev),
               to_dev(inst.old_logp[lo:hi], torch.float32, dev), row_begin=lo)
    with pytest.raises(EspoError) as e:              # emulation: the gather has not run
        c.loss_finalize()
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    c.close()


@pytest.mark.parametrize("cp", [2, 3])
def test_context_parallel_factored_equals_unsharded_factored(cp):
    """CP ranks running the factored sweep on their token blocks: loss, statistics and every
    scale·G row bitwise those of the unsharded factored run (rows are independent of the
    block cut; K3 sees the same gathered values), hence at parity with the oracle."""
    dev = require_cuda()
    inst = workload_instance("C0")
    g = run_cp(inst, dev, cp, factored=True)
    u = run_gpu(inst, dev, factored=True)
    assert all(l == u["loss"] for l in g["losses"])
    assert g["stats"] == u["stats"]
    assert np.array_equal(g["dlogits"], u["dlogits"])
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))
