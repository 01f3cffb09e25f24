"""libespo's world > 1 arithmetic on one GPU, through the split finalize
(espo_loss_reduce_local → caller-side sum → espo_loss_finalize_reduced).

SURVEY §8(e): prompt groups are sharded over DP ranks (sharding.plan_shards, LPT), each rank
sweeps only its groups, and the one exchange of the pass is the sum of the 26 fp64
reduction terms. Here W contexts on the same device play the W ranks one after another (no
kernel of one waits on another), their partial vectors are summed on the device in rank
order, and each context finalizes with the sum. Checks: every rank's dlogits
rows are BITWISE the rows of one context holding the whole batch; counts exact; loss and the
fp64 statistics within 1e-12 relative (only the order of the fp64 sum differs); and the loss
matches the oracle at the usual tolerance. This is the code path the NCCL all-reduce feeds
in a real multi-GPU run (espo_loss_finalize = reduce_local + ncclAllReduce + finalize)."""
import numpy as np
import pytest
import torch

from paper_2512_07710_b200.sharding import plan_shards, shard_batch
from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import (check_loss, decision_aware_reference, oracle_cfg, require_cuda,
                              run_gpu, to_dev)

pytestmark = pytest.mark.gpu


def _run_sharded(inst, dev, world, method="lpt", logits_dtype=torch.float32, cfgkw=None):
    from paper_2512_07710_b200.espo import REDUCE_LEN, Espo, stats_to_dict
    plan = plan_shards(inst.group_ids, inst.seq_offsets, world, rewards=inst.rewards,
                       method=method)
    ctxs, parts, shards = [], [], []
    z_all = to_dev(inst.logits, torch.float32, dev).to(logits_dtype)
    for r in range(world):
        rollouts, toks, gid, so = shard_batch(plan[r], inst.group_ids, inst.seq_offsets)
        ti = torch.from_numpy(toks).to(dev)
        c = Espo(inst.V, logits_dtype=logits_dtype, device=dev.index, **(cfgkw or {}))
        z = z_all[ti].contiguous() if len(toks) else torch.zeros((0, inst.V), dtype=logits_dtype,
                                                                  device=dev)
        c.prepare(to_dev(inst.rewards[rollouts], torch.float32, dev), to_dev(gid, torch.int32, dev),
                  to_dev(so, torch.int64, dev), n_tokens=len(toks))
        if len(toks):
            c.loss_fwd(z, to_dev(inst.tokens[toks], torch.int32, dev),
                       to_dev(inst.old_logp[toks], torch.float32, dev),
                       to_dev(inst.mask[toks], torch.uint8, dev))
        parts.append(c.loss_reduce_local())
        ctxs.append(c)
        shards.append((toks, z))
    red = torch.zeros(REDUCE_LEN, dtype=torch.float64, device=dev)
    for p in parts:                               # the all-reduce, in rank order
        red += p
    out = []
    for c, (toks, z) in zip(ctxs, shards):
        loss, stats = c.loss_finalize_reduced(red)
        dz = c.loss_bwd(z) if len(toks) else None
        c.get_error()
        out.append(dict(loss=float(loss.item()), stats=stats_to_dict(stats), toks=toks,
                        dz=None if dz is None else dz.float().cpu().numpy()))
        c.close()
    return out, plan


@pytest.mark.parametrize("world,method", [(2, "lpt"), (3, "block"), (4, "lpt")])
def test_sharded_ranks_bitwise_equal_single_context(world, method):
    dev = require_cuda()
    inst = tiny_instance(41, V=1024, group_sizes=(4, 4, 3, 4, 2, 4, 1, 4), L=24, mask_tail=5,
                         rewards=[1, 0, 0, 1, 1, 1, 1, 1, 0, 1, 0, 1, 0, 1, 1, 0.5, 0.5,
                                  0.25, 0.75, 0.2, 0, 1, 1, 0, 1, 0])
    single = run_gpu(inst, dev)
    out, plan = _run_sharded(inst, dev, world, method)
    assert sorted(sum(plan, [])) == list(range(8))
    for o in out:
        for k in ("n_active_rollouts", "n_active_tokens", "n_zv_groups", "n_groups",
                  "n_clipped_tokens"):
            assert o["stats"][k] == single["stats"][k], k
        assert o["stats"]["loss"] == pytest.approx(single["stats"]["loss"], rel=1e-12, abs=1e-15)
        for k in ("mean_entropy", "mean_abs_logratio", "mean_k3"):
            assert o["stats"][k] == pytest.approx(single["stats"][k], rel=1e-12, abs=1e-15)
        if o["dz"] is not None:
            assert np.array_equal(o["dz"], single["dlogits"][o["toks"]])    # bitwise
    assert len({o["stats"]["loss"] for o in out}) == 1                     # same on every rank
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    ref2, _ = decision_aware_reference(single, inst, ref, cfg)
    check_loss(out[0], ref2, 1e-5)


def test_sharded_c3_shape_bf16_compact():
    """Variable lengths and many eliminated groups (the C3 recipe, shrunk), bf16 logits,
    compact mode: LPT plan over 4 ranks, bitwise dlogits rows vs one context."""
    dev = require_cuda()
    inst = workload_instance("C3", n_prompts=12, L=96, V=2048)
    single = run_gpu(inst, dev, logits_dtype=torch.bfloat16, grad_dtype=torch.float32,
                     cfgkw=dict(zero_fill_inactive_rows=0))
    out, _ = _run_sharded(inst, dev, 4, logits_dtype=torch.bfloat16,
                          cfgkw=dict(zero_fill_inactive_rows=0, grad_dtype=torch.float32))
    written = np.isfinite(single["dlogits"]).all(axis=1)   # compact: rows with gradient only
    assert written.sum() == single["stats"]["n_active_tokens"] - single["stats"]["n_clipped_tokens"]
    for o in out:
        assert o["stats"]["n_active_tokens"] == single["stats"]["n_active_tokens"]
        assert o["stats"]["loss"] == pytest.approx(single["stats"]["loss"], rel=1e-12, abs=1e-15)
        if o["dz"] is None:
            continue
        rows = o["toks"]
        v = written[rows]
        assert np.array_equal(o["dz"][v], single["dlogits"][rows][v])


def test_split_finalize_call_order():
    from paper_2512_07710_b200.espo import EspoError, Espo
    dev = require_cuda()
    inst = tiny_instance(43, V=256, group_sizes=(2, 2), L=6)
    c = Espo(inst.V, logits_dtype=torch.float32, device=dev.index)
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    z = to_dev(inst.logits, torch.float32, dev)
    tok, old = to_dev(inst.tokens, torch.int32, dev), to_dev(inst.old_logp, torch.float32, dev)
    c.prepare(*args, n_tokens=inst.T)
    with pytest.raises(EspoError) as e:
        c.loss_reduce_local()                     # rows not covered
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    c.loss_fwd(z, tok, old)
    with pytest.raises(EspoError) as e:
        c.loss_finalize_reduced(torch.zeros(26, dtype=torch.float64, device=dev))
    assert e.value.code == "ESPO_ERR_BAD_STATE"   # before reduce_local
    p = c.loss_reduce_local()
    with pytest.raises(EspoError) as e:
        c.loss_bwd(z)                             # before finalize_reduced
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    loss, _ = c.loss_finalize_reduced(p)          # world 1: the sum is the local vector
    c.loss_bwd(z)
    c.get_error()
    ref = run_gpu(inst, dev)
    assert float(loss.item()) == ref["loss"]
    c.close()
