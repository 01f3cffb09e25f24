"""The NCCL code paths on one GPU, through one-rank communicators (no rank waits on another):
the DP all-reduce in espo_loss_finalize and espo_set_mask, the TP all-gather of partials in
espo_loss_fwd, and the CP all-gather at finalize. A one-rank collective is an identity, so
each run must equal the communicator-free run bit for bit — which checks the dlopen'd NCCL
entry points, datatypes, counts and in-place buffer layouts that multi-GPU runs use."""
import numpy as np
import pytest
import torch

from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import require_cuda, run_gpu, to_dev

pytestmark = pytest.mark.gpu


def _args(inst, dev):
    return (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))


def _pass(ctx, inst, dev, z, single=False):
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev)
    ctx.prepare(*_args(inst, dev), n_tokens=inst.T)
    dz = torch.empty_like(z)
    if single:
        ctx.set_mask(mask)
        ctx.loss_fwd_bwd(z, tok, old, dz)
        loss, _ = ctx.loss_finalize()
    else:
        ctx.loss_fwd(z, tok, old, mask)
        loss, _ = ctx.loss_finalize()
        ctx.loss_bwd(z, dz)
    ctx.get_error()
    return float(loss.item()), dz.cpu().numpy()


@pytest.mark.parametrize("single", [False, True], ids=["two_sweep", "single_pass"])
def test_dp_one_rank_nccl(single):
    from paper_2512_07710_b200.espo import Espo, new_unique_id
    dev = require_cuda()
    inst = workload_instance("C0")
    z = to_dev(inst.logits, torch.float32, dev)
    a = Espo(inst.V, logits_dtype=torch.float32, device=dev.index)
    b = Espo(inst.V, logits_dtype=torch.float32, device=dev.index, nccl_id=new_unique_id())
    la, da = _pass(a, inst, dev, z, single)
    lb, db = _pass(b, inst, dev, z, single)
    assert la == lb and np.array_equal(da, db)
    a.close()
    b.close()


def test_tp_one_rank_nccl_allgather():
    """vocab shard [0, 512) of V = 1024 with every token inside it: espo_loss_fwd's
    partial → ncclAllGather → combine equals partial + explicit combine, bitwise."""
    from paper_2512_07710_b200.espo import Espo, new_unique_id
    dev = require_cuda()
    inst = tiny_instance(91, V=1024, group_sizes=(4, 4), L=20, mask_tail=3)
    inst.tokens = (inst.tokens % 512).astype(np.int32)
    z = to_dev(inst.logits[:, :512], torch.float32, dev).contiguous()
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev)
    out = []
    for use_nccl in (False, True):
        c = Espo(1024, logits_dtype=torch.float32, device=dev.index, vocab_shard=(0, 512))
        if use_nccl:
            c.attach_tp_id(new_unique_id(), 0, 1)
        c.prepare(*_args(inst, dev), n_tokens=inst.T)
        if use_nccl:
            c.loss_fwd(z, tok, old, mask)
        else:
            part = c.loss_fwd_partial(z, tok, old, mask)
            c.loss_fwd_combine(part.unsqueeze(0))
        loss, _ = c.loss_finalize()
        dz = c.loss_bwd(z)
        c.get_error()
        out.append((float(loss.item()), dz.cpu().numpy(),
                    {k: v.cpu().numpy() for k, v in c.export_token_stats().items()}))
        c.close()
    assert out[0][0] == out[1][0] and np.array_equal(out[0][1], out[1][1])
    for k in ("lse", "lp", "H", "q"):
        assert np.array_equal(out[0][2][k], out[1][2][k], equal_nan=True)


def test_cp_one_rank_nccl_allgather():
    from paper_2512_07710_b200.espo import Espo, new_unique_id
    dev = require_cuda()
    inst = workload_instance("C0")
    z = to_dev(inst.logits, torch.float32, dev)
    c = Espo(inst.V, logits_dtype=torch.float32, device=dev.index)
    c.attach_cp(0, 1, nccl_id=new_unique_id())
    lb, db = _pass(c, inst, dev, z)
    u = run_gpu(inst, dev)
    assert lb == u["loss"] and np.array_equal(db, u["dlogits"])
    c.close()
