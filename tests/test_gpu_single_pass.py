"""Single-pass mode (espo_set_mask + espo_loss_fwd_bwd): D is fixed from the mask, then each
chunk of complete rollouts runs forward → K3 → backward in one call. Results must be
bitwise those of the two-sweep path (same kernels, same D) and match the oracle; chunks may
arrive in any order; misaligned chunks and mixed-mode calls are rejected."""
import numpy as np
import pytest
import torch

from oracle import espo_oracle as O
from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import (check_dlogits_f32, check_exact_fields, check_loss,
                              check_token_stats, decision_aware_reference, oracle_cfg,
                              oracle_dlogits, require_cuda, run_gpu, to_dev)

pytestmark = pytest.mark.gpu


def run_single(inst, dev, roll_chunks, cfgkw=None, logits_dtype=torch.float32, grad_dtype=None,
               in_place=False, grad_loss=None):
    from paper_2512_07710_b200.espo import Espo, stats_to_dict
    V, T = inst.V, inst.T
    ctx = Espo(V, logits_dtype=logits_dtype, grad_dtype=grad_dtype, device=dev.index,
               **(cfgkw or {}))
    z = to_dev(inst.logits, torch.float32, dev).to(logits_dtype)
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    ctx.prepare(to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
                to_dev(inst.seq_offsets, torch.int64, dev), n_tokens=T)
    ctx.set_mask(None if inst.mask is None else to_dev(inst.mask, torch.uint8, dev))
    dz = z if in_place else torch.full((T, V), float("nan"), dtype=ctx.grad_dtype, device=dev)
    gl = None if grad_loss is None else torch.tensor([grad_loss], dtype=torch.float32, device=dev)
    so = inst.seq_offsets
    for i0, i1 in roll_chunks:
        b, e = int(so[i0]), int(so[i1])
        ctx.loss_fwd_bwd(z[b:e], tok[b:e], old[b:e], dz[b:e], row_begin=b, grad_loss=gl)
    loss, stats = ctx.loss_finalize()
    ctx.get_error()
    out = dict(loss=float(loss.item()), stats=stats_to_dict(stats),
               dlogits=dz.float().cpu().numpy(),
               tok={k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()},
               rol={k: v.cpu().numpy() for k, v in ctx.export_rollout_stats().items()})
    out["zv_out"] = out["rol"]["zv"]
    ctx.close()
    return out


def check_vs_oracle(g, inst, cfg, rtol=1e-5, grad_loss=1.0):
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, rtol)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T), grad_loss))


@pytest.mark.parametrize("cfgkw", [{}, {"norm": O.NORM_TOKEN}, {"zv_mode": O.ZV_RLZVP}],
                         ids=["default", "token_norm", "rlzvp"])
def test_single_pass_equals_two_sweeps_and_oracle(cfgkw):
    dev = require_cuda()
    inst = workload_instance("C0")
    chunks = [(11, 16), (0, 3), (4, 11), (3, 4)]          # out of order, ragged
    g = run_single(inst, dev, chunks, cfgkw)
    two = run_gpu(inst, dev, cfgkw)
    assert g["loss"] == two["loss"]
    assert np.array_equal(g["dlogits"], two["dlogits"])
    okw = {k: v for k, v in cfgkw.items()}
    check_vs_oracle(g, inst, oracle_cfg(inst.V, **okw))


def test_single_pass_variable_lengths_empty_rollouts_bf16_in_place():
    dev = require_cuda()
    lengths = [7, 0, 12, 5, 9, 0, 3, 11, 6, 0]
    inst = tiny_instance(61, V=1544, group_sizes=(4, 3, 3), lengths=lengths, dtype="bf16",
                         mask_tail=3)
    chunks = [(0, 2), (2, 3), (3, 7), (7, 10)]
    g = run_single(inst, dev, chunks, logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16,
                   in_place=True, grad_loss=0.5)
    two = run_gpu(inst, dev, logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16,
                  in_place=True, grad_loss=0.5)
    assert g["loss"] == two["loss"]
    assert np.array_equal(g["dlogits"], two["dlogits"])


def test_single_pass_rejects_misaligned_chunks_and_mixed_calls():
    from paper_2512_07710_b200.espo import Espo, EspoError
    dev = require_cuda()
    inst = workload_instance("C0")
    T, V = inst.T, inst.V
    z = to_dev(inst.logits, torch.float32, dev)
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
    # fwd_bwd before set_mask; set_mask after a forward chunk
    ctx.prepare(*args, n_tokens=T)
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd_bwd(z[:64], tok[:64], old[:64])
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    ctx.loss_fwd(z[:64], tok[:64], old[:64])
    with pytest.raises(EspoError) as e:
        ctx.set_mask()
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    # two-sweep calls in single-pass mode
    ctx.prepare(*args, n_tokens=T)
    ctx.set_mask()
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd(z, tok, old)
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd_partial(z, tok, old)
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    hb = torch.zeros((T, 64), dtype=torch.bfloat16, device=dev)
    Wb = torch.zeros((V, 64), dtype=torch.bfloat16, device=dev)
    with pytest.raises(EspoError) as e:
        ctx.lmhead_fwd(hb, Wb, tok, old)
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    ctx.loss_fwd_bwd(z, tok, old)
    ctx.loss_finalize()
    with pytest.raises(EspoError) as e:
        ctx.loss_bwd(z)
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    ctx.get_error()
    # a chunk ending inside a rollout: device-detected
    ctx.prepare(*args, n_tokens=T)
    ctx.set_mask()
    ctx.loss_fwd_bwd(z[:100], tok[:100], old[:100])
    with pytest.raises(EspoError) as e:
        ctx.get_error()
    assert e.value.code == "ESPO_ERR_INVALID_ARGUMENT"
    ctx.close()


@pytest.mark.parametrize("cfgkw,dtype", [
    ({"zero_fill_inactive_rows": False}, "bf16"),
    ({"zv_mode": O.ZV_RLZVP, "norm": O.NORM_TOKEN}, "bf16"),
    ({"partition": O.PARTITION_SINGLETON,
      "ratio_mode": O.RATIO_LITERAL_OLD}, "f32"),
    ({"n_buckets": 3, "logit_scale": 1.3}, "f32"),
], ids=["compact_bf16", "rlzvp_token_bf16", "singleton_literal_f32", "k3_lambda_f32"])
def test_single_pass_config_matrix(cfgkw, dtype):
    """Single-pass ≡ two sweeps, bitwise, across modes (compact output, RL-ZVP + TOKEN
    normalisation, singleton partition with the literal ratio, K = 3 with a temperature)."""
    dev = require_cuda()
    inst = tiny_instance(71, V=2056, group_sizes=(4, 3, 4), L=21, mask_tail=4,
                         dtype=dtype, rewards=[1, 0, 1, 1, 1, 1, 1, 0, 0, 1, 0],
                         logit_scale=cfgkw.get("logit_scale", 1.0))
    kw = dict(cfgkw=cfgkw)
    if dtype == "bf16":
        kw.update(logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16)
    chunks = [(7, 11), (0, 2), (2, 7)]
    g = run_single(inst, dev, chunks, grad_loss=1.7, **kw)
    two = run_gpu(inst, dev, grad_loss=1.7, **kw)
    assert g["loss"] == two["loss"]
    assert np.array_equal(g["dlogits"], two["dlogits"], equal_nan=True)
