"""GPU edge cases and error behaviour of the C ABI: eliminated groups,
G=1, empty and fully-masked rollouts, −inf logits, extreme log-probs (slow path), sticky
device errors, host-side validation, and the P3 elimination invariant."""
import numpy as np
import pytest
import torch

from paper_2512_07710_b200.espo import Espo, EspoError
from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import (check_dlogits_f32, check_exact_fields, check_loss,
                              check_token_stats, decision_aware_reference, oracle_cfg,
                              oracle_dlogits, require_cuda, run_gpu, to_dev)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return require_cuda()


def parity(inst, dev, **kw):
    g = run_gpu(inst, dev, **kw)
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))
    return g, ref2


def test_all_zv_batch_is_zero(dev):
    inst = tiny_instance(1, V=256, group_sizes=(3, 2, 1), L=10, rewards=[1, 1, 1, 0, 0, 0.25])
    g = run_gpu(inst, dev)
    assert g["loss"] == 0.0
    assert g["stats"]["n_active_rollouts"] == 0 and g["stats"]["n_zv_groups"] == 3
    assert not np.any(g["dlogits"])


def test_singletons_empty_and_masked_rollouts(dev):
    inst = tiny_instance(2, V=512, group_sizes=(1, 4, 3), lengths=[5, 0, 7, 6, 9, 3, 0, 4],
                         mask_tail=2)
    inst.mask[inst.seq_offsets[3]:inst.seq_offsets[4]] = 0   # rollout 3 fully masked
    g, ref = parity(inst, dev)
    assert not ref.active[0] and not ref.active[1] and not ref.active[3]


def test_minus_inf_logits_are_legal(dev):
    inst = tiny_instance(3, V=1024, group_sizes=(4, 4), L=16)
    rng = np.random.default_rng(0)
    inst.logits[:, 1000:] = -np.inf                     # padded vocabulary
    for t in range(inst.T):
        cols = rng.choice(1000, size=20, replace=False)
        cols = cols[cols != inst.tokens[t]]
        inst.logits[t, cols] = -np.inf
    inst.tokens = np.minimum(inst.tokens, 999)
    inst.logits[np.arange(inst.T), inst.tokens] = np.maximum(
        inst.logits[np.arange(inst.T), inst.tokens], -5.0)
    parity(inst, dev)


def test_extreme_logprob_slow_path(dev):
    """Target logit 90 below the row max (lp ≈ −90): the fast path's reference overflows,
    the batch is recomputed with a max-based reference."""
    inst = tiny_instance(4, V=2048, group_sizes=(4, 4), L=8, sigma_seq=0.0, sigma_tok=0.0)
    for t in range(0, inst.T, 3):
        inst.logits[t, inst.tokens[t]] = inst.logits[t].max() - 90.0
    from tests._instances import exact_lp
    import espo_synth as S
    inst.old_logp = S.drift_old_logp(exact_lp(inst.logits, inst.tokens), inst.seq_offsets, 4)
    g, ref = parity(inst, dev)
    assert np.nanmin(ref.lp) < -85


def test_elimination_invariant_nan_rows_never_read(dev):
    inst = workload_instance("C0")
    a = run_gpu(inst, dev)
    ref = inst.run(oracle_cfg(inst.V))
    bad = inst.logits.copy()
    for i in range(inst.R):
        if ref.zv[i]:
            bad[inst.seq_offsets[i]:inst.seq_offsets[i + 1]] = np.nan
    bad[inst.mask == 0] = np.nan
    inst.logits = bad
    b = run_gpu(inst, dev)      # get_error inside run_gpu raises if any NaN row was read
    assert a["loss"] == b["loss"] and a["stats"] == b["stats"]
    keep = ~np.isnan(bad).any(axis=1)
    assert np.array_equal(a["dlogits"][keep], b["dlogits"][keep])
    assert not np.any(b["dlogits"][~keep])


def _ctx_with(inst, dev, dtype=torch.float32):
    ctx = Espo(inst.V, logits_dtype=dtype, device=dev.index)
    z = to_dev(inst.logits, torch.float32, dev).to(dtype)
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    return ctx, z, tok, old, args


@pytest.mark.parametrize("bad,code", [(np.nan, "ESPO_ERR_NONFINITE_INPUT"),
                                      (np.inf, "ESPO_ERR_NONFINITE_INPUT")])
def test_nonfinite_logit_sets_sticky_error(dev, bad, code):
    inst = tiny_instance(5, V=512, group_sizes=(4,), L=6)
    inst.logits[3, 7 if inst.tokens[3] != 7 else 8] = bad
    ctx, z, tok, old, args = _ctx_with(inst, dev)
    ctx.prepare(*args, n_tokens=inst.T)
    ctx.loss_fwd(z, tok, old)
    loss, _ = ctx.loss_finalize()
    with pytest.raises(EspoError) as e:
        ctx.get_error()
    assert e.value.code == code
    assert np.isnan(loss.item())


def test_target_minus_inf_and_token_range(dev):
    inst = tiny_instance(6, V=512, group_sizes=(4,), L=6)
    inst.logits[2, inst.tokens[2]] = -np.inf
    ctx, z, tok, old, args = _ctx_with(inst, dev)
    ctx.prepare(*args, n_tokens=inst.T)
    ctx.loss_fwd(z, tok, old)
    ctx.loss_finalize()
    with pytest.raises(EspoError) as e:
        ctx.get_error()
    assert e.value.code == "ESPO_ERR_NONFINITE_INPUT"
    inst = tiny_instance(6, V=512, group_sizes=(4,), L=6)
    inst.tokens[5] = 512
    ctx, z, tok, old, args = _ctx_with(inst, dev)
    ctx.prepare(*args, n_tokens=inst.T)
    ctx.loss_fwd(z, tok, old)
    ctx.loss_finalize()
    with pytest.raises(EspoError) as e:
        ctx.get_error()
    assert e.value.code == "ESPO_ERR_TOKEN_OUT_OF_RANGE"


def test_device_detected_group_and_reward_errors(dev):
    inst = tiny_instance(7, V=256, group_sizes=(2, 2), L=4)
    ctx, z, tok, old, (r, gid, so) = _ctx_with(inst, dev)
    gid = torch.tensor([0, 1, 0, 1], dtype=torch.int32, device=dev)
    ctx.prepare(r, gid, so, n_tokens=inst.T)
    with pytest.raises(EspoError) as e:
        ctx.get_error()
    assert e.value.code == "ESPO_ERR_GROUPS_NOT_CONTIGUOUS"
    r2 = r.clone()
    r2[1] = float("nan")
    ctx.prepare(r2, to_dev(inst.group_ids, torch.int32, dev), so, n_tokens=inst.T)
    with pytest.raises(EspoError) as e:
        ctx.get_error()
    assert e.value.code == "ESPO_ERR_NONFINITE_INPUT"
    ctx.prepare(r, to_dev(inst.group_ids, torch.int32, dev), so, n_tokens=inst.T + 1)
    with pytest.raises(EspoError) as e:
        ctx.get_error()
    assert e.value.code == "ESPO_ERR_INVALID_ARGUMENT"


def test_host_validation_and_call_order(dev):
    inst = tiny_instance(8, V=256, group_sizes=(2, 2), L=8)
    ctx, z, tok, old, args = _ctx_with(inst, dev)
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd(z, tok, old)                      # before prepare
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    ctx.prepare(*args, n_tokens=inst.T)
    with pytest.raises(EspoError) as e:
        ctx.loss_finalize()                            # rows not covered
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    with pytest.raises(EspoError) as e:
        ctx.loss_bwd(z)                                # before finalize
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    raw = torch.zeros(inst.T * inst.V + 1, dtype=torch.float32, device=dev)
    mis = raw[1:].view(inst.T, inst.V)
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd(mis, tok, old)                    # 4-byte aligned only
    assert e.value.code == "ESPO_ERR_ALIGNMENT"
    ctx.loss_fwd(z[:10], tok[:10], old[:10], row_begin=0)
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd(z[5:12], tok[5:12], old[5:12], row_begin=5)   # overlap
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd(z[10:], tok[10:], old[10:], row_begin=inst.T)  # out of range
    assert e.value.code == "ESPO_ERR_INVALID_ARGUMENT"
    ctx.loss_fwd(z[10:], tok[10:], old[10:], row_begin=10)
    ctx.loss_finalize()
    ctx.loss_bwd(z)
    ctx.get_error()
    ctx.close()
