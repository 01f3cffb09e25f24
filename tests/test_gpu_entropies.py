"""Caller-supplied selection entropies (espo_set_entropies; reading Q4's alternative,
SPEC.md:460 — the rollout policy's entropies pick the buckets and set Eq. 3's ε_τ).

Against the oracle run with the same entropies (`espo_loss(entropy=...)`): exact fields,
token statistics (still the sweep's), bucket decisions bit for bit (both sides split the same
fp32 values), loss and dlogits at the usual tolerances; in RL-ZVP mode the token advantages
use the supplied entropies too. Supplying the sweep's own entropies reproduces the default
run bit for bit. Coverage, overlap, value and mode errors."""
import numpy as np
import pytest
import torch

from oracle import espo_oracle as O
from tests._instances import workload_instance
from tests.gpu_common import (check_dlogits_f32, check_exact_fields, check_loss,
                              check_token_stats, decision_aware_reference, oracle_cfg,
                              oracle_dlogits, require_cuda, run_gpu, to_dev)

pytestmark = pytest.mark.gpu


def _entropies(T, seed):
    """Rollout-engine-like entropies: lognormal, a few exact ties and zeros (and a −0)."""
    rng = np.random.default_rng(seed)
    e = rng.lognormal(-0.5, 1.0, T).astype(np.float32)
    e[rng.choice(T, T // 10, replace=False)] = np.float32(0.75)
    e[rng.choice(T, T // 20, replace=False)] = np.float32(0.0)
    e[3] = np.float32(-0.0)
    return e


@pytest.mark.parametrize("zv_mode", ["mask", "rlzvp"])
def test_supplied_entropies_match_oracle(zv_mode):
    dev = require_cuda()
    inst = workload_instance("C0")
    kw = {} if zv_mode == "mask" else dict(zv_mode=O.ZV_RLZVP, zvp_beta=0.2)
    e = _entropies(inst.T, 5)
    T = inst.T
    g = run_gpu(inst, dev, cfgkw=kw, chunks=[(300, T), (0, 300)], entropy=e,
                entropy_chunks=[(500, T), (0, 137), (137, 500)])
    cfg = oracle_cfg(inst.V, **kw)
    ref = inst.run(cfg, entropy=e)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)                  # exported lse / lp / H / q: the sweep's own
    v = ref.kappa >= 0
    assert np.array_equal(g["tok"]["bucket"][v].astype(np.int64), ref.bucket[v])
    ref2, _ = decision_aware_reference(g, inst, ref, cfg, entropy=e)
    check_loss(g, ref2, 1e-5)
    dc = np.abs(g["tok"]["coef"].astype(np.float64) - ref2.coef)
    assert np.all(dc[v] <= 1e-5 * np.abs(ref2.coef[v]) + 1e-12)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(T)))
    assert g["stats"]["mean_entropy"] == pytest.approx(ref.stats["mean_entropy"], rel=1e-6)
    base = inst.run(cfg)                       # the supplied entropies changed the split
    assert not np.array_equal(base.bucket[v], ref.bucket[v])


def test_supplying_the_sweeps_entropies_is_the_default():
    dev = require_cuda()
    inst = workload_instance("C0")
    a = run_gpu(inst, dev)
    H = a["tok"]["H"].astype(np.float32)
    H[~a["tok"]["valid"].astype(bool)] = 1.0   # rows never read: any value
    b = run_gpu(inst, dev, entropy=H)
    assert b["loss"] == a["loss"]
    assert np.array_equal(b["dlogits"], a["dlogits"])
    assert np.array_equal(b["tok"]["bucket"], a["tok"]["bucket"])


def test_supplied_entropies_errors():
    from paper_2512_07710_b200.espo import Espo, EspoError
    dev = require_cuda()
    inst = workload_instance("C0")
    T, V = inst.T, inst.V
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    z = to_dev(inst.logits, torch.float32, dev)
    tok, old = to_dev(inst.tokens, torch.int32, dev), to_dev(inst.old_logp, torch.float32, dev)
    e = torch.ones(T, dtype=torch.float32, device=dev)
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)

    def fresh():
        ctx.prepare(*args, n_tokens=T)
        ctx.get_error()

    fresh()                                    # partial coverage → finalize refuses
    ctx.set_entropies(e[:100])
    ctx.loss_fwd(z, tok, old)
    with pytest.raises(EspoError, match="BAD_STATE"):
        ctx.loss_finalize()
    fresh()                                    # overlapping chunks
    ctx.set_entropies(e[:100])
    with pytest.raises(EspoError, match="BAD_STATE"):
        ctx.set_entropies(e[50:150], row_begin=50)
    with pytest.raises(EspoError, match="INVALID_ARGUMENT"):
        ctx.set_entropies(e[:10], row_begin=T - 5)          # past T
    for bad, code in ((-0.5, "INVALID_ARGUMENT"), (float("nan"), "NONFINITE"),
                      (float("inf"), "NONFINITE")):
        fresh()
        x = e.clone()
        x[7] = bad
        ctx.set_entropies(x)
        with pytest.raises(EspoError, match=code):
            ctx.get_error()
    fresh()                                    # single-pass mode: either order refused
    ctx.set_entropies(e)
    with pytest.raises(EspoError, match="UNSUPPORTED"):
        ctx.set_mask(None)
    fresh()
    ctx.set_mask(None)
    with pytest.raises(EspoError, match="UNSUPPORTED"):
        ctx.set_entropies(e)
    ctx.close()
