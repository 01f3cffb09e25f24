"""The PyTorch integration: EspoLossFunction inside an autograd graph (logits = h·Wᵀ computed
by torch, loss scaled by 2 after the ESPO node) must give torch the same dW and dh as the
oracle's chain rule (O9) with grad_loss = 2; espo_loss (the single-chunk convenience) must
equal the explicit calls."""
import numpy as np
import pytest
import torch

import espo_synth as S
from oracle import espo_oracle as O
from tests._instances import Instance
from tests.gpu_common import oracle_cfg, require_cuda, to_dev

pytestmark = pytest.mark.gpu


def test_autograd_function_through_lm_head():
    from paper_2512_07710_b200.espo import Espo, EspoLossFunction
    dev = require_cuda()
    torch.backends.cuda.matmul.allow_tf32 = False
    rng = np.random.default_rng(4)
    ng, G, L, V, d = 3, 4, 24, 700, 48
    R, T = ng * G, ng * G * L
    h = rng.standard_normal((T, d))
    W = rng.standard_normal((V, d)) * 0.7
    z64 = h @ W.T
    tokens = S.sample_tokens_gumbel(z64.astype(np.float32), 4)
    gid = np.repeat(np.arange(ng, dtype=np.int32), G)
    so = np.arange(R + 1, dtype=np.int64) * L
    rewards = np.array([1, 0, 1, 1, 1, 1, 1, 1, 0, 0, 1, 0], np.float32)   # group 1 is ZV
    lp = np.array([O.row_stats(z64[t], int(tokens[t]))[1] for t in range(T)])
    old = S.drift_old_logp(lp, so, 4)
    mask = np.ones(T, np.uint8)
    mask[L - 4:L] = 0

    ht = torch.tensor(h, device=dev, requires_grad=True)
    Wt = torch.tensor(W, device=dev, requires_grad=True)
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
    logits = (ht @ Wt.T).float()                 # torch computes the LM head in fp64 → f32
    loss = EspoLossFunction.apply(logits, ctx, to_dev(tokens, torch.int32, dev),
                                  to_dev(old, torch.float32, dev), to_dev(rewards, torch.float32, dev),
                                  to_dev(gid, torch.int32, dev), to_dev(so, torch.int64, dev),
                                  to_dev(mask, torch.uint8, dev))
    (2.0 * loss).backward()
    ctx.get_error()
    got_dh, got_dW = ht.grad.cpu().numpy(), Wt.grad.cpu().numpy()
    ctx.close()

    z32 = (torch.tensor(h) @ torch.tensor(W).T).float().numpy()   # the logits the GPU saw
    inst = Instance(z32, tokens, old, mask, rewards, gid, so, V)
    cfg = oracle_cfg(V)
    ref = inst.run(cfg)
    assert float(loss.item()) == pytest.approx(ref.loss, rel=1e-5, abs=1e-7)
    dz, dh, dW = O.lmhead_grads(ref, h, W, tokens, cfg, grad_loss=2.0)
    # the GPU's fp32 dz carries ≤ 1e-5 relative error per row; the fp64 GEMMs add nothing
    for got, want in ((got_dh, dh), (got_dW, dW)):
        assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want) + 1e-12
    assert np.all(got_dh[L - 4:L] == 0) and np.all(got_dh[G * L:2 * G * L] == 0)


def test_espo_loss_convenience_matches_calls():
    from paper_2512_07710_b200.espo import Espo, espo_loss
    from tests._instances import workload_instance
    from tests.gpu_common import run_gpu
    dev = require_cuda()
    inst = workload_instance("C0")
    ctx = Espo(inst.V, logits_dtype=torch.float32, device=dev.index)
    z = to_dev(inst.logits, torch.float32, dev)
    loss, stats, dz = espo_loss(ctx, z, to_dev(inst.tokens, torch.int32, dev),
                                to_dev(inst.old_logp, torch.float32, dev),
                                to_dev(inst.rewards, torch.float32, dev),
                                to_dev(inst.group_ids, torch.int32, dev),
                                to_dev(inst.seq_offsets, torch.int64, dev),
                                mask=to_dev(inst.mask, torch.uint8, dev))
    ctx.get_error()
    u = run_gpu(inst, dev)
    assert float(loss.item()) == u["loss"]
    assert np.array_equal(dz.cpu().numpy(), u["dlogits"])
    ctx.close()
