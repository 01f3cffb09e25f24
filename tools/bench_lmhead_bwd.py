"""Fused LM head + ESPO forward AND backward (espo_lmhead_fwd → finalize → espo_lmhead_bwd:
tcgen05 recompute with the bf16 dz epilogue, then dh = dz·W and dW += dzᵀ·h) vs the unfused
pipeline on the same data (torch.matmul logits in bf16 → espo_loss_fwd/bwd in place →
torch.matmul dh and dW) vs the factored pipeline (torch.matmul logits → espo_loss_fwd_factored
in place, G = onehot − p → espo_loss_row_scale s → dh = diag(s)·(G·W), dW += Gᵀ·(diag(s)·h):
each logits row is read once). One chunk of n rows, V = 151,936. Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07710_b200.espo import Espo  # noqa: E402


def main(d=4096, n=16384, V=151936, iters=3, realistic=False):
    """realistic=False: one prompt group of 8 rollouts with rewards [1,0,…] and old_logp within
    0.02 of the policy (every row carries gradient — the dense case). realistic=True: the C1
    reward and drift recipe (bench.py): groups of 8 rollouts with Bernoulli(p ~ U(0,1)) rewards
    (≈22 % zero-variance groups), old_logp = lp + b_i + 0.02·n_t with b_i ~ N(0, 0.04) per
    rollout (≈1/3 of active tokens clipped) — rows without gradient are then skipped by the
    fused backward."""
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    # realistic: logits std ≈ 7 (peaked next-token distributions, entropy ~1 nat, so Eq. 3's
    # ε_τ is small and drifted rollouts clip) and tokens sampled from softmax (Gumbel-max)
    h = (torch.randn(n, d, device=dev) / d ** 0.5 * (7 if realistic else 3)).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev).to(torch.bfloat16)
    if realistic:
        tokens = torch.empty(n, dtype=torch.int32, device=dev)
        for r0 in range(0, n, 2048):
            z = torch.matmul(h[r0:r0 + 2048], W.T).float()
            g = -torch.log(-torch.log(torch.rand_like(z).clamp_min(1e-20)))
            tokens[r0:r0 + 2048] = (z + g).argmax(1).to(torch.int32)
            del z, g
    else:
        tokens = torch.randint(0, V, (n,), device=dev, dtype=torch.int32)
    G = 8
    if realistic:
        import numpy as np
        R = 8 * max(1, n // 4096)                 # rollouts of 4096 / (n/R) tokens
        rng = np.random.default_rng(1)
        rw = np.concatenate([(rng.uniform(size=8) < rng.uniform()).astype(np.float32)
                             for _ in range(R // 8)])
        rewards = torch.from_numpy(rw).to(dev)
        gid = torch.from_numpy(np.repeat(np.arange(R // 8, dtype=np.int32), 8)).to(dev)
        so = torch.arange(R + 1, device=dev, dtype=torch.int64) * (n // R)
    else:
        rewards = torch.tensor([1.0, 0.0] * (G // 2), device=dev)
        gid = torch.zeros(G, dtype=torch.int32, device=dev)
        so = torch.arange(G + 1, device=dev, dtype=torch.int64) * (n // G)
    fctx = Espo(V, logits_dtype=torch.bfloat16, device=0)
    uctx = Espo(V, logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16, device=0)
    # rollout log-probs near the current policy's (untimed): old = lp + N(0, 0.02²), so the
    # clip fraction is realistic (a constant old_logp would clip nearly every token)
    uctx.prepare(rewards, gid, so, n_tokens=n)
    uctx.loss_fwd(torch.matmul(h, W.T), tokens, torch.zeros(n, device=dev))
    uctx.loss_finalize()
    old = (uctx.export_token_stats()["lp"] + 0.02 * torch.randn(n, device=dev)).contiguous()
    if realistic:                                  # + per-rollout drift b_i ~ N(0, 0.04)
        R = int(so.numel()) - 1
        old = (old + torch.repeat_interleave(0.04 * torch.randn(R, device=dev),
                                             torch.diff(so))).contiguous()
    xctx = Espo(V, logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16, device=0)
    dh = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
    dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
    sc = torch.empty(n, dtype=torch.float32, device=dev)

    def fused():
        fctx.prepare(rewards, gid, so, n_tokens=n)
        fctx.lmhead_fwd(h, W, tokens, old)
        fctx.loss_finalize()
        fctx.lmhead_bwd(h, W, dh, dW)

    def unfused():
        uctx.prepare(rewards, gid, so, n_tokens=n)
        z = torch.matmul(h, W.T)
        uctx.loss_fwd(z, tokens, old)
        uctx.loss_finalize()
        uctx.loss_bwd(z, z)                       # in place: z becomes dz (bf16)
        torch.matmul(z, W, out=dh)
        dW.add_(torch.matmul(z.T, h))             # bf16 GEMM, fp32 accumulate into dW

    def factored():
        xctx.prepare(rewards, gid, so, n_tokens=n)
        z = torch.matmul(h, W.T)
        xctx.loss_fwd_factored(z, tokens, old, grad=z)   # in place: z becomes G (bf16)
        xctx.loss_finalize()
        xctx.loss_row_scale(out=sc)
        torch.matmul(z, W, out=dh)
        dh.mul_(sc[:, None])                              # dh = diag(s)·(G·W)
        dW.add_(torch.matmul(z.T, h * sc[:, None].to(h.dtype)))   # dW += Gᵀ·(diag(s)·h)

    # agreement of the three backward results on one pass (dW from zero)
    outs = {}
    for name, fn in (("fused", fused), ("unfused", unfused), ("factored", factored)):
        dW.zero_()
        fn()
        torch.cuda.synchronize()
        outs[name] = (dh.float().clone(), dW.clone())
    agree = {}
    for name in ("fused", "factored"):
        a, b = outs[name], outs["unfused"]
        agree[name] = {"dh_rel_err": float((a[0] - b[0]).norm() / b[0].norm()),
                       "dW_rel_err": float((a[1] - b[1]).norm() / b[1].norm())}
    del outs

    res = {}
    for name, fn in (("fused", fused), ("unfused", unfused), ("factored", factored)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        res[name] = {"ms": ms, "tokens_per_s": n / (ms * 1e-3),
                     "model_TFLOPs": 6.0 * n * V * d / (ms * 1e-3) / 1e12}
    fctx.get_error()
    uctx.get_error()
    xctx.get_error()
    res["agreement_vs_unfused"] = agree
    # fused backward alone (recompute + dz + 2 GEMMs): the library's tcgen05 GEMMs (0), cuBLAS
    # GEMMs (ESPO_OPT_LMHEAD_BWD_GEMM = 1) and one-CTA tiles (2), interleaved over 3 rounds
    # with a warm-up call each (medians), so no setting inherits another's thermal state
    from paper_2512_07710_b200.espo import OPT_LMHEAD_BWD_GEMM
    fctx.prepare(rewards, gid, so, n_tokens=n)
    fctx.lmhead_fwd(h, W, tokens, old)
    fctx.loss_finalize()
    fctx.set_option(OPT_LMHEAD_BWD_GEMM, 1)
    dh2, dW2 = torch.empty_like(dh), torch.zeros_like(dW)
    fctx.lmhead_bwd(h, W, dh2, dW2)
    dW.zero_()
    fctx.set_option(OPT_LMHEAD_BWD_GEMM, 0)
    fctx.lmhead_bwd(h, W, dh, dW)
    torch.cuda.synchronize()
    res["native_vs_cublas"] = {"dh_rel": float((dh.float() - dh2.float()).norm() / dh2.float().norm()),
                               "dW_rel": float((dW - dW2).norm() / dW2.norm())}
    del dh2, dW2
    import statistics
    times = {0: [], 1: [], 2: []}
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        for g in (0, 1, 2):
            fctx.set_option(OPT_LMHEAD_BWD_GEMM, g)
            fctx.lmhead_bwd(h, W, dh, dW)
            torch.cuda.synchronize()
            s.record()
            for _ in range(iters):
                fctx.lmhead_bwd(h, W, dh, dW)
            e.record()
            torch.cuda.synchronize()
            times[g].append(s.elapsed_time(e) / iters)
    fctx.set_option(OPT_LMHEAD_BWD_GEMM, 0)
    for g, key in ((0, "fused_bwd_only"), (1, "fused_bwd_only_cublas"), (2, "fused_bwd_only_1cta")):
        ms = statistics.median(times[g])
        res[key] = {"ms": ms, "TFLOPs_3gemm": 6.0 * n * V * d / (ms * 1e-3) / 1e12,
                    "rounds_ms": times[g]}
    res["fused_bwd_only"]["gemm"] = "tcgen05 (k_gemm.cuh)"
    uctx.prepare(rewards, gid, so, n_tokens=n)
    uctx.loss_fwd(torch.matmul(h, W.T), tokens, old)
    from paper_2512_07710_b200.espo import stats_to_dict
    st = stats_to_dict(uctx.loss_finalize()[1])
    res["clipped_fraction"] = st["n_clipped_tokens"] / max(st["n_active_tokens"], 1)
    res["rows_with_gradient"] = (st["n_active_tokens"] - st["n_clipped_tokens"]) / n
    res["zv_groups"] = st["n_zv_groups"]
    res["config"] = {"n": n, "V": V, "d": d, "realistic": realistic,
                     "model_flops": "6·n·V·d (fwd logits GEMM + dh + dW GEMMs)"}
    print(json.dumps(res))


if __name__ == "__main__":
    main(d=int(sys.argv[1]) if len(sys.argv) > 1 else 4096,
         n=int(sys.argv[2]) if len(sys.argv) > 2 else 16384,
         realistic=len(sys.argv) > 3 and sys.argv[3] == "realistic")
