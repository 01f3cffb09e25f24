"""Fused LM head + ESPO forward AND backward (espo_lmhead_fwd → finalize → espo_lmhead_bwd:
tcgen05 recompute with the bf16 dz epilogue, then dh = dz·W and dW += dzᵀ·h) vs the unfused
pipeline on the same data (torch.matmul logits in bf16 → espo_loss_fwd/bwd in place →
torch.matmul dh and dW). One chunk of n rows, V = 151,936. Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07710_b200.espo import Espo  # noqa: E402


def main(d=4096, n=16384, V=151936, iters=3):
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    h = (torch.randn(n, d, device=dev) / d ** 0.5 * 3).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev).to(torch.bfloat16)
    tokens = torch.randint(0, V, (n,), device=dev, dtype=torch.int32)
    old = torch.full((n,), -1.0, device=dev)
    G = 8
    rewards = torch.tensor([1.0, 0.0] * (G // 2), device=dev)
    gid = torch.zeros(G, dtype=torch.int32, device=dev)
    so = torch.arange(G + 1, device=dev, dtype=torch.int64) * (n // G)
    fctx = Espo(V, logits_dtype=torch.bfloat16, device=0)
    uctx = Espo(V, logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16, device=0)
    dh = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
    dW = torch.zeros((V, d), dtype=torch.float32, device=dev)

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

    res = {}
    for name, fn in (("fused", fused), ("unfused", unfused)):
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
    # fused backward alone (recompute + dz + 2 GEMMs)
    fctx.prepare(rewards, gid, so, n_tokens=n)
    fctx.lmhead_fwd(h, W, tokens, old)
    fctx.loss_finalize()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fctx.lmhead_bwd(h, W, dh, dW)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    res["fused_bwd_only"] = {"ms": ms, "TFLOPs_3gemm": 6.0 * n * V * d / (ms * 1e-3) / 1e12}
    res["config"] = {"n": n, "V": V, "d": d,
                     "model_flops": "6·n·V·d (fwd logits GEMM + dh + dW GEMMs)"}
    print(json.dumps(res))


if __name__ == "__main__":
    main(d=int(sys.argv[1]) if len(sys.argv) > 1 else 4096,
         n=int(sys.argv[2]) if len(sys.argv) > 2 else 16384)
