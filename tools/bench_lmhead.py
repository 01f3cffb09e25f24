"""Throughput of the fused LM head + ESPO forward (espo_lmhead_fwd) vs cuBLAS for the same
GEMM (torch.matmul, bf16 → bf16 logits), one 32,768-row chunk (one C1 prompt group), V=151,936."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07710_b200.espo import Espo  # noqa: E402


def main(d=4096, n=32768, V=151936, iters=5, parts=0, two_cta=0):
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
    ctx = Espo(V, logits_dtype=torch.bfloat16, device=0)
    ctx.set_option(3, parts)
    ctx.set_option(5, two_cta)

    def fused():
        ctx.prepare(rewards, gid, so, n_tokens=n)
        ctx.lmhead_fwd(h, W, tokens, old)
        ctx.loss_finalize()

    def cublas():
        return torch.matmul(h, W.T)

    res = {}
    for name, fn in (("fused_lmhead_fwd", fused), ("cublas_matmul_bf16", cublas)):
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
        res[name] = {"ms": ms, "TFLOPs": 2.0 * n * V * d / (ms * 1e-3) / 1e12,
                     "tokens_per_s": n / (ms * 1e-3)}
    ctx.get_error()
    res["config"] = {"n": n, "V": V, "d": d, "parts": parts or "auto", "two_cta": two_cta}
    print(json.dumps(res))


if __name__ == "__main__":
    main(d=int(sys.argv[1]) if len(sys.argv) > 1 else 4096,
         parts=int(sys.argv[2]) if len(sys.argv) > 2 else 0,
         two_cta=int(sys.argv[3]) if len(sys.argv) > 3 else 0)
