"""One espo_lmhead_bwd call (after a warm-up call) on synthetic h, W — the target of the
ncu launch list / full captures of the backward's kernels (k_lmhead_dz, k_umma_gemm).
usage: python tools/lmhead_bwd_once.py [d] [n] [gemm: 0 pair | 1 cuBLAS | 2 one CTA] [sync]
       [group option] [hints option]   (ESPO_OPT_GEMM_GROUP_M / _GEMM_HINTS; -1 = default)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07710_b200.espo import (OPT_GEMM_GROUP_M, OPT_GEMM_HINTS, OPT_GEMM_SYNC,  # noqa: E402
                                        OPT_LMHEAD_BWD_GEMM, Espo)


def main(d=4096, n=8192, gemm=0, sync=-1, group=-1, hints=-1, V=151936):
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    h = (torch.randn(n, d, device=dev) / d ** 0.5 * 3).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev).to(torch.bfloat16)
    tokens = torch.randint(0, V, (n,), device=dev, dtype=torch.int32)
    G = 8
    rewards = torch.tensor([1.0, 0.0] * (G // 2), device=dev)
    gid = torch.zeros(G, dtype=torch.int32, device=dev)
    so = torch.arange(G + 1, device=dev, dtype=torch.int64) * (n // G)
    ctx = Espo(V, logits_dtype=torch.bfloat16, device=0)
    ctx.set_option(OPT_LMHEAD_BWD_GEMM, gemm)
    ctx.set_option(OPT_GEMM_SYNC, sync)
    if group >= 0:
        ctx.set_option(OPT_GEMM_GROUP_M, group)
    ctx.set_option(OPT_GEMM_HINTS, hints)
    ctx.prepare(rewards, gid, so, n_tokens=n)
    ctx.lmhead_fwd(h, W, tokens, torch.zeros(n, device=dev))
    ctx.loss_finalize()
    old = (ctx.export_token_stats()["lp"] + 0.02 * torch.randn(n, device=dev)).contiguous()
    ctx.prepare(rewards, gid, so, n_tokens=n)
    ctx.lmhead_fwd(h, W, tokens, old)
    ctx.loss_finalize()
    dh = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
    dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
    for _ in range(2):
        ctx.lmhead_bwd(h, W, dh, dW)
    torch.cuda.synchronize()
    ctx.get_error()
    print("ok", flush=True)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
