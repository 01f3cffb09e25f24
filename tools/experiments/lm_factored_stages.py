"""Stage times of the unfused and factored LM-head backward pipelines (n = 16,384, d = 4096)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2512_07710_b200.espo import Espo  # noqa: E402

d, n, V = int(sys.argv[1]) if len(sys.argv) > 1 else 4096, 16384, 151936
dev = torch.device("cuda", 0)
torch.manual_seed(0)
h = (torch.randn(n, d, device=dev) / d ** 0.5 * 3).to(torch.bfloat16)
W = torch.randn(V, d, device=dev).to(torch.bfloat16)
tokens = torch.randint(0, V, (n,), device=dev, dtype=torch.int32)
G = 8
rewards = torch.tensor([1.0, 0.0] * (G // 2), device=dev)
gid = torch.zeros(G, dtype=torch.int32, device=dev)
so = torch.arange(G + 1, device=dev, dtype=torch.int64) * (n // G)
ctx = Espo(V, logits_dtype=torch.bfloat16, grad_dtype=torch.bfloat16, device=0)
dh = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
sc = torch.empty(n, dtype=torch.float32, device=dev)
z = torch.empty((n, V), dtype=torch.bfloat16, device=dev)
ctx.prepare(rewards, gid, so, n_tokens=n)
ctx.loss_fwd(torch.matmul(h, W.T), tokens, torch.zeros(n, device=dev))
ctx.loss_finalize()
old = (ctx.export_token_stats()["lp"] + 0.02 * torch.randn(n, device=dev)).contiguous()


def stages(kind):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    ev[0].record()
    ctx.prepare(rewards, gid, so, n_tokens=n)
    torch.matmul(h, W.T, out=z)
    ev[1].record()
    if kind == "unfused":
        ctx.loss_fwd(z, tokens, old)
        ctx.loss_finalize()
        ctx.loss_bwd(z, z)
    else:
        ctx.loss_fwd_factored(z, tokens, old, grad=z)
        ctx.loss_finalize()
        ctx.loss_row_scale(out=sc)
    ev[2].record()
    torch.matmul(z, W, out=dh)
    ev[3].record()
    if kind == "factored":
        dh.mul_(sc[:, None])
    ev[4].record()
    hs = h * sc[:, None].to(h.dtype) if kind == "factored" else h
    ev[5].record()
    dW.add_(torch.matmul(z.T, hs))
    ev[6].record()
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(6)]


for kind in ("unfused", "factored", "unfused", "factored"):
    for _ in range(2):
        stages(kind)
    t = stages(kind)
    print(kind, "logits %.2f | espo %.2f | dh %.2f | scale %.2f | hs %.2f | dW %.2f | total %.2f ms" % (*t, sum(t)))
