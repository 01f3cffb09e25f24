"""One espo_lmhead_fwd call (after a warm-up call) on synthetic h, W — the target of ncu
captures of the forward GEMM-core kernel. usage:
python tools/lmhead_fwd_once.py [d] [n] [impl: -1 = cuBLAS logits GEMM] [raster option] [calls]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07710_b200.espo import OPT_LMHEAD_IMPL, OPT_LMHEAD_RASTER, Espo  # noqa: E402


def main(d=4096, n=32768, impl=0, raster=0, calls=2, V=151936):
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
    if impl >= 0:
        ctx.set_option(OPT_LMHEAD_IMPL, impl)
        ctx.set_option(OPT_LMHEAD_RASTER, raster)
    for _ in range(calls):
        if impl < 0:
            torch.matmul(h, W.T)
            continue
        ctx.prepare(rewards, gid, so, n_tokens=n)
        ctx.lmhead_fwd(h, W, tokens, torch.full((n,), -1.0, device=dev))
        ctx.loss_finalize()
    torch.cuda.synchronize()
    ctx.get_error()
    print("ok", flush=True)


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
