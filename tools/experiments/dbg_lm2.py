"""Debug: run the CTA-pair LM-head forward once and print the CUDA error string."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2512_07710_b200.espo import Espo, OPT_LMHEAD_2CTA  # noqa: E402


def main(n=256, V=512, d=128, two=1):
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    h = (torch.randn(n, d, device=dev) / d ** 0.5).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev).to(torch.bfloat16)
    tok = torch.randint(0, V, (n,), device=dev, dtype=torch.int32)
    old = torch.full((n,), -1.0, device=dev)
    rew = torch.tensor([1.0, 0.0], device=dev)
    gid = torch.zeros(2, dtype=torch.int32, device=dev)
    so = torch.tensor([0, n // 2, n], device=dev, dtype=torch.int64)
    ctx = Espo(V, logits_dtype=torch.float32, device=0)
    ctx.set_option(OPT_LMHEAD_2CTA, two)
    ctx.prepare(rew, gid, so, n_tokens=n)
    ctx.lmhead_fwd(h, W, tok, old)
    try:
        torch.cuda.synchronize()
        print("ok")
    except Exception as e:  # noqa: BLE001
        print("ERR", e)
        return
    lse = ctx.export_token_stats()["lse"]
    ref = torch.logsumexp(h.float() @ W.float().T, dim=1)
    print("max |lse - ref|", (lse - ref).abs().max().item())


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
