"""K2 tail effect: forward-sweep bandwidth for chunks of n rows with n = m·(warps) and
n = m·(warps) + small, all rows active (no ZV), V = 151,936 bf16."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2512_07710_b200.espo import Espo  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    V = 151936
    warps = 148 * 16
    nmax = 12 * warps + 512
    z = (torch.randn(nmax, V, device=dev) - 14).to(torch.bfloat16)
    tok = torch.randint(0, V, (nmax,), device=dev, dtype=torch.int32)
    old = torch.full((nmax,), -5.0, device=dev)
    res = {}
    for n in (11 * warps, 11 * warps + 64, 11 * warps + 512, 12 * warps, 12 * warps + 64):
        G = 8
        R = G
        L = n // R
        n = L * R
        rew = torch.tensor([1.0, 0.0] * (G // 2), device=dev)
        gid = torch.zeros(R, dtype=torch.int32, device=dev)
        so = torch.arange(R + 1, device=dev, dtype=torch.int64) * L
        ctx = Espo(V, logits_dtype=torch.bfloat16, device=0)
        for _ in range(2):
            ctx.prepare(rew, gid, so, n_tokens=n)
            ctx.loss_fwd(z[:n], tok[:n], old[:n])
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            ctx.prepare(rew, gid, so, n_tokens=n)
            s.record()
            ctx.loss_fwd(z[:n], tok[:n], old[:n])
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = sorted(ts)[2]
        res[n] = {"rows_per_warp": n / warps, "ms": ms, "TBps": n * V * 2 / (ms * 1e-3) / 1e12}
        ctx.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
