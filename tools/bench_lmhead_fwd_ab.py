"""A/B of the fused LM-head forward implementations against cuBLAS on one 32,768-row chunk,
V = 151,936: ESPO_OPT_LMHEAD_IMPL 0 (GEMM core, pair 256×512 tiles, per-tile partials) over a
few raster groups, impl 1 (dedicated one-CTA kernel), and torch.matmul bf16 (cuBLAS, writing
the logits). Settings interleaved over rounds, `burst` calls back to back each (sustained
clocks). usage: python tools/bench_lmhead_fwd_ab.py [d] [rounds] [burst] [set]
sets "sync" / "sync2" (raster groups × lockstep chunk / slack) were measured while
ESPO_OPT_GEMM_SYNC still governed these launches (tools/experiments/r2aq.sh, r2ar.sh); now a 4th
element 0 turns the forward's lockstep off (ESPO_OPT_LMHEAD_RASTER bit 27) and any other value
keeps the default (8 K-steps, slack 2). Set "default2": the default against the earlier rasters."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07710_b200.espo import (OPT_GEMM_SYNC, OPT_LMHEAD_IMPL, OPT_LMHEAD_RASTER,  # noqa: E402
                                        Espo)


def main(d=4096, rounds=3, burst=4, which="default", n=32768, V=151936):
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
    MC = 1 << 9                      # (hints << 16): bit 25 of the raster option = multicast
    cfgs = {"gemm_g32": (0, 32, 0), "gemm_g64": (0, 64, 0), "mc_g16": (0, 16, MC),
            "mc_g32": (0, 32, MC), "mc_g64": (0, 64, MC), "mc_g128": (0, 128, MC),
            "dedicated_1cta": (1, 8, 0), "cublas": None}
    if which == "sync":          # (impl, group, hints, lockstep chunk | slack << 16)
        cfgs = {"gemm_g32": (0, 32, 0, 0), "g32_sync8": (0, 32, 0, 8 | 2 << 16),
                "g16_sync8": (0, 16, 0, 8 | 2 << 16), "g12_sync8": (0, 12, 0, 8 | 2 << 16),
                "g12": (0, 12, 0, 0), "g32_sync4": (0, 32, 0, 4 | 1 << 16), "cublas": None}
    if which == "default2":      # the default (g16 + lockstep) against the earlier g32
        cfgs = {"default": (0, 0, 0), "g32_nolock": (0, 32, 0, 0), "g64_nolock": (0, 64, 0, 0),
                "cublas": None}
    if which == "half":          # accumulator released in halves (default) or whole (bit 28)
        cfgs = {"default": (0, 0, 0), "whole_release": (0, 0, 1 << 12), "cublas": None}
    if which == "dyn":           # (measured while bit 29 selected the dynamic scheduler, r2bm)
        cfgs = {"default": (0, 0, 0), "static": (0, 0, 1 << 13), "nolock": (0, 0, 0, 0),
                "static_nolock": (0, 0, 1 << 13, 0), "cublas": None}
    if which == "groups":        # raster group under the dynamic scheduler (lockstep on)
        cfgs = {"g16": (0, 16, 0), "g8": (0, 8, 0), "g32": (0, 32, 0), "g64": (0, 64, 0),
                "g24": (0, 24, 0), "cublas": None}
    if which == "sync2":
        cfgs = {"g16_s8_2": (0, 16, 0, 8 | 2 << 16), "g16_s16_2": (0, 16, 0, 16 | 2 << 16),
                "g16_s8_4": (0, 16, 0, 8 | 4 << 16), "g16_s4_2": (0, 16, 0, 4 | 2 << 16),
                "g24_s8_2": (0, 24, 0, 8 | 2 << 16), "g8_s8_2": (0, 8, 0, 8 | 2 << 16),
                "g32_s8_2": (0, 32, 0, 8 | 2 << 16), "g16_s8_1": (0, 16, 0, 8 | 1 << 16),
                "cublas": None}
    times = {k: [] for k in cfgs}
    losses = {}
    for _ in range(rounds):
        for k, c in cfgs.items():
            if c is None:
                fn = lambda: torch.matmul(h, W.T)
            else:
                impl, g, hints = c[:3]
                ctx.set_option(OPT_LMHEAD_IMPL, impl)
                ctx.set_option(OPT_LMHEAD_RASTER, g | (hints << 16))
                ctx.set_option(OPT_GEMM_SYNC, -1)
                if len(c) > 3 and c[3] == 0:
                    ctx.set_option(OPT_LMHEAD_RASTER, g | (hints << 16) | (1 << 27))

                def fn():
                    ctx.prepare(rewards, gid, so, n_tokens=n)
                    ctx.lmhead_fwd(h, W, tokens, old)
                    return ctx.loss_finalize()[0]
            fn()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(burst):
                out = fn()
            e.record()
            torch.cuda.synchronize()
            times[k].append(s.elapsed_time(e) / burst)
            if c is not None:
                losses[k] = float(out.item())
    ctx.get_error()
    res = {k: {"ms": statistics.median(v),
               "TFLOPs": 2.0 * n * V * d / (statistics.median(v) * 1e-3) / 1e12}
           for k, v in times.items()}
    res["loss_by_impl"] = losses
    res["config"] = {"n": n, "V": V, "d": d, "rounds": rounds, "burst": burst}
    print(json.dumps(res))


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:4]] + sys.argv[4:5]
    main(*a)
