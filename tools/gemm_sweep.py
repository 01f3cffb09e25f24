"""A/B sweep of the LM-head backward's GEMM settings (ESPO_OPT_LMHEAD_BWD_GEMM, _GEMM_GROUP_M,
_GEMM_HINTS): time espo_lmhead_bwd on one 8192-row sub-chunk per setting, interleaved over
rounds (median), same data. Prints one JSON line.
usage: python tools/gemm_sweep.py [d] [n] [V] [rounds] [burst] [set: default | sync]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07710_b200.espo import (OPT_GEMM_GROUP_M, OPT_GEMM_HINTS,  # noqa: E402
                                        OPT_GEMM_SYNC, OPT_LMHEAD_BWD_GEMM, OPT_LMHEAD_BWD_ROWS,
                                        OPT_LMHEAD_COMPACT,
                                        OPT_LMHEAD_IMPL, OPT_LMHEAD_RASTER, Espo)


def main(d=4096, n=8192, V=151936, rounds=5, burst=1, which="default"):
    """burst = back-to-back timed calls per setting and round (burst > 1: sustained clocks)."""
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
    ctx.prepare(rewards, gid, so, n_tokens=n)
    ctx.lmhead_fwd(h, W, tokens, torch.zeros(n, device=dev))
    ctx.loss_finalize()
    old = (ctx.export_token_stats()["lp"] + 0.02 * torch.randn(n, device=dev)).contiguous()
    ctx.prepare(rewards, gid, so, n_tokens=n)
    ctx.lmhead_fwd(h, W, tokens, old)
    ctx.loss_finalize()
    dh = torch.empty((n, d), dtype=torch.bfloat16, device=dev)
    dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
    H = lambda a, b, c: a | (b << 2) | (c << 4)
    dw_auto = H(1, 2, 1)
    G = lambda dh_m, dw_n: dh_m | (dw_n << 16)
    H2 = lambda dh, dw: dh | (dw << 8)
    MC = 1 << 25
    NOSPLIT = 1 << 26
    cfgs = {                     # (gemm, group, hints, compact, sync (-1 auto), lmhead impl, lm raster)
        # cuBLAS doing dh / dW on the same GEMM-core recompute and row compaction (only the two
        # GEMMs differ; until the end of round 2 this leg ran the dedicated dz kernel and no
        # compaction, which flattered the native default by ~2 ms per sub-chunk)
        "cublas": (1, 0, -1, 1, -1, 0, 0),
        "default": (0, 0, -1, 1, -1, 0, 0),
        "nosplit": (0, 0, -1, 1, -1, 0, NOSPLIT),
        "dh256": (0, 0, -1, 1, -1, 0, 0),
    }
    cfgs["dh256"] = (3, G(0, 8), -1, 1, -1, 0, 0)
    NOLOCK = 1 << 27
    cfgs["dz_g32_nolock"] = (0, 0, -1, 1, -1, 0, 32 | NOLOCK)    # round-2 dz raster
    cfgs["dz_g16_nolock"] = (0, 0, -1, 1, -1, 0, 16 | NOLOCK)
    rows_opt = {}
    if which == "rows":          # backward sub-chunk rows (A / B panel sizes of dW and dh)
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "rows4096": cfgs["default"], "rows16384": cfgs["default"],
                "cublas_rows16384": cfgs["cublas"]}
        rows_opt = {"rows4096": 4096, "rows16384": 16384, "cublas_rows16384": 16384}
    if which == "mc":            # TMA multicast across two CTA pairs (4-CTA clusters)
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "mc_both": (5, 0, -1, 1, -1, 0, 0), "mc_dh": (6, 0, -1, 1, -1, 0, 0),
                "mc_dh_nosplit": (6, 0, -1, 1, -1, 0, 1 << 26),
                "dw256_g1": (0, G(0, 1), -1, 1, -1, 0, 0)}
    if which == "dyn":           # tile scheduler: dynamic (default) vs static round robin (bit 29)
        ST, NL = 1 << 29, 1 << 27  # (r2bm measured this set while bit 29 meant "dynamic")
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "static": (0, 0, -1, 1, -1, 0, ST), "static_nolock_dz": (0, 0, -1, 1, -1, 0, ST | NL),
                "dyn_nolock_all": (0, 0, -1, 1, 0, 0, NL), "dyn_dw_n16": (0, G(0, 16), -1, 1, -1, 0, 0)}
    if which == "wide":          # d > 4096 under the dynamic scheduler: dW tiles / groups, dh groups
        L = lambda ch, sl: ch | (sl << 16)
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "dw256_n8": (3, G(16, 8), -1, 1, -1, 0, 0),
                "dw512_n4": (4, G(16, 4), -1, 1, -1, 0, 0), "dw512_n8": (4, G(16, 8), -1, 1, -1, 0, 0),
                "dh8": (0, G(8, 0), -1, 1, -1, 0, 0), "dh32": (0, G(32, 0), -1, 1, -1, 0, 0),
                "sync8": (0, 0, -1, 1, L(8, 2), 0, 0)}
    if which == "wide2":         # d > 4096: lockstep on dh only / dW only / dW with more slack
        L = lambda ch, sl: ch | (sl << 16)
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "dh_lock_dw_off": (0, 0, -1, 1, L(16, 2) | (L(0, 1) << 32), 0, 0),
                "dh_off_dw_lock": (0, 0, -1, 1, L(0, 2) | (L(16, 2) << 32), 0, 0),
                "dw_slack8": (0, 0, -1, 1, L(16, 2) | (L(16, 8) << 32), 0, 0),
                "dw_chunk32": (0, 0, -1, 1, L(16, 2) | (L(32, 2) << 32), 0, 0)}
    if which == "wide3":         # d > 4096: 256-wide dW tiles with the default 512-wide dh
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "dw256": (7, 0, -1, 1, -1, 0, 0), "dw256_n16": (7, G(0, 16), -1, 1, -1, 0, 0),
                "dw256_n4": (7, G(0, 4), -1, 1, -1, 0, 0)}
    if which == "red":           # dW epilogue: TMA reduce-add (default) vs SM read-add-write (bit 30)
        RMW = 1 << 30             # (r2bs measured this set while bit 30 meant "TMA reduce")
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "sm_rmw": (0, 0, -1, 1, -1, 0, RMW), "dw256": (7, 0, -1, 1, -1, 0, 0)}
    if which == "dwel":          # dW: A (dz panels) evict_last, B evict_last, C evict_first
        Hd = lambda a, b, c: (a | (b << 2) | (c << 4)) << 8
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "n16_el": (0, G(0, 16), Hd(2, 2, 1), 1, -1, 0, 0),
                "n8_el": (0, G(0, 8), Hd(2, 2, 1), 1, -1, 0, 0),
                "n16_el_sync16": (0, G(0, 16), Hd(2, 2, 1), 1, (16 | (4 << 16)) << 32, 0, 0)}
    if which == "dwr":           # dW raster / L2 policies / tile width (dense sub-chunks)
        Hd = lambda a, b, c: (a | (b << 2) | (c << 4)) << 8          # dW's byte of GEMM_HINTS
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "dw_n16": (0, G(0, 16), -1, 1, -1, 0, 0), "dw_n4": (0, G(0, 4), -1, 1, -1, 0, 0),
                "dw_n16_Bnorm": (0, G(0, 16), Hd(1, 0, 1), 1, -1, 0, 0),
                "dw_n8_allnorm": (0, G(0, 8), Hd(0, 0, 0), 1, -1, 0, 0),
                "dw512_n8": (4, G(0, 8), -1, 1, -1, 0, 0)}
    if which == "half":          # 512-column accumulators released in halves (default) or whole
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "whole_release": (0, 0, -1, 1, -1, 0, 1 << 28)}
    if which == "dw":            # dW on 256 × 512 pair tiles (kind 4: dh too) × N-groups × lockstep
        L = lambda ch, sl: ch | (sl << 16)
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "dw512_n8": (4, G(0, 8), -1, 1, -1, 0, 0), "dw512_n4": (4, G(0, 4), -1, 1, -1, 0, 0),
                "dw512_n2": (4, G(0, 2), -1, 1, -1, 0, 0),
                "dw512_n8_sync8": (4, G(0, 8), -1, 1, L(8, 2), 0, 0),
                "default_sync8": (0, 0, -1, 1, L(8, 2), 0, 0)}
    if which == "syncdw":        # soft lockstep of the dW GEMM alone (bits 32+)
        Ldw = lambda ch, sl: (ch | (sl << 16)) << 32
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "dw_sync4": (0, 0, -1, 1, Ldw(4, 2), 0, 0), "dw_sync8": (0, 0, -1, 1, Ldw(8, 2), 0, 0),
                "dw_sync16": (0, 0, -1, 1, Ldw(16, 2), 0, 0), "dw_sync8_s1": (0, 0, -1, 1, Ldw(8, 1), 0, 0),
                "dw_sync8_n4": (0, G(0, 4), -1, 1, Ldw(8, 2), 0, 0),
                "dw_sync8_n16": (0, G(0, 16), -1, 1, Ldw(8, 2), 0, 0)}
    if which == "syncdw2":       # dW lockstep with more slack (chunk, slack in chunks)
        Ldw = lambda ch, sl: (ch | (sl << 16)) << 32
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "dw_8_4": (0, 0, -1, 1, Ldw(8, 4), 0, 0), "dw_8_8": (0, 0, -1, 1, Ldw(8, 8), 0, 0),
                "dw_16_4": (0, 0, -1, 1, Ldw(16, 4), 0, 0), "dw_4_8": (0, 0, -1, 1, Ldw(4, 8), 0, 0),
                "dw_4_16": (0, 0, -1, 1, Ldw(4, 16), 0, 0), "dw_32_2": (0, 0, -1, 1, Ldw(32, 2), 0, 0)}
    if which == "sync":          # soft lockstep of the dh / dW GEMMs (ESPO_OPT_GEMM_SYNC)
        L = lambda ch, sl: ch | (sl << 16)
        cfgs = {"cublas": cfgs["cublas"], "default": cfgs["default"],
                "nolock": (0, 0, -1, 1, 0, 0, 0), "nolock_dh8": (0, G(8, 0), -1, 1, 0, 0, 0),
                "sync8": (0, 0, -1, 1, L(8, 2), 0, 0), "sync16": (0, 0, -1, 1, L(16, 2), 0, 0),
                "sync32": (0, 0, -1, 1, L(32, 2), 0, 0),
                "sync16_dh16": (0, G(16, 0), -1, 1, L(16, 2), 0, 0),
                "sync16_dh4": (0, G(4, 0), -1, 1, L(16, 2), 0, 0),
                "sync16_dw4": (0, G(0, 4), -1, 1, L(16, 2), 0, 0)}
    times = {k: [] for k in cfgs}
    for _ in range(rounds):
        for k, (impl, gm, hints, compact, sync, lmi, lmr) in cfgs.items():
            ctx.set_option(OPT_GEMM_SYNC, sync)
            ctx.set_option(OPT_LMHEAD_IMPL, lmi)
            ctx.set_option(OPT_LMHEAD_RASTER, lmr)
            ctx.set_option(OPT_LMHEAD_BWD_GEMM, impl)
            ctx.set_option(OPT_GEMM_GROUP_M, gm)
            ctx.set_option(OPT_GEMM_HINTS, hints)
            ctx.set_option(OPT_LMHEAD_COMPACT, compact)
            ctx.set_option(OPT_LMHEAD_BWD_ROWS, rows_opt.get(k, 0))
            ctx.lmhead_bwd(h, W, dh, dW)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(burst):
                ctx.lmhead_bwd(h, W, dh, dW)
            e.record()
            torch.cuda.synchronize()
            times[k].append(s.elapsed_time(e) / burst)
    ctx.get_error()
    flops = 6.0 * n * V * d
    out = {k: {"ms": statistics.median(v), "TFLOPs_3gemm": flops / (statistics.median(v) * 1e-3) / 1e12}
           for k, v in times.items()}
    out["config"] = {"n": n, "d": d, "V": V, "rounds": rounds, "burst": burst}
    print(json.dumps(out))


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:6]] + sys.argv[6:7]
    main(*a)
