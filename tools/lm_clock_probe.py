"""Clocks/power while the fused LM head and cuBLAS run back to back (d = 4096): is the gap a
clock (power-cap) effect? Samples nvidia-smi every 50 ms during each 3 s loop."""
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07710_b200.espo import Espo  # noqa: E402


def sample(fn, seconds=3.0):
    q = "clocks.sm,power.draw,clocks_event_reasons.sw_power_cap"
    p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    n = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < seconds:
        fn()
        n += 1
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    clk = sorted(float(l.split(",")[0]) for l in out if l.strip())
    pw = sorted(float(l.split(",")[1]) for l in out if l.strip())
    return {"ms_per_iter": s.elapsed_time(e) / n, "sm_mhz_median": clk[len(clk) // 2],
            "power_w_median": pw[len(pw) // 2], "samples": len(clk)}


def main(d=4096, n=32768, V=151936):
    dev = torch.device("cuda", 0)
    h = (torch.randn(n, d, device=dev) / d ** 0.5 * 3).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev).to(torch.bfloat16)
    tok = torch.randint(0, V, (n,), device=dev, dtype=torch.int32)
    old = torch.full((n,), -1.0, device=dev)
    rew = torch.tensor([1.0, 0.0] * 4, device=dev)
    gid = torch.zeros(8, dtype=torch.int32, device=dev)
    so = torch.arange(9, device=dev, dtype=torch.int64) * (n // 8)
    ctx = Espo(V, logits_dtype=torch.bfloat16, device=0)
    ctx2 = Espo(V, logits_dtype=torch.bfloat16, device=0)
    ctx2.set_option(5, 1)

    def fused_2cta():
        ctx2.prepare(rew, gid, so, n_tokens=n)
        ctx2.lmhead_fwd(h, W, tok, old)
        ctx2.loss_finalize()

    def fused():
        ctx.prepare(rew, gid, so, n_tokens=n)
        ctx.lmhead_fwd(h, W, tok, old)
        ctx.loss_finalize()

    def cublas():
        torch.matmul(h, W.T)

    out = {}
    for name, fn in (("fused", fused), ("cublas", cublas), ("fused_2cta", fused_2cta), ("fused2", fused)):
        fn()
        r = sample(fn)
        r["TFLOPs"] = 2.0 * n * V * d / (r["ms_per_iter"] * 1e-3) / 1e12
        out[name] = r
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4096)
