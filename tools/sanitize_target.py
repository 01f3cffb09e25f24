"""Target program for the compute-sanitizer tier (tests/test_gpu_sanitizer.py).

Runs every kernel family of libespo once at small sizes through the C ABI, on the device and
stream the sanitizer watches:
  - C0 (fp32) two-sweep pass in two chunks (K1 prepare, K2 TMA-ring sweep, K3, K4, K5 tiled
    backward), single-pass mode, factored mode (k_fwd_grad_ring), compact mode;
  - a C1-shaped bf16 slice (4 rollouts × 96 tokens, V = 151,936): K2 at full width (dynamic
    row claiming), K5, the factored ring at full width;
  - the fused LM head: forward (one CTA and CTA pairs), backward (dz recompute, the CTA-pair and
    one-CTA tcgen05 GEMMs);
  - vocabulary-parallel exchange over peer memory between two same-device contexts
    (espo_tp_p2p_connect_local: the fused sweep stores partials into both buffers, flags,
    combine) and the partial + combine path;
  - the split finalize (espo_loss_reduce_local / espo_loss_finalize_reduced).
Prints "sanitize target ok" at the end. Sizes keep memcheck/racecheck runs to minutes.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_07710_b200.espo import (OPT_FACTORED_IMPL, OPT_LMHEAD_2CTA,  # noqa: E402
                                        OPT_LMHEAD_BWD_GEMM, Espo)
from tests._instances import tiny_instance, workload_instance  # noqa: E402


def t(a, dt, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dt)


def args_of(inst, dev):
    return (t(inst.rewards, torch.float32, dev), t(inst.group_ids, torch.int32, dev),
            t(inst.seq_offsets, torch.int64, dev))


def c0_modes(dev):
    inst = workload_instance("C0")
    T, V = inst.T, inst.V
    z = t(inst.logits, torch.float32, dev)
    tok, old = t(inst.tokens, torch.int32, dev), t(inst.old_logp, torch.float32, dev)
    mask = t(inst.mask, torch.uint8, dev)
    a = args_of(inst, dev)
    for compact in (False, True):
        c = Espo(V, logits_dtype=torch.float32, device=dev.index, zero_fill_inactive_rows=not compact)
        c.prepare(*a, n_tokens=T)
        c.loss_fwd(z[:300], tok[:300], old[:300], mask[:300], row_begin=0)
        c.loss_fwd(z[300:], tok[300:], old[300:], mask[300:], row_begin=300)
        c.loss_finalize()
        dz = torch.zeros_like(z)
        c.loss_bwd(z[:300], dz[:300], row_begin=0)
        c.loss_bwd(z[300:], dz[300:], row_begin=300)
        c.get_error()
        c.close()
    c = Espo(V, logits_dtype=torch.float32, device=dev.index)          # single pass
    c.prepare(*a, n_tokens=T)
    c.set_mask(mask)
    so = inst.seq_offsets
    for i, j in ((0, 5), (5, 16)):
        b, e = int(so[i]), int(so[j])
        c.loss_fwd_bwd(z[b:e], tok[b:e], old[b:e], row_begin=b)
    c.loss_finalize()
    c.get_error()
    c.close()
    c = Espo(V, logits_dtype=torch.float32, device=dev.index)          # factored
    c.prepare(*a, n_tokens=T)
    c.loss_fwd_factored(z, tok, old, mask)
    c.loss_finalize()
    c.loss_row_scale()
    c.get_error()
    c.close()
    c = Espo(V, logits_dtype=torch.float32, device=dev.index)          # split finalize
    c.prepare(*a, n_tokens=T)
    c.loss_fwd(z, tok, old, mask)
    p = c.loss_reduce_local()
    c.loss_finalize_reduced(p)
    c.loss_bwd(z)
    c.get_error()
    c.close()


def c1_slice(dev):
    inst = tiny_instance(11, V=151936, group_sizes=(4,), L=96, dtype="bf16")
    T, V = inst.T, inst.V
    z = t(inst.logits, torch.float32, dev).to(torch.bfloat16)
    tok, old = t(inst.tokens, torch.int32, dev), t(inst.old_logp, torch.float32, dev)
    a = args_of(inst, dev)
    c = Espo(V, logits_dtype=torch.bfloat16, device=dev.index)
    c.prepare(*a, n_tokens=T)
    c.loss_fwd(z, tok, old)
    c.loss_finalize()
    c.loss_bwd(z)
    c.get_error()
    c.set_option(OPT_FACTORED_IMPL, 0)
    c.prepare(*a, n_tokens=T)
    c.loss_fwd_factored(z, tok, old)
    c.loss_finalize()
    c.get_error()
    c.close()


def lmhead(dev):
    rng = np.random.default_rng(3)
    V, d, G, L = 4099, 512, 4, 64
    T = G * L
    h = torch.from_numpy((rng.standard_normal((T, d)) / np.sqrt(d) * 3).astype(np.float32)).to(dev).to(torch.bfloat16)
    W = torch.from_numpy(rng.standard_normal((V, d)).astype(np.float32)).to(dev).to(torch.bfloat16)
    tok = torch.from_numpy(rng.integers(0, V, T).astype(np.int32)).to(dev)
    a = (torch.tensor([1.0, 0.0, 1.0, 0.0], device=dev), torch.zeros(G, dtype=torch.int32, device=dev),
         torch.arange(G + 1, dtype=torch.int64, device=dev) * L)
    for two, gemm in ((0, 0), (1, 2)):
        c = Espo(V, logits_dtype=torch.bfloat16, device=dev.index)
        c.set_option(OPT_LMHEAD_2CTA, two)
        c.set_option(OPT_LMHEAD_BWD_GEMM, gemm)
        c.prepare(*a, n_tokens=T)
        c.lmhead_fwd(h, W, tok, torch.zeros(T, device=dev) - 8.0)
        c.loss_finalize()
        dW = torch.zeros((V, d), dtype=torch.float32, device=dev)
        c.lmhead_bwd(h, W, None, dW)
        c.get_error()
        c.close()


def tp(dev):
    inst = tiny_instance(19, V=512, group_sizes=(4, 4), L=16)
    T = inst.T
    z = t(inst.logits, torch.float32, dev)
    tok, old = t(inst.tokens, torch.int32, dev), t(inst.old_logp, torch.float32, dev)
    a = args_of(inst, dev)
    shards = [(0, 256), (256, 256)]
    ctxs = [Espo(512, logits_dtype=torch.float32, device=dev.index, vocab_shard=s) for s in shards]
    for c in ctxs:
        c.tp_p2p_buffer(T, 2)
    for k, c in enumerate(ctxs):
        c.tp_p2p_connect_local(ctxs, k)
    for c in ctxs:
        c.prepare(*a, n_tokens=T)
    for c, (v0, w) in zip(ctxs, shards):
        c.loss_fwd_p2p_send(z[:, v0:v0 + w].contiguous(), tok, old)
    for c in ctxs:
        c.loss_fwd_p2p_recv(0, T)
    for c, (v0, w) in zip(ctxs, shards):
        c.loss_finalize()
        c.loss_bwd(z[:, v0:v0 + w].contiguous())
        c.get_error()
    for c in ctxs:
        c.tp_p2p_unmap()
    torch.cuda.synchronize(dev)
    for c in ctxs:
        c.close()
    ctxs = [Espo(512, logits_dtype=torch.float32, device=dev.index, vocab_shard=s) for s in shards]
    parts = []
    for c, (v0, w) in zip(ctxs, shards):
        c.prepare(*a, n_tokens=T)
        parts.append(c.loss_fwd_partial(z[:, v0:v0 + w].contiguous(), tok, old))
    g = torch.stack(parts)
    for c in ctxs:
        c.loss_fwd_combine(g)
        c.loss_finalize()
        c.get_error()
        c.close()


def main(which="all"):
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    steps = {"c0": c0_modes, "c1": c1_slice, "lmhead": lmhead, "tp": tp}
    for k, f in steps.items():
        if which in ("all", k):
            f(dev)
            torch.cuda.synchronize(dev)
            print(f"[sanitize] {k} done", flush=True)
    print("sanitize target ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
