"""Guard-band tier (SURVEY §4c T5 substitute): compute-sanitizer is closed on this GPU pool, so
out-of-bounds accesses and races are hunted with the library's own data instead.

Every buffer a kernel family touches is a view into a larger allocation:
- INPUT margins (rows before/after the chunk, columns between vocab and the row pitch) hold
  NaN: a kernel that reads outside its rows/columns trips ESPO_ERR_NONFINITE_INPUT or turns
  its results NaN (the GEMM paths) — both fail the test;
- OUTPUT margins hold a sentinel bit pattern that must survive bit for bit: a kernel that
  writes outside its rows/columns (dlogits, G, dh, dW, partials, row scales) fails.
Each family also runs twice on the same inputs and must reproduce its outputs bitwise (a
racing reduction or a dynamic-scheduling bug shows up as run-to-run differences).
Families: K2/K3/K4/K5 two-sweep (fp32 C0 and a bf16 C1-shaped slice at V = 151,936, the
TMA-ring forward with dynamic row claiming), compact mode, single pass, factored, vocabulary
partial + combine, the fused LM head forward and backward (dz recompute + both tcgen05 GEMMs,
CTA-pair and one-CTA)."""
import numpy as np
import pytest
import torch

from paper_2512_07710_b200.espo import Espo
from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import require_cuda, to_dev

pytestmark = pytest.mark.gpu

PAD_R, PAD_C = 7, 24          # margin rows above/below, extra columns per row
SENT32 = 0x7FBADBAD           # NaN payload sentinel (f32 bits)
SENT16 = 0x7FBA               # NaN payload sentinel (bf16 bits)


def _fill_sentinel(t):
    if t.dtype == torch.float32:
        t.view(torch.int32).fill_(SENT32)
    else:
        t.view(torch.int16).fill_(SENT16)


def _bits(t):
    return t.view(torch.int32 if t.dtype == torch.float32 else torch.int16)


class Guarded:
    """2-D: base[PAD_R : PAD_R + rows, :cols] is the view (row pitch cols + PAD_C); everything
    else is margin. fill = "nan" for inputs, else the sentinel bit pattern."""

    def __init__(self, rows, cols, dtype, dev, fill=None, value=None):
        pitch = -(-(cols + PAD_C) // 8) * 8          # 16-byte aligned row pitch
        self.base = torch.empty((rows + 2 * PAD_R, pitch), dtype=dtype, device=dev)
        if fill == "nan":
            self.base.fill_(float("nan"))
        else:
            _fill_sentinel(self.base)
        self.view = self.base[PAD_R:PAD_R + rows, :cols]
        if value is not None:
            self.view.copy_(value)
        self.mask = torch.ones(self.base.shape, dtype=torch.bool, device=dev)
        self.mask[PAD_R:PAD_R + rows, :cols] = False
        self.snapshot = self.base.clone()

    def margins_intact(self):
        return bool(torch.equal(_bits(self.base)[self.mask], _bits(self.snapshot)[self.mask]))


class GuardedFlat:
    """Contiguous [n, k] view inside a flat allocation with PAD elements on both sides."""
    PAD = 64

    def __init__(self, n, k, dtype, dev):
        self.base = torch.empty(n * k + 2 * self.PAD, dtype=dtype, device=dev)
        _fill_sentinel(self.base)
        self.view = self.base[self.PAD:self.PAD + n * k].view(n, k) if k > 1 else \
            self.base[self.PAD:self.PAD + n]
        self.n = n * k
        self.snapshot = self.base.clone()

    def margins_intact(self):
        a, b = _bits(self.base), _bits(self.snapshot)
        return bool(torch.equal(a[:self.PAD], b[:self.PAD]) and
                    torch.equal(a[self.PAD + self.n:], b[self.PAD + self.n:]))


def _args(inst, dev):
    return (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))


def _two_sweep(inst, dev, dtype, compact=False, chunks=None):
    T, V = inst.T, inst.V
    z = Guarded(T, V, dtype, dev, fill="nan", value=to_dev(inst.logits, torch.float32, dev).to(dtype))
    tok, old = to_dev(inst.tokens, torch.int32, dev), to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev) if inst.mask is not None else None
    outs = []
    for _ in range(2):
        dz = Guarded(T, V, dtype, dev)
        ctx = Espo(V, logits_dtype=dtype, device=dev.index, zero_fill_inactive_rows=not compact)
        ctx.prepare(*_args(inst, dev), n_tokens=T)
        for b, e in chunks or [(0, T)]:
            ctx.loss_fwd(z.view[b:e], tok[b:e], old[b:e], None if mask is None else mask[b:e],
                         row_begin=b)
        loss, stats = ctx.loss_finalize()
        for b, e in chunks or [(0, T)]:
            ctx.loss_bwd(z.view[b:e], dz.view[b:e], row_begin=b)
        ctx.get_error()
        ctx.close()
        assert dz.margins_intact(), "dlogits written outside its rows / columns"
        assert np.isfinite(float(loss.item()))
        outs.append((loss.clone(), stats.clone(), dz.base.clone()))
    assert z.margins_intact()
    (l0, s0, d0), (l1, s1, d1) = outs
    assert torch.equal(l0, l1) and torch.equal(s0, s1)
    assert torch.equal(_bits(d0), _bits(d1))


@pytest.mark.parametrize("compact", [False, True], ids=["zero_fill", "compact"])
def test_guard_two_sweep_c0(compact):
    dev = require_cuda()
    inst = workload_instance("C0")
    _two_sweep(inst, dev, torch.float32, compact, chunks=[(0, 333), (333, inst.T)])


def test_guard_two_sweep_c1_slice_bf16():
    dev = require_cuda()
    inst = tiny_instance(11, V=151936, group_sizes=(4, 2), L=80, dtype="bf16", mask_tail=9)
    _two_sweep(inst, dev, torch.bfloat16, chunks=[(0, 200), (200, inst.T)])


def test_guard_single_pass_and_factored():
    dev = require_cuda()
    inst = workload_instance("C0")
    T, V = inst.T, inst.V
    z = Guarded(T, V, torch.float32, dev, fill="nan", value=to_dev(inst.logits, torch.float32, dev))
    tok, old = to_dev(inst.tokens, torch.int32, dev), to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev)
    so = inst.seq_offsets
    res = []
    for _ in range(2):
        dz = Guarded(T, V, torch.float32, dev)
        ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
        ctx.prepare(*_args(inst, dev), n_tokens=T)
        ctx.set_mask(mask)
        for i, j in ((0, 7), (7, 16)):
            b, e = int(so[i]), int(so[j])
            ctx.loss_fwd_bwd(z.view[b:e], tok[b:e], old[b:e], dz.view[b:e], row_begin=b)
        loss, _ = ctx.loss_finalize()
        ctx.get_error()
        ctx.close()
        assert dz.margins_intact()
        G = Guarded(T, V, torch.float32, dev)
        sc = GuardedFlat(T, 1, torch.float32, dev)
        ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
        ctx.prepare(*_args(inst, dev), n_tokens=T)
        ctx.loss_fwd_factored(z.view, tok, old, mask, grad=G.view)
        ctx.loss_finalize()
        ctx.loss_row_scale(out=sc.view)
        ctx.get_error()
        ctx.close()
        assert G.margins_intact() and sc.margins_intact()
        res.append((loss.clone(), dz.base.clone(), G.base.clone(), sc.base.clone()))
    assert z.margins_intact()
    for a, b in zip(res[0], res[1]):
        assert torch.equal(_bits(a), _bits(b))


def test_guard_vocab_partial_combine():
    dev = require_cuda()
    inst = tiny_instance(19, V=1000, group_sizes=(4, 4), L=24)
    T = inst.T
    zf = to_dev(inst.logits, torch.float32, dev)
    tok, old = to_dev(inst.tokens, torch.int32, dev), to_dev(inst.old_logp, torch.float32, dev)
    shards = [(0, 400), (400, 600)]
    zs = [Guarded(T, w, torch.float32, dev, fill="nan", value=zf[:, v0:v0 + w]) for v0, w in shards]
    ctxs = [Espo(1000, logits_dtype=torch.float32, device=dev.index, vocab_shard=s) for s in shards]
    parts = []
    for c, z in zip(ctxs, zs):
        c.prepare(*_args(inst, dev), n_tokens=T)
        p = GuardedFlat(T, 4, torch.float32, dev)
        c.loss_fwd_partial(z.view, tok, old, partial=p.view)
        assert p.margins_intact()
        parts.append(p.view.clone())
    g = torch.stack(parts)
    for c, z, (v0, w) in zip(ctxs, zs, shards):
        c.loss_fwd_combine(g)
        c.loss_finalize()
        dz = Guarded(T, w, torch.float32, dev)
        c.loss_bwd(z.view, dz.view)
        c.get_error()
        assert dz.margins_intact() and z.margins_intact()
        c.close()


@pytest.mark.parametrize("impl,two_cta,gemm,d", [(0, 0, 0, 320), (1, 0, 0, 320), (1, 1, 2, 320),
                                                 (0, 0, 4, 320), (0, 0, 0, 4168)],
                         ids=["gemm_core", "1cta_fwd+pair_gemm", "2cta_fwd+1cta_gemm",
                              "gemm_core+pair512", "gemm_core_wide_lockstep"])
def test_guard_lmhead(impl, two_cta, gemm, d):
    """d = 4168 > 4096 also runs the dh / dW soft lockstep, 512-wide dW tiles and split-K dh."""
    from paper_2512_07710_b200.espo import (OPT_LMHEAD_2CTA, OPT_LMHEAD_BWD_GEMM,
                                            OPT_LMHEAD_BWD_ROWS, OPT_LMHEAD_IMPL)
    dev = require_cuda()
    rng = np.random.default_rng(5)
    V, G, L = 3001, 4, 70                           # V, d, n: none a multiple of the tiles
    T = G * L
    hv = torch.from_numpy((rng.standard_normal((T, d)) / np.sqrt(d) * 3).astype(np.float32)).to(dev)
    Wv = torch.from_numpy(rng.standard_normal((V, d)).astype(np.float32)).to(dev)
    h = Guarded(T, d, torch.bfloat16, dev, fill="nan", value=hv.to(torch.bfloat16))
    W = Guarded(V, d, torch.bfloat16, dev, fill="nan", value=Wv.to(torch.bfloat16))
    tok = torch.from_numpy(rng.integers(0, V, T).astype(np.int32)).to(dev)
    args = (torch.tensor([1.0, 0.0, 1.0, 1.0], device=dev), torch.tensor([0, 0, 1, 1], dtype=torch.int32, device=dev),
            torch.arange(G + 1, dtype=torch.int64, device=dev) * L)
    res = []
    for _ in range(2):
        c = Espo(V, logits_dtype=torch.bfloat16, device=dev.index)
        c.set_option(OPT_LMHEAD_IMPL, impl)
        c.set_option(OPT_LMHEAD_2CTA, two_cta)
        c.set_option(OPT_LMHEAD_BWD_GEMM, gemm)
        c.set_option(OPT_LMHEAD_BWD_ROWS, 128)        # several backward sub-chunks
        c.prepare(*args, n_tokens=T)
        c.lmhead_fwd(h.view, W.view, tok, torch.full((T,), -8.0, device=dev))
        loss, _ = c.loss_finalize()
        dh = Guarded(T, d, torch.float32, dev)
        dW = Guarded(V, d, torch.float32, dev, value=torch.zeros((V, d), device=dev))
        c.lmhead_bwd(h.view, W.view, dh.view, dW.view)
        c.get_error()
        c.close()
        assert dh.margins_intact(), "dhidden written outside its rows / columns"
        assert dW.margins_intact(), "dweight written outside its rows / columns"
        assert torch.isfinite(dh.view).all() and torch.isfinite(dW.view).all()   # no NaN margin read
        assert np.isfinite(float(loss.item()))
        res.append((loss.clone(), dh.view.clone(), dW.view.clone()))
    assert h.margins_intact() and W.margins_intact()
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)


def test_guard_two_sweep_ragged_vocab_bf16():
    """V = 2051 (not a multiple of the 8-element vector): the row end falls inside a 16-byte
    vector whose tail lies in the NaN margin."""
    dev = require_cuda()
    inst = tiny_instance(23, V=2051, group_sizes=(3, 4), L=33, dtype="bf16", mask_tail=4)
    _two_sweep(inst, dev, torch.bfloat16, chunks=[(0, 100), (100, inst.T)])
