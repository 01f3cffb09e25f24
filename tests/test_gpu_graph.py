"""CUDA-graph capture of the whole pass (prepare → fwd → finalize → bwd).

The C ABI is stream-ordered with no host synchronisation inside the pass, so
a trainer can capture one step into a CUDA graph and replay it with new inputs copied into
the same device buffers. Checks: (1) replaying the captured graph on the captured inputs
reproduces the eager results bit for bit; (2) replaying after overwriting the inputs with a
different seeded instance of the same shape matches the oracle at the usual tolerances."""
import numpy as np
import pytest
import torch

from tests._instances import workload_instance
from tests.gpu_common import (check_dlogits_f32, check_exact_fields, check_loss,
                              check_token_stats, decision_aware_reference, oracle_cfg,
                              oracle_dlogits, require_cuda, to_dev)

pytestmark = pytest.mark.gpu


def _inputs(inst, dev):
    return dict(z=to_dev(inst.logits, torch.float32, dev),
                tok=to_dev(inst.tokens, torch.int32, dev),
                old=to_dev(inst.old_logp, torch.float32, dev),
                mask=to_dev(inst.mask, torch.uint8, dev),
                rew=to_dev(inst.rewards, torch.float32, dev),
                gid=to_dev(inst.group_ids, torch.int32, dev),
                off=to_dev(inst.seq_offsets, torch.int64, dev))


def test_graph_capture_and_replay():
    from paper_2512_07710_b200.espo import STATS_LEN, Espo, stats_to_dict
    dev = require_cuda()
    a = workload_instance("C0")
    b = workload_instance("C0", seed=12345)
    assert a.logits.shape == b.logits.shape and np.array_equal(a.seq_offsets, b.seq_offsets)
    T, V = a.T, a.V
    buf = _inputs(a, dev)
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    stats = torch.empty(STATS_LEN, dtype=torch.float64, device=dev)
    dz = torch.empty((T, V), dtype=torch.float32, device=dev)

    def step():
        ctx.prepare(buf["rew"], buf["gid"], buf["off"], n_tokens=T)
        ctx.loss_fwd(buf["z"], buf["tok"], buf["old"], buf["mask"])
        ctx.loss_finalize(loss, stats)
        ctx.loss_bwd(buf["z"], dz)

    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        step()                                   # warm-up: allocates the workspace
    torch.cuda.current_stream(dev).wait_stream(s)
    ctx.get_error()
    eager_loss, eager_dz = loss.clone(), dz.clone()
    launches_eager = ctx.launch_count

    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    assert ctx.launch_count > launches_eager     # kernels were recorded, not run
    loss.zero_()
    dz.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize(dev)
    ctx.get_error()
    assert torch.equal(loss, eager_loss)
    assert torch.equal(dz, eager_dz)

    nb = _inputs(b, dev)                         # new step: same shapes, new data
    for k in buf:
        buf[k].copy_(nb[k])
    g.replay()
    torch.cuda.synchronize(dev)
    ctx.get_error()
    got = dict(loss=float(loss.item()), stats=stats_to_dict(stats), dlogits=dz.cpu().numpy(),
               tok={k: v.cpu().numpy() for k, v in ctx.export_token_stats().items()},
               rol={k: v.cpu().numpy() for k, v in ctx.export_rollout_stats().items()})
    got["zv_out"] = got["rol"]["zv"]
    ctx.close()
    cfg = oracle_cfg(V)
    ref = b.run(cfg)
    check_exact_fields(got, ref)
    check_token_stats(got, ref)
    ref2, _ = decision_aware_reference(got, b, ref, cfg)
    check_loss(got, ref2, 1e-5)
    check_dlogits_f32(got["dlogits"], oracle_dlogits(ref2, b, cfg, np.arange(T)))


def test_graph_capture_single_pass():
    """The single-pass mode captures too: prepare → set_mask → fwd_bwd per rollout chunk →
    finalize, replayed on new data equals an eager run on that data, bitwise."""
    from paper_2512_07710_b200.espo import STATS_LEN, Espo
    dev = require_cuda()
    a = workload_instance("C0")
    b = workload_instance("C0", seed=777)
    T, V = a.T, a.V
    buf = _inputs(a, dev)
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    stats = torch.empty(STATS_LEN, dtype=torch.float64, device=dev)
    dz = torch.empty((T, V), dtype=torch.float32, device=dev)
    so = a.seq_offsets
    chunks = [(int(so[i]), int(so[j])) for i, j in ((0, 5), (5, 9), (9, 16))]

    def step():
        ctx.prepare(buf["rew"], buf["gid"], buf["off"], n_tokens=T)
        ctx.set_mask(buf["mask"])
        for lo, hi in chunks:
            ctx.loss_fwd_bwd(buf["z"][lo:hi], buf["tok"][lo:hi], buf["old"][lo:hi], dz[lo:hi],
                             row_begin=lo)
        ctx.loss_finalize(loss, stats)

    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream(dev).wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    nb = _inputs(b, dev)
    for k in buf:
        buf[k].copy_(nb[k])
    g.replay()
    torch.cuda.synchronize(dev)
    ctx.get_error()
    got_loss, got_dz = loss.clone(), dz.clone()
    step()                                       # eager on the same (new) data
    torch.cuda.synchronize(dev)
    ctx.get_error()
    assert torch.equal(got_loss, loss) and torch.equal(got_dz, dz)
    ctx.close()


def test_graph_capture_compact_mode():
    """Compact mode (rows without gradient untouched) captures too: espo_prepare skips its
    host copy of the rollout layout under capture and espo_loss_bwd's grid then covers whole
    chunks; the replay on new data equals an eager run on that data, bitwise."""
    from paper_2512_07710_b200.espo import STATS_LEN, Espo
    dev = require_cuda()
    a = workload_instance("C0")
    b = workload_instance("C0", seed=4242)
    T, V = a.T, a.V
    buf = _inputs(a, dev)
    ctx = Espo(V, logits_dtype=torch.float32, device=dev.index, zero_fill_inactive_rows=False)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    stats = torch.empty(STATS_LEN, dtype=torch.float64, device=dev)
    dz = torch.zeros((T, V), dtype=torch.float32, device=dev)
    chunks = [(0, 300), (300, T)]

    def step():
        ctx.prepare(buf["rew"], buf["gid"], buf["off"], n_tokens=T)
        for lo, hi in chunks:
            ctx.loss_fwd(buf["z"][lo:hi], buf["tok"][lo:hi], buf["old"][lo:hi], buf["mask"][lo:hi],
                         row_begin=lo)
        ctx.loss_finalize(loss, stats)
        for lo, hi in chunks:
            ctx.loss_bwd(buf["z"][lo:hi], dz[lo:hi], row_begin=lo)

    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream(dev).wait_stream(s)
    ctx.get_error()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    nb = _inputs(b, dev)
    for k in buf:
        buf[k].copy_(nb[k])
    dz.zero_()
    g.replay()
    torch.cuda.synchronize(dev)
    ctx.get_error()
    got_loss, got_dz = loss.clone(), dz.clone()
    dz.zero_()
    step()                                       # eager on the same (new) data
    torch.cuda.synchronize(dev)
    ctx.get_error()
    assert torch.equal(got_loss, loss) and torch.equal(got_dz, dz)
    assert torch.count_nonzero(got_dz.abs().sum(1)) > 0
    ctx.close()


@pytest.mark.parametrize("d", [256, 4160])
def test_graph_capture_lmhead(d):
    """The fused LM head (GEMM-core forward with the soft lockstep, compacted backward with
    split-K dh; d = 4160 also runs the dh / dW lockstep) captured after one warm-up step: the
    replay reproduces the eager loss, dhidden and dweight bit for bit — the lockstep's progress
    counters are zeroed inside the graph, and no call synchronises with the host."""
    from paper_2512_07710_b200.espo import Espo
    dev = require_cuda()
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    n, V = 1024, 4104
    h = (torch.randn(n, d, device=dev, generator=g) / d ** 0.5 * 3).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev, generator=g).to(torch.bfloat16)
    tok = torch.randint(0, V, (n,), device=dev, dtype=torch.int32, generator=g)
    G = 8
    rew = torch.tensor([1.0, 0.0, 1.0, 1.0, 0.0, 0.0, 1.0, 0.0], device=dev)
    gid = torch.zeros(G, dtype=torch.int32, device=dev)
    off = torch.arange(G + 1, device=dev, dtype=torch.int64) * (n // G)
    ctx = Espo(V, logits_dtype=torch.bfloat16, device=dev.index)
    ctx.prepare(rew, gid, off, n_tokens=n)
    ctx.lmhead_fwd(h, W, tok, torch.zeros(n, device=dev))
    ctx.loss_finalize()
    old = (ctx.export_token_stats()["lp"] + 0.05 * torch.randn(n, device=dev, generator=g))
    old = old.contiguous()
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    from paper_2512_07710_b200.espo import STATS_LEN
    stats = torch.empty(STATS_LEN, dtype=torch.float64, device=dev)
    dh = torch.empty((n, d), dtype=torch.float32, device=dev)
    dW = torch.empty((V, d), dtype=torch.float32, device=dev)

    def step():
        ctx.prepare(rew, gid, off, n_tokens=n)
        ctx.lmhead_fwd(h, W, tok, old)
        ctx.loss_finalize(loss, stats)
        dW.zero_()
        ctx.lmhead_bwd(h, W, dh, dW)

    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        step()                                   # warm-up: grows every scratch buffer
    torch.cuda.current_stream(dev).wait_stream(s)
    ctx.get_error()
    e_loss, e_dh, e_dW = loss.clone(), dh.clone(), dW.clone()
    assert float(e_dh.abs().max()) > 0 and float(e_dW.abs().max()) > 0
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(2):
        loss.zero_()
        dh.fill_(float("nan"))
        dW.fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize(dev)
        ctx.get_error()
        assert torch.equal(loss, e_loss)
        assert torch.equal(dh, e_dh)
        assert torch.equal(dW, e_dW)
    ctx.close()
