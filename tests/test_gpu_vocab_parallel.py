"""Vocabulary-parallel ESPO: logits sharded by vocabulary columns as in
a Megatron vocab-parallel LM head. Each shard's sweep produces per-row partials
{R, S, W, u_y}; the partials of all shards are combined into the exact row statistics; the
backward writes each shard's columns. On one GPU the shards run as independent launches of
independent contexts and the all-gather is a device copy (no kernel waits on another);
results must match the oracle (and the unsharded run) at the usual tolerances."""
import numpy as np
import pytest
import torch

from paper_2512_07710_b200.espo import Espo
from tests._instances import tiny_instance, workload_instance
from tests.gpu_common import (check_dlogits_bf16, check_dlogits_f32, check_exact_fields,
                              check_loss, check_token_stats, decision_aware_reference,
                              oracle_cfg, oracle_dlogits, require_cuda, run_gpu, to_dev)

pytestmark = pytest.mark.gpu


def run_sharded(inst, dev, shards, logits_dtype=torch.float32, grad_dtype=None, cfgkw=None,
                fwd_impl=0, bwd_impl=0):
    from paper_2512_07710_b200.espo import OPT_BWD_IMPL, OPT_FWD_IMPL, stats_to_dict
    cfgkw = dict(cfgkw or {})
    T, V = inst.T, inst.V
    align = 8 if logits_dtype == torch.bfloat16 else 4
    zfull = to_dev(inst.logits, torch.float32, dev)
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev)
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    ctxs, zs = [], []
    for v0, w in shards:
        ctx = Espo(V, logits_dtype=logits_dtype, grad_dtype=grad_dtype, device=dev.index,
                   vocab_shard=(v0, w), **cfgkw)
        ctx.set_option(OPT_FWD_IMPL, fwd_impl)
        ctx.set_option(OPT_BWD_IMPL, bwd_impl)
        ld = (w + align - 1) // align * align
        z = torch.zeros((T, ld), dtype=logits_dtype, device=dev)
        z[:, :w] = zfull[:, v0:v0 + w].to(logits_dtype)
        ctx.prepare(*args, n_tokens=T)
        ctxs.append(ctx)
        zs.append(z)
    parts = [c.loss_fwd_partial(z, tok, old, mask) for c, z in zip(ctxs, zs)]
    gathered = torch.stack(parts)                      # the TP all-gather, as a device copy
    out = []
    for (v0, w), c, z in zip(shards, ctxs, zs):
        c.loss_fwd_combine(gathered)
        loss, stats = c.loss_finalize()
        dz = c.loss_bwd(z)
        c.get_error()
        out.append((float(loss.item()), stats_to_dict(stats), dz[:, :w].float().cpu().numpy()))
    tokst = {k: v.cpu().numpy() for k, v in ctxs[0].export_token_stats().items()}
    rol = {k: v.cpu().numpy() for k, v in ctxs[0].export_rollout_stats().items()}
    for c in ctxs:
        c.close()
    dl = np.concatenate([o[2] for o in out], axis=1)
    return dict(loss=out[0][0], stats=out[0][1], losses=[o[0] for o in out], dlogits=dl,
                tok=tokst, rol=rol, zv_out=rol["zv"])


@pytest.mark.parametrize("impl", [0, 1], ids=["tma", "ldg"])
def test_vocab_parallel_fp32_three_shards(impl):
    dev = require_cuda()
    inst = workload_instance("C0")
    g = run_sharded(inst, dev, [(0, 300), (300, 400), (700, 324)], fwd_impl=impl, bwd_impl=impl)
    assert len(set(g["losses"])) == 1                 # every shard sees the same loss
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))
    u = run_gpu(inst, dev)                            # unsharded run: same result
    assert g["loss"] == pytest.approx(u["loss"], rel=1e-6)


def test_vocab_parallel_bf16_ragged_eight_shards():
    dev = require_cuda()
    inst = tiny_instance(17, V=4099, group_sizes=(8, 8), L=24, dtype="bf16", mask_tail=4)
    w = [512] * 7 + [4099 - 7 * 512]
    shards = [(sum(w[:k]), w[k]) for k in range(8)]
    g = run_sharded(inst, dev, shards, logits_dtype=torch.bfloat16, grad_dtype=torch.float32)
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))


@pytest.mark.parametrize("impl", [0, 1], ids=["tma", "ldg"])
def test_vocab_parallel_reference_seeding_extreme_range(impl):
    """Rows whose target lies in another shard start each lane from its first vector's
    largest element (K2 seed_ref). Logits 100 above that in later vectors (2^144: the batch
    sums overflow) must still take the max-referenced fallback, and a −inf first vector must
    leave the lane unseeded; parity with the oracle and with the unsharded run. (The far
    elements are moved down, not the near ones up: logits of magnitude 100 would carry fp32
    rounding of ~1e-5 relative into p, beyond the test's element bound.)"""
    from tests._instances import exact_lp
    import espo_synth as S
    dev = require_cuda()
    inst = tiny_instance(23, V=2048, group_sizes=(4, 4), L=12, sigma_seq=0.0, sigma_tok=0.0)
    for t in range(0, inst.T, 2):
        inst.logits[t, :600] -= 100.0                # later vectors of shard 1 (600..999)
        inst.logits[t, 1000:] -= 100.0               # lie 100 above everything else
        inst.logits[t, 1536:1600] = -np.inf          # first vectors of shard 3
    inst.tokens[inst.tokens >= 1536] = 1700          # targets stay finite
    inst.old_logp = S.drift_old_logp(exact_lp(inst.logits, inst.tokens), inst.seq_offsets, 4)
    shards = [(0, 512), (512, 512), (1024, 512), (1536, 512)]
    g = run_sharded(inst, dev, shards, fwd_impl=impl, bwd_impl=impl)
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    assert np.nanmin(ref.lp) < -90
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))
    u = run_gpu(inst, dev)          # lp ≈ −100 carries ~1e-5 relative fp32 rounding into
    assert g["loss"] == pytest.approx(u["loss"], rel=5e-5)    # the ratios of either run


def test_sharded_context_requires_partial_path():
    """A sharded context without a TP communicator cannot run the fused espo_loss_fwd."""
    from paper_2512_07710_b200.espo import EspoError
    dev = require_cuda()
    inst = tiny_instance(18, V=256, group_sizes=(2,), L=4)
    ctx = Espo(256, logits_dtype=torch.float32, device=dev.index, vocab_shard=(0, 128))
    ctx.prepare(to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
                to_dev(inst.seq_offsets, torch.int64, dev), n_tokens=inst.T)
    z = torch.zeros((inst.T, 128), dtype=torch.float32, device=dev)
    with pytest.raises(EspoError) as e:
        ctx.loss_fwd(z, to_dev(inst.tokens, torch.int32, dev), to_dev(inst.old_logp, torch.float32, dev))
    assert e.value.code == "ESPO_ERR_BAD_STATE"
    ctx.close()


def run_p2p(inst, dev, shards, chunks, logits_dtype=torch.float32, cfgkw=None, single_pass=False):
    """Peer-memory TP on one device: one context per shard connected with
    espo_tp_p2p_connect_local; per chunk every rank sends (fused sweep stores its partials into
    every rank's exchange buffer, then signals) before any rank receives (waits, combines) —
    so no kernel waits on a kernel launched after it."""
    from paper_2512_07710_b200.espo import stats_to_dict
    T = inst.T
    align = 8 if logits_dtype == torch.bfloat16 else 4
    zfull = to_dev(inst.logits, torch.float32, dev)
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev)
    args = (to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
            to_dev(inst.seq_offsets, torch.int64, dev))
    ctxs, zs = [], []
    max_rows = max(e - b for b, e in chunks)
    for v0, w in shards:
        ctx = Espo(inst.V, logits_dtype=logits_dtype, device=dev.index, vocab_shard=(v0, w),
                   **(cfgkw or {}))
        ctx.tp_p2p_buffer(max_rows, len(shards))
        ld = (w + align - 1) // align * align
        z = torch.zeros((T, ld), dtype=logits_dtype, device=dev)
        z[:, :w] = zfull[:, v0:v0 + w].to(logits_dtype)
        ctxs.append(ctx)
        zs.append(z)
    for k, c in enumerate(ctxs):
        c.tp_p2p_connect_local(ctxs, k)
    for step in range(2):                        # two steps: epochs keep running across them
        for c in ctxs:
            c.prepare(*args, n_tokens=T)
        for b, e in chunks:
            for c, z in zip(ctxs, zs):
                c.loss_fwd_p2p_send(z[b:e], tok[b:e], old[b:e], mask[b:e], row_begin=b)
            for c in ctxs:
                c.loss_fwd_p2p_recv(b, e - b)
        out = []
        for (v0, w), c, z in zip(shards, ctxs, zs):
            loss, stats = c.loss_finalize()
            dz = c.loss_bwd(z)
            c.get_error()
            out.append((float(loss.item()), stats_to_dict(stats), dz[:, :w].float().cpu().numpy()))
    tokst = {k: v.cpu().numpy() for k, v in ctxs[0].export_token_stats().items()}
    rol = {k: v.cpu().numpy() for k, v in ctxs[0].export_rollout_stats().items()}
    for c in ctxs:
        c.close()
    return dict(loss=out[0][0], stats=out[0][1], losses=[o[0] for o in out],
                dlogits=np.concatenate([o[2] for o in out], axis=1), tok=tokst, rol=rol,
                zv_out=rol["zv"])


def test_vocab_parallel_peer_memory_exchange():
    """Fused exchange over peer memory ≡ the device-copy all-gather path, bitwise (the same
    partials are merged in the same order), and ≡ the oracle at fp32 tolerances; chunks split
    sequences, arrive out of order, and reuse both exchange slots over two steps."""
    dev = require_cuda()
    inst = workload_instance("C0")
    shards = [(0, 300), (300, 400), (700, 324)]
    chunks = [(700, inst.T), (0, 130), (130, 700)]
    g = run_p2p(inst, dev, shards, chunks)
    ref_path = run_sharded(inst, dev, shards)
    assert len(set(g["losses"])) == 1
    assert g["loss"] == ref_path["loss"]
    assert np.array_equal(g["dlogits"], ref_path["dlogits"])
    cfg = oracle_cfg(inst.V)
    ref = inst.run(cfg)
    check_exact_fields(g, ref)
    check_token_stats(g, ref)
    ref2, _ = decision_aware_reference(g, inst, ref, cfg)
    check_loss(g, ref2, 1e-5)
    check_dlogits_f32(g["dlogits"], oracle_dlogits(ref2, inst, cfg, np.arange(inst.T)))


def test_peer_memory_recv_without_peer_times_out():
    """A rank whose peer never sends reports ESPO_ERR_PEER_TIMEOUT instead of hanging."""
    from paper_2512_07710_b200.espo import EspoError
    dev = require_cuda()
    inst = tiny_instance(19, V=256, group_sizes=(2,), L=4)
    ctxs = [Espo(256, logits_dtype=torch.float32, device=dev.index, vocab_shard=(128 * k, 128))
            for k in range(2)]
    from paper_2512_07710_b200.espo import OPT_PEER_TIMEOUT_MS
    for c in ctxs:
        c.tp_p2p_buffer(16, 2)
        c.set_option(OPT_PEER_TIMEOUT_MS, 300)     # default 120 s; bound the test's wait
    for k, c in enumerate(ctxs):
        c.tp_p2p_connect_local(ctxs, k)
    z = torch.zeros((inst.T, 128), dtype=torch.float32, device=dev)
    c = ctxs[0]
    c.prepare(to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
              to_dev(inst.seq_offsets, torch.int64, dev), n_tokens=inst.T)
    c.loss_fwd_p2p_send(z, to_dev(inst.tokens, torch.int32, dev), to_dev(inst.old_logp, torch.float32, dev))
    c.loss_fwd_p2p_recv(0, inst.T)               # rank 1 never sends
    with pytest.raises(EspoError) as e:
        c.get_error()
    assert e.value.code == "ESPO_ERR_PEER_TIMEOUT"
    for x in ctxs:
        x.close()


def test_peer_memory_exchange_over_cuda_ipc_two_processes():
    """The multi-process path of the peer-memory exchange (IPC handles all-gathered over a
    process group, cudaIpcOpenMemHandle, NVLink-style stores into the other process's buffer)
    with two processes sharing the one GPU; phases ordered by the host so no kernel waits on a
    running kernel of the other process. Loss and gradient equal the single-process run."""
    import multiprocessing as mp
    import socket
    from tests import ipc_workers
    dev = require_cuda()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    ps = [ctxm.Process(target=ipc_workers.worker_p2p_ipc, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted([q.get(timeout=300) for _ in ps], key=lambda x: x[0])
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    inst = workload_instance("C0")
    u = run_gpu(inst, dev)
    assert out[0][1] == out[1][1]
    assert out[0][1] == pytest.approx(u["loss"], rel=1e-6)
    dl = np.concatenate([out[0][2], out[1][2]], axis=1)
    np.testing.assert_allclose(dl, u["dlogits"], rtol=1e-5, atol=1e-7 * np.abs(u["dlogits"]).max())
