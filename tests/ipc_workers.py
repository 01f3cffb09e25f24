"""Spawned workers for the two-process CUDA-IPC test (module-level for multiprocessing)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def worker_p2p_ipc(rank, world, port, out_q):
    """TP rank `rank` of 2 on the same GPU, connected through real CUDA IPC handles. The host
    orders the phases (both sends complete → barrier → both receives), so no kernel ever waits
    on a kernel of the other process that has not finished."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2512_07710_b200.espo import Espo
    from tests._instances import workload_instance
    from tests.gpu_common import to_dev
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    inst = workload_instance("C0")
    T, V = inst.T, inst.V
    w = V // world
    v0 = rank * w
    ctx = Espo(V, logits_dtype=torch.float32, device=0, vocab_shard=(v0, w))
    h = ctx.tp_p2p_buffer(T, world)
    hs = [None] * world
    dist.all_gather_object(hs, h)
    ctx.tp_p2p_open(b"".join(hs), rank, world)
    z = to_dev(inst.logits[:, v0:v0 + w], torch.float32, dev).contiguous()
    tok = to_dev(inst.tokens, torch.int32, dev)
    old = to_dev(inst.old_logp, torch.float32, dev)
    mask = to_dev(inst.mask, torch.uint8, dev)
    ctx.prepare(to_dev(inst.rewards, torch.float32, dev), to_dev(inst.group_ids, torch.int32, dev),
                to_dev(inst.seq_offsets, torch.int64, dev), n_tokens=T)
    ctx.loss_fwd_p2p_send(z, tok, old, mask)
    torch.cuda.synchronize()
    dist.barrier()                               # every rank's partials are in every buffer
    ctx.loss_fwd_p2p_recv(0, T)
    loss, _ = ctx.loss_finalize()
    dz = ctx.loss_bwd(z)
    ctx.get_error()
    out_q.put((rank, float(loss.item()), dz.cpu().numpy().astype(np.float32)))
    dist.barrier()
    ctx.tp_p2p_unmap()
    dist.barrier()                               # no mapping outlives its exporter
    ctx.close()
    dist.destroy_process_group()
