"""Worker functions for the world_size-2 gloo tests (module-level so spawn can import them)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _init(rank, world, port):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    return dist


def partial_vector(res):
    """The 26 rank-local fp64 terms libespo all-reduces (layout of kRedLen in common.cuh)."""
    st = res.stats
    tok = np.array(st["tokens_per_bucket"])
    v = np.zeros(26)
    v[0] = res.J_sum
    v[1] = st["n_active_rollouts"]
    v[2] = st["n_active_tokens"]
    v[3] = st["n_zv_groups"]
    v[4] = st["n_groups"]
    v[5] = st["n_clipped_tokens"]
    v[6] = st["mean_abs_logratio"] * st["n_active_tokens"]
    v[7] = st["mean_entropy"] * st["n_active_tokens"]
    v[8:12] = tok
    v[12:16] = np.array(st["clip_frac"]) * tok
    v[16:20] = np.array(st["mean_ratio"]) * tok
    v[20:24] = np.array(st["mean_eps"]) * tok
    v[24] = st["mean_sq_logratio"] * st["n_active_tokens"]
    v[25] = st["mean_k3"] * st["n_active_tokens"]
    return v


def worker_unique_id(rank, world, port, out_q):
    dist = _init(rank, world, port)
    from paper_2512_07710_b200.espo import bootstrap_unique_id
    uid = bootstrap_unique_id(rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, uid)
    out_q.put((rank, len(uid), all(g == gathered[0] for g in gathered)))
    dist.destroy_process_group()


def worker_sharded_oracle(rank, world, port, out_q):
    import torch
    dist = _init(rank, world, port)
    from oracle import espo_oracle as O
    from paper_2512_07710_b200.sharding import plan_shards, shard_batch
    from tests._instances import tiny_instance
    inst = tiny_instance(31, V=97, group_sizes=(4, 4, 3, 4, 2, 4, 1), lengths=None, L=9,
                         mask_tail=3, sigma_seq=0.1,
                         rewards=[1, 0, 0, 1, 1, 1, 1, 1, 0, 1, 0, 1, 0, 1, 1, 0.5, 0.5,
                                  0.25, 0.75, 0.2, 0, 1])
    cfg = O.OracleConfig(vocab=inst.V)
    plan = plan_shards(inst.group_ids, inst.seq_offsets, world, rewards=inst.rewards)
    rollouts, toks, gid, so = shard_batch(plan[rank], inst.group_ids, inst.seq_offsets)
    res = O.espo_loss(inst.logits[toks], inst.tokens[toks], inst.old_logp[toks],
                      inst.mask[toks], inst.rewards[rollouts], gid, so, cfg)
    v = torch.tensor(partial_vector(res), dtype=torch.float64)
    dist.all_reduce(v)                       # the one exchange of the pass
    D = v[1].item()
    loss = -v[0].item() / D
    # rank-local coefficients divided by the GLOBAL D: the scale every rank applies in bwd
    g = res.coef / D
    plans = [None] * world
    dist.all_gather_object(plans, plan)
    out_q.put((rank, loss, v.numpy().tolist(), toks.tolist(), g.tolist(), plans))
    dist.destroy_process_group()


def worker_subgroup_unique_id(rank, world, port, out_q):
    """bootstrap over a sub-group that does not contain global rank 0 (a TP group)."""
    dist = _init(rank, world, port)
    from paper_2512_07710_b200.espo import bootstrap_unique_id
    sub = dist.new_group(ranks=[1])
    uid = bootstrap_unique_id(0, sub) if rank == 1 else None
    full = bootstrap_unique_id(rank)
    out_q.put((rank, None if uid is None else len(uid), len(full)))
    dist.destroy_process_group()


def worker_bench_strong_batch(rank, world, port, out_q):
    """bench.py's strong-scaling data path on the CPU (C0 recipe): this rank's share of the
    global batch — global row id, token, old log-prob and the buffer row each local row reads."""
    import torch
    dist = _init(rank, world, port)
    import bench
    import espo_synth as S
    w = S.WORKLOADS["C0"]
    seed = S.config_seed(w.index)
    d = bench.make_batch(w, seed, torch.device("cpu"), 64, lambda m: None,
                         shard=(world, rank), drift=(0.04, 0.02))
    bufrow = np.empty(d["T"], np.int64)
    for b, e in d["chunks"]:
        bufrow[b:e] = np.arange(e - b)
    g = d["global_row"].numpy()
    out = (rank, g.tolist(), d["tokens"].numpy().tolist(), d["old"].numpy().tolist(),
           bufrow.tolist(), [list(c) for c in d["chunks"]], d["np"]["group_ids"].tolist(),
           d["np"]["seq_offsets"].tolist())
    dist.barrier()
    out_q.put(out)
    dist.destroy_process_group()
