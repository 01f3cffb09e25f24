#!/usr/bin/env python3
"""ESPO loss fwd+bwd benchmark (BASELINE.json metric) — one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--scaling weak|strong] [--config C1..C4] [--verify]

A step = one whole ESPO pass (espo_prepare → espo_loss_fwd over every chunk →
espo_loss_finalize → espo_loss_bwd over every chunk) over one synthetic batch.

--gpus N: one process per GPU. Under torchrun (WORLD_SIZE set) N must equal WORLD_SIZE;
without it and N > 1 this script re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (127.0.0.1 rendezvous). Fewer visible
GPUs than N is an error (exit 2): a world is never silently shrunk.

--scaling weak (default): each rank owns its own batch of the configuration (C1 =
64 prompts × 8 rollouts × 4096 tokens, vocab 151,936, bf16 logits); the one NCCL all-reduce of
the pass normalises the loss over all ranks. --scaling strong (north_star's C4 scaling
config): one fixed global batch, identical on every rank, whose prompt groups are split over
the ranks by sharding.plan_shards (LPT on expected sweep cost, PAPER.md:244's length
balancing); each rank sweeps only its groups. --verify adds an untimed pass that hashes every
dlogits row with its global row id (order-independent, summed over ranks): in strong mode the
digest and the loss must not depend on N.

Logits do not fit in HBM (637 GB per C1 batch), so they stream through a device chunk buffer
of --buffer-rows rows (9.96 GB at 32,768 rows, well above the 126 MB L2): a row at offset o
inside its chunk reads buffer row o (chunks are fixed R_c slabs of the batch in weak mode, and
R_c slabs of each prompt group in strong mode, so a row's data never depends on N). Timing:
CUDA events on the launching stream, W warm-up steps, barrier + synchronize around exactly K
steps, max over ranks. `--impl reference` times the CPU oracle (oracle/) on bounded samples.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import espo_synth as S  # noqa: E402

NOMINAL_HBM_GBS = 8000.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=None,
                   help="GPUs = ranks (default: WORLD_SIZE under torchrun, else 1)")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: a batch of --config per rank; strong: one global batch split "
                        "over the ranks by prompt group (LPT)")
    p.add_argument("--emulate-ranks", type=int, default=0,
                   help="with --scaling strong on one GPU: run the N ranks' shards one after "
                        "another (split finalize for the exchange); projected step = slowest rank")
    p.add_argument("--verify", action="store_true",
                   help="untimed extra pass: order-independent digest of every dlogits row")
    p.add_argument("--drift-seq", type=float, default=0.01,
                   help="std of the per-rollout log-prob drift of the rollout engine (SURVEY "
                        "§8(d) recipe: b_i ~ N(0, 0.01))")
    p.add_argument("--drift-tok", type=float, default=0.02,
                   help="std of the per-token log-prob drift")
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C1", help="C1 (default), C2, C3, C4 (BASELINE.json)")
    p.add_argument("--compact", action="store_true",
                   help="compact mode: rows without gradient are not zero-filled (C3)")
    p.add_argument("--buffer-rows", type=int, default=65536,
                   help="rows per chunk call (the chunk buffer is rows × V bf16: 19.9 GB at C1)")
    p.add_argument("--fwd-impl", type=int, default=0, help="0/2/3/4 = TMA ring variants, 1 = LDG")
    p.add_argument("--bwd-impl", type=int, default=0, help="0/7 = tiled grid, 1 = LDG, 2-6 = TMA rings")
    p.add_argument("--blocks-per-sm", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--e2e-host-rows", type=int, default=8192,
                   help="host ring rows (≥ the longest rollout; chunks pack whole rollouts)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-tokens", type=int, default=128, help="tokens per rollout")
    p.add_argument("--single-pass", action="store_true",
                   help="device leg through espo_set_mask + espo_loss_fwd_bwd (chunks of whole rollouts)")
    p.add_argument("--factored", action="store_true",
                   help="factored-gradient leg: espo_loss_fwd_factored (one sweep per row writes "
                        "G = onehot - p) + espo_loss_row_scale")
    p.add_argument("--no-factored-leg", action="store_true",
                   help="skip the factored-gradient leg reported beside the headline")
    p.add_argument("--factored-impl", type=int, default=0, help="ESPO_OPT_FACTORED_IMPL (0 = default)")
    p.add_argument("--e2e-mode", default="single-pass", choices=["single-pass", "two-sweep"],
                   help="e2e leg: logits chunks cross PCIe once (single-pass) or twice")
    p.add_argument("--zv-mode", default="mask", choices=["mask", "rlzvp"],
                   help="zero-variance groups: eliminated (default) or RL-ZVP advantages")
    p.add_argument("--tp-p2p", action="store_true",
                   help="with --vocab-shards: exchange partials through the fused peer-memory "
                        "path (espo_tp_p2p_*) instead of partial + device-copy gather + combine")
    p.add_argument("--vocab-shards", type=int, default=1,
                   help="S > 1: vocabulary-parallel leg, S shard contexts back to back on this "
                        "GPU (partials gathered by a device copy)")
    a = p.parse_args()
    if a.emulate_ranks and (a.scaling != "strong" or (a.gpus or 1) != 1 or a.impl != "ours"):
        p.error("--emulate-ranks N needs --scaling strong on one GPU (our arm)")
    return a


# ------------------------------------------------------------------------------ launch
def resolve_world(args):
    """--gpus vs the torchrun environment. Returns the world size this process runs in, or
    re-executes the script under torchrun (never returns) when N > 1 ranks are requested
    from a plain `python bench.py --gpus N`."""
    env = os.environ.get("WORLD_SIZE")
    if env is not None:
        world = int(env)
        if args.gpus is not None and args.gpus != world:
            raise SystemExit(f"bench.py: --gpus {args.gpus} != WORLD_SIZE {world}")
        args.gpus = world
        return world
    n = 1 if args.gpus is None else args.gpus
    if n < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    args.gpus = n
    if n == 1:
        return 1
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < n:
            print(f"bench.py: --gpus {n} but only {have} CUDA device(s) visible", file=sys.stderr)
            raise SystemExit(2)
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


# ------------------------------------------------------------------------------ helpers
def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{index}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        load = [s for s, p in zip(sm, power) if p > 200] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------------------ workload
def rollout_chunks(seq_offsets, max_rows):
    """Greedy chunks of whole rollouts with ≤ max_rows rows each (single-pass mode needs
    rollout-aligned chunks); a rollout longer than max_rows is an error."""
    so = [int(x) for x in seq_offsets]
    chunks, b = [], 0
    for i in range(1, len(so)):
        if so[i] - so[i - 1] > max_rows:
            raise SystemExit(f"rollout {i - 1} has {so[i] - so[i - 1]} rows > chunk {max_rows}")
        if so[i] - b > max_rows:
            chunks.append((b, so[i - 1]))
            b = so[i - 1]
    if so[-1] > b:
        chunks.append((b, so[-1]))
    return chunks


def strong_plan(w, seed, world):
    """Strong scaling: the global layout/rewards (identical on every rank) and the LPT plan."""
    from paper_2512_07710_b200.sharding import plan_shards
    group_ids, seq_offsets = S.make_layout(w, seed)
    rewards = S.make_rewards(w, seed)
    plan = plan_shards(group_ids, seq_offsets, world, rewards=rewards)
    return group_ids, seq_offsets, rewards, plan


def group_chunks(local_so, local_gid, Rc):
    """Chunks of ≤ Rc rows that never cross a prompt group and start at multiples of Rc
    inside their group: a row at offset o in its group reads buffer row o mod Rc, whatever
    other groups the rank holds."""
    from paper_2512_07710_b200.sharding import group_spans
    chunks = []
    for a, b in group_spans(local_gid):
        g0, g1 = int(local_so[a]), int(local_so[b])
        chunks += [(x, min(g1, x + Rc)) for x in range(g0, g1, Rc)]
    return chunks


def make_batch(w, seed, dev, buffer_rows, log, single_pass=False, shard=None,
               drift=(0.01, 0.02), bufs=None):
    """Device-resident synthetic batch: chunk buffer + per-token arrays. shard = (world,
    rank): strong scaling, this rank's groups of the global batch (seed shared by all ranks).
    bufs = (buf, buf_tok, buf_lp) of an earlier call with the same seed: reused, not redrawn."""
    import torch
    V = w.V
    t0 = time.time()
    if shard is None:
        group_ids, seq_offsets = S.make_layout(w, seed)
        rewards = S.make_rewards(w, seed)
        g_so, rows_global = seq_offsets, None
    else:
        world, rank = shard
        from paper_2512_07710_b200.sharding import shard_batch
        g_gid, g_so, g_rw, plan = strong_plan(w, seed, world)
        rollouts, _, group_ids, seq_offsets = shard_batch(plan[rank], g_gid, g_so)
        rewards = g_rw[rollouts]
        # global row of each local rollout's first row (for the per-token drift and digest)
        rows_global = (rollouts, g_so)
    T = int(seq_offsets[-1])
    if shard is None:
        Rc = max(1, min(buffer_rows, T))
    else:                       # the same buffer for every N: bounded by the largest group
        from paper_2512_07710_b200.sharding import group_spans
        Rc = max(1, min(buffer_rows, max(int(g_so[b] - g_so[a]) for a, b in group_spans(g_gid))))
    if bufs is not None:
        buf, buf_tok, buf_lp = bufs
        assert buf.shape[0] == Rc
    else:
        buf = S.make_logit_rows_torch(Rc, V, seed, dev, torch.bfloat16)
        buf_tok = S.sample_tokens_gumbel_torch(buf, seed)
        # bench setup only (untimed): rollout-engine log-probs = log_softmax + drift
        buf_lp = torch.empty(Rc, dtype=torch.float32, device=dev)
        for r0 in range(0, Rc, 2048):
            r1 = min(Rc, r0 + 2048)
            ls = torch.log_softmax(buf[r0:r1].float(), dim=1)
            buf_lp[r0:r1] = ls.gather(1, buf_tok[r0:r1].long().unsqueeze(1)).squeeze(1)
            del ls
    # chunks: fixed R_c tiles (two sweeps), R_c tiles of each group (strong scaling) or
    # whole-rollout packs (single pass); batch row t reads buffer row t − (its chunk's first row)
    if single_pass:
        chunks = rollout_chunks(seq_offsets, Rc)
    elif shard is not None:
        chunks = group_chunks(seq_offsets, group_ids, Rc)
    else:
        chunks = [(b, min(T, b + Rc)) for b in range(0, T, Rc)]
    idx_np = np.empty(T, dtype=np.int64)
    for b, e in chunks:
        idx_np[b:e] = np.arange(e - b)
    idx = torch.from_numpy(idx_np).to(dev)
    tokens = buf_tok[idx].contiguous()
    lp = buf_lp[idx]
    # drift: per-rollout b_i and per-token noise, drawn over the GLOBAL batch (the same on
    # every rank and for every N in strong mode), then this rank's rows gathered
    g = torch.Generator(device=dev)
    g.manual_seed(seed & ((1 << 62) - 1))
    Tg = int(g_so[-1]) if shard is not None else T
    Rg = len(g_so) - 1
    lengths = torch.from_numpy(np.diff(g_so)).to(dev)
    b = torch.repeat_interleave(torch.randn(Rg, generator=g, device=dev) * drift[0], lengths)
    drift_g = b + drift[1] * torch.randn(Tg, generator=g, device=dev)
    if shard is not None:
        rl, gso = rows_global
        starts = torch.from_numpy(gso[rl]).to(dev)
        lens = torch.from_numpy(gso[rl + 1] - gso[rl]).to(dev)
        first_local = torch.from_numpy(seq_offsets[:-1]).to(dev)
        roll = torch.repeat_interleave(torch.arange(len(rl), device=dev), lens)
        grow = starts[roll] + (torch.arange(T, device=dev) - first_local[roll])
        drift_l = drift_g[grow]
        del drift_g
    else:
        grow = None
        drift_l = drift_g
    old = (lp + drift_l).contiguous()
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)
    log(f"generated batch T={T} buffer={Rc} rows, {len(chunks)} chunks in {time.time() - t0:.1f}s")
    return dict(buf=buf, tokens=tokens, old=old, T=T, Rc=Rc, buf_tok=buf_tok, buf_lp=buf_lp,
                drift=drift_l, chunks=chunks, global_row=grow,
                rewards=torch.from_numpy(rewards).to(dev),
                group_ids=torch.from_numpy(group_ids).to(dev),
                seq_offsets=torch.from_numpy(seq_offsets).to(dev),
                np=dict(rewards=rewards, group_ids=group_ids, seq_offsets=seq_offsets,
                        chunk_of_row=None))


def chunk_digest(dlog_rows, grow_rows):
    """Order-independent 64-bit digest of dlogits rows (bit patterns) with their global ids."""
    import torch
    w32 = dlog_rows.view(torch.int32)
    s1 = w32.sum(1, dtype=torch.int64).cpu().numpy().astype(np.uint64)
    s2 = w32[:, ::7].sum(1, dtype=torch.int64).cpu().numpy().astype(np.uint64)
    gid = grow_rows.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = gid * np.uint64(0x9E3779B97F4A7C15) ^ s1 * np.uint64(0xBF58476D1CE4E5B9) ^ \
            s2 * np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
        x *= np.uint64(0xD6E8FEB86659FD93)
        x ^= x >> np.uint64(32)
        return int(x.sum(dtype=np.uint64))


def emulate_ranks(args, w, dev, log):
    """`--emulate-ranks N` (strong scaling on ONE GPU, for evidence only — not a multi-GPU
    measurement): the N ranks' shards of the global batch run one after another on this GPU,
    each on its own context; the one exchange of the pass is done with the split finalize
    (every rank's espo_loss_reduce_local vector summed on the device, then
    espo_loss_finalize_reduced on each rank), so every rank's dlogits rows are those a real
    N-GPU run computes. Per rank, its step (fwd sweeps + reduce_local, then finalize_reduced +
    bwd sweeps) is timed with CUDA events; the projected N-GPU step = the slowest rank's time
    (the NCCL all-reduce of 26 doubles, ~10-20 µs, is not included). Prints one JSON line."""
    import torch
    from paper_2512_07710_b200.espo import REDUCE_LEN, Espo, stats_to_dict
    N = args.emulate_ranks
    seed = S.config_seed(w.index)
    ranks, bufs = [], None
    for r in range(N):
        d = make_batch(w, seed, dev, args.buffer_rows, log, shard=(N, r),
                       drift=(args.drift_seq, args.drift_tok), bufs=bufs)
        bufs = (d["buf"], d["buf_tok"], d["buf_lp"])
        ctx = Espo(w.V, logits_dtype=torch.bfloat16, device=dev.index)
        ranks.append((d, ctx))
    dlog = torch.empty((bufs[0].shape[0], w.V), dtype=torch.bfloat16, device=dev)
    red = torch.zeros(REDUCE_LEN, dtype=torch.float64, device=dev)

    def step(times=None, digest=None):
        parts = []
        for r, (d, ctx) in enumerate(ranks):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.prepare(d["rewards"], d["group_ids"], d["seq_offsets"], n_tokens=d["T"])
            for b, e in d["chunks"]:
                ctx.loss_fwd(d["buf"][:e - b], d["tokens"][b:e], d["old"][b:e], None, row_begin=b)
            parts.append(ctx.loss_reduce_local())
            e1.record()
            if times is not None:
                times[r].append((e0, e1))
        red.zero_()
        for p_ in parts:                          # the all-reduce, in rank order
            red.add_(p_)
        out = None
        for r, (d, ctx) in enumerate(ranks):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            loss, stats = ctx.loss_finalize_reduced(red)
            for b, e in d["chunks"]:
                ctx.loss_bwd(d["buf"][:e - b], dlog[:e - b], row_begin=b)
                if digest is not None:
                    gid = d["global_row"][b:e].cpu().numpy()
                    digest[0] = (digest[0] + chunk_digest(dlog[:e - b], gid)) & ((1 << 64) - 1)
            e1.record()
            if times is not None:
                times[r].append((e0, e1))
            out = (loss, stats)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    times = [[] for _ in range(N)]
    for _ in range(args.steps):
        loss, stats = step(times)
    torch.cuda.synchronize(dev)
    per_rank = [sum(a.elapsed_time(b) for a, b in t) / args.steps for t in times]
    for _, ctx in ranks:
        ctx.get_error()
    digest = [0]
    if args.verify:
        step(digest=digest)
        torch.cuda.synchronize(dev)
    T_total = sum(d["T"] for d, _ in ranks)
    ms = max(per_rank)
    st = stats_to_dict(stats)
    out = {"metric": "ESPO loss fwd+bwd tokens/sec (projected from emulated ranks)",
           "value_projected": T_total / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1,
           "emulated_ranks": N, "steps": args.steps, "warmup": args.warmup,
           "scaling": "strong (emulated: ranks run one after another on one GPU)",
           "ms_per_step_max_rank": ms, "ms_per_rank": per_rank,
           "rank_tokens": [d["T"] for d, _ in ranks],
           "imbalance_max_over_mean": ms / (sum(per_rank) / N),
           "loss_f64": st["loss"],
           "dlogits_digest": ("%016x" % digest[0]) if args.verify else None,
           "config": {"workload": f"{w.name} global batch split over {N} emulated ranks (LPT plan)",
                      "global_batch_tokens": T_total, "drift": {"seq_sigma": args.drift_seq}},
           "note": "evidence of load balance and of N-independent results (dlogits digest, loss) "
                   "of the strong-scaling path; not a multi-GPU measurement"}
    print(json.dumps(out), flush=True)
    for _, ctx in ranks:
        ctx.close()


def dlogits_digest(ctx, d, dlog, log):
    """Untimed verification pass (--verify): one more full step; after each backward chunk,
    per-row sums of the dlogits bits (all elements, and every 7th 32-bit word) are mixed with
    the row's GLOBAL id and summed mod 2^64. The sum is order-independent, so rank digests
    add up (all-reduce) to the digest one GPU would print for the same global batch."""
    import torch
    T, buf = d["T"], d["buf"]
    ctx.prepare(d["rewards"], d["group_ids"], d["seq_offsets"], n_tokens=T)
    for b, e in d["chunks"]:
        ctx.loss_fwd(buf[:e - b], d["tokens"][b:e], d["old"][b:e], None, row_begin=b)
    loss, stats = ctx.loss_finalize()
    acc = 0
    grow = d["global_row"]
    for b, e in d["chunks"]:
        ctx.loss_bwd(buf[:e - b], dlog[:e - b], row_begin=b)
        gid = np.arange(b, e, dtype=np.int64) if grow is None else grow[b:e].cpu().numpy()
        acc = (acc + chunk_digest(dlog[:e - b], gid)) & ((1 << 64) - 1)
    ctx.get_error()
    return int(acc), loss, stats


def run_step(ctx, d, dlog, ev=None):
    """One full pass. ev: optional dict of lists to record per-call CUDA events."""
    import torch
    T, Rc, buf = d["T"], d["Rc"], d["buf"]
    ctx.prepare(d["rewards"], d["group_ids"], d["seq_offsets"], n_tokens=T)
    for b, e in d["chunks"]:
        if ev is not None:
            s0 = torch.cuda.Event(enable_timing=True)
            s0.record()
        ctx.loss_fwd(buf[:e - b], d["tokens"][b:e], d["old"][b:e], None, row_begin=b)
        if ev is not None:
            s1 = torch.cuda.Event(enable_timing=True)
            s1.record()
            ev["fwd"].append((s0, s1))
    loss, stats = ctx.loss_finalize()
    for b, e in d["chunks"]:
        if ev is not None:
            s0 = torch.cuda.Event(enable_timing=True)
            s0.record()
        ctx.loss_bwd(buf[:e - b], dlog[:e - b], row_begin=b)
        if ev is not None:
            s1 = torch.cuda.Event(enable_timing=True)
            s1.record()
            ev["bwd"].append((s0, s1))
    return loss, stats


class ShardedStep:
    """Vocabulary-parallel leg on one GPU: S contexts, shard k owns columns [v0_k, v0_k + w_k)
    of the same chunk buffer (a column view with the full row pitch); per chunk: S partial
    sweeps → gathered partials (one device tensor) → S combines; after finalize, S backward
    sweeps each writing its columns of the dlogits buffer."""

    def __init__(self, ctxs, shards, Rc, dev, p2p=False):
        import torch
        self.ctxs, self.shards, self.p2p = ctxs, shards, p2p
        self.part = torch.empty((len(ctxs), Rc, 4), dtype=torch.float32, device=dev)
        if p2p:
            for c in ctxs:
                c.tp_p2p_buffer(Rc, len(ctxs))
            for k, c in enumerate(ctxs):
                c.tp_p2p_connect_local(ctxs, k)

    @property
    def launch_count(self):
        return sum(c.launch_count for c in self.ctxs)

    def get_error(self):
        for c in self.ctxs:
            c.get_error()

    def close(self):
        for c in self.ctxs:
            c.close()


def run_step_sharded(sh, d, dlog, ev=None):
    import torch
    T, Rc, buf = d["T"], d["Rc"], d["buf"]
    for c in sh.ctxs:
        c.prepare(d["rewards"], d["group_ids"], d["seq_offsets"], n_tokens=T)
    for b in range(0, T, Rc):
        e = min(T, b + Rc)
        if ev is not None:
            s0 = torch.cuda.Event(enable_timing=True)
            s0.record()
        if sh.p2p:     # fused: each sweep stores its partials into every rank's buffer
            for c, (v0, w) in zip(sh.ctxs, sh.shards):
                c.loss_fwd_p2p_send(buf[:e - b, v0:v0 + w], d["tokens"][b:e], d["old"][b:e],
                                    None, row_begin=b)
            for c in sh.ctxs:
                c.loss_fwd_p2p_recv(b, e - b)
        else:
            for k, (c, (v0, w)) in enumerate(zip(sh.ctxs, sh.shards)):
                c.loss_fwd_partial(buf[:e - b, v0:v0 + w], d["tokens"][b:e], d["old"][b:e], None,
                                   row_begin=b, partial=sh.part[k, :e - b])
            for c in sh.ctxs:
                c.loss_fwd_combine(sh.part[:, :e - b], row_begin=b)
        if ev is not None:
            s1 = torch.cuda.Event(enable_timing=True)
            s1.record()
            ev["fwd"].append((s0, s1))
    outs = [c.loss_finalize() for c in sh.ctxs]
    for b in range(0, T, Rc):
        e = min(T, b + Rc)
        if ev is not None:
            s0 = torch.cuda.Event(enable_timing=True)
            s0.record()
        for c, (v0, w) in zip(sh.ctxs, sh.shards):
            c.loss_bwd(buf[:e - b, v0:v0 + w], dlog[:e - b, v0:v0 + w], row_begin=b)
        if ev is not None:
            s1 = torch.cuda.Event(enable_timing=True)
            s1.record()
            ev["bwd"].append((s0, s1))
    return outs[0]


def run_step_single(ctx, d, dlog, ev=None):
    """Single-pass step: prepare → set_mask → fwd_bwd per chunk of whole rollouts → finalize.
    ev["fwdbwd"] gets one event pair per chunk."""
    import torch
    buf = d["buf"]
    ctx.prepare(d["rewards"], d["group_ids"], d["seq_offsets"], n_tokens=d["T"])
    ctx.set_mask(None)
    for b, e in d["chunks"]:
        if ev is not None:
            s0 = torch.cuda.Event(enable_timing=True)
            s0.record()
        ctx.loss_fwd_bwd(buf[:e - b], d["tokens"][b:e], d["old"][b:e], dlog[:e - b], row_begin=b)
        if ev is not None:
            s1 = torch.cuda.Event(enable_timing=True)
            s1.record()
            ev["fwdbwd"].append((s0, s1))
    return ctx.loss_finalize()


def run_step_factored(ctx, d, dlog, ev=None):
    """Factored-gradient step: prepare → espo_loss_fwd_factored per chunk (statistics + the
    row factor G = onehot − p into dlog, one sweep) → finalize → espo_loss_row_scale (the
    per-row scale a consumer applies in its GEMM). ev["fwdbwd"] gets one pair per chunk."""
    import torch
    buf = d["buf"]
    ctx.prepare(d["rewards"], d["group_ids"], d["seq_offsets"], n_tokens=d["T"])
    for b, e in d["chunks"]:
        if ev is not None:
            s0 = torch.cuda.Event(enable_timing=True)
            s0.record()
        ctx.loss_fwd_factored(buf[:e - b], d["tokens"][b:e], d["old"][b:e], None,
                              grad=dlog[:e - b], row_begin=b)
        if ev is not None:
            s1 = torch.cuda.Event(enable_timing=True)
            s1.record()
            ev["fwdbwd"].append((s0, s1))
    out = ctx.loss_finalize()
    if "scale" not in d:
        d["scale"] = torch.empty(d["T"], dtype=torch.float32, device=buf.device)
    ctx.loss_row_scale(out=d["scale"])
    return out


def run_e2e(ctx, d, dlog, args, dev):
    """End-to-end through the public API with HOST inputs: every step copies its inputs
    (rewards, group ids, offsets, tokens, old log-probs and every logits chunk) from pinned
    host memory and reads the loss back. Logits stream through a pinned host ring of
    --e2e-host-rows rows in chunks of whole rollouts; copies run on a side stream,
    double-buffered against the kernels. single-pass (default): each chunk crosses PCIe once
    (espo_set_mask + espo_loss_fwd_bwd); two-sweep: once for the forward and again for the
    backward sweep."""
    import torch
    T, V = d["T"], d["buf"].shape[1]
    Hr = min(args.e2e_host_rows, d["Rc"])
    chunks = rollout_chunks(d["np"]["seq_offsets"], Hr)
    host = torch.empty((Hr, V), dtype=torch.bfloat16, pin_memory=True)
    host.copy_(d["buf"][:Hr].cpu())
    # batch row t reads host ring row t − (its chunk's first row): tokens / old follow it
    idx_np = np.empty(T, dtype=np.int64)
    for b, e in chunks:
        idx_np[b:e] = np.arange(e - b)
    idx = torch.from_numpy(idx_np).to(dev)
    h_tok = d["buf_tok"][idx].cpu().pin_memory()
    h_old = (d["buf_lp"][idx] + d["drift"]).cpu().pin_memory()
    h_rw = d["rewards"].cpu().pin_memory()
    h_gid = d["group_ids"].cpu().pin_memory()
    h_so = d["seq_offsets"].cpu().pin_memory()
    stage = [torch.empty((Hr, V), dtype=torch.bfloat16, device=dev) for _ in range(2)]
    d_tok = torch.empty_like(d["tokens"])
    d_old = torch.empty_like(d["old"])
    d_rw, d_gid, d_so = (torch.empty_like(d[k]) for k in ("rewards", "group_ids", "seq_offsets"))
    h_loss = torch.empty(1, dtype=torch.float32, pin_memory=True)
    copy_s = torch.cuda.Stream(dev)
    comp = torch.cuda.current_stream(dev)
    single = args.e2e_mode == "single-pass"

    def one_step():
        h2d = 0
        for dst, src in ((d_rw, h_rw), (d_gid, h_gid), (d_so, h_so), (d_tok, h_tok), (d_old, h_old)):
            dst.copy_(src, non_blocking=True)
            h2d += src.numel() * src.element_size()
        ctx.prepare(d_rw, d_gid, d_so, n_tokens=T)
        if single:
            ctx.set_mask(None)
        done = [torch.cuda.Event() for _ in range(2)]
        for sweep in (("fwdbwd",) if single else ("fwd", "bwd")):
            if sweep == "bwd":
                loss, _ = ctx.loss_finalize()
            used = [None, None]
            for k, (b, e) in enumerate(chunks):
                sb = stage[k % 2]
                with torch.cuda.stream(copy_s):
                    if used[k % 2] is not None:
                        copy_s.wait_event(used[k % 2])
                    sb[:e - b].copy_(host[:e - b], non_blocking=True)
                    done[k % 2].record(copy_s)
                h2d += (e - b) * V * 2
                comp.wait_event(done[k % 2])
                if sweep == "fwd":
                    ctx.loss_fwd(sb[:e - b], d_tok[b:e], d_old[b:e], None, row_begin=b)
                elif sweep == "bwd":
                    ctx.loss_bwd(sb[:e - b], dlog[:e - b], row_begin=b)
                else:
                    ctx.loss_fwd_bwd(sb[:e - b], d_tok[b:e], d_old[b:e], dlog[:e - b], row_begin=b)
                ev = torch.cuda.Event()
                ev.record(comp)
                used[k % 2] = ev
        if single:
            loss, _ = ctx.loss_finalize()
        h_loss.copy_(loss, non_blocking=True)
        return h2d, 4

    one_step()                         # warm-up
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        h2d, d2h = one_step()
    torch.cuda.synchronize(dev)
    dt = (time.perf_counter() - t0) / args.e2e_steps
    return T / dt, h2d, d2h, dt


def cpu_baseline(d, w, n_tok_per_rollout, log):
    """The oracle, as it stands, on a bounded sample of the same workload: the first prompt
    group that is not eliminated (G rollouts), truncated to the first n tokens of each rollout, fwd (O1-O6) + dlogits
    (O7) for every sampled row, on this host."""
    import torch
    from oracle import espo_oracle as O
    G, V = w.G, w.V
    L = n_tok_per_rollout
    so = d["np"]["seq_offsets"]
    rw_all = d["np"]["rewards"].reshape(-1, G)
    g0 = next(g for g in range(rw_all.shape[0]) if rw_all[g].min() != rw_all[g].max())
    rows = np.concatenate([np.arange(so[i], so[i] + L) for i in range(g0 * G, (g0 + 1) * G)])
    bufrows = rows % d["Rc"]
    z = d["buf"][torch.from_numpy(bufrows).to(d["buf"].device)].float().cpu().numpy()
    tok = d["tokens"][torch.from_numpy(rows).to(d["buf"].device)].cpu().numpy()
    old = d["old"][torch.from_numpy(rows).to(d["buf"].device)].cpu().numpy()
    rw = rw_all[g0]
    gid = np.zeros(G, np.int32)
    so_s = np.arange(G + 1, dtype=np.int64) * L
    cfg = O.OracleConfig(vocab=V, alpha=float(np.float32(0.4)), eps_min=float(np.float32(0.01)))
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):          # the oracle as it stands, on one core
        t0 = time.perf_counter()
        res = O.espo_loss(z, tok, old, None, rw, gid, so_s, cfg)
        for t in range(len(rows)):
            O.dlogits_row(res, t, z[t], int(tok[t]), cfg)
        dt = time.perf_counter() - t0
    n = len(rows)
    log(f"cpu oracle: {n} tokens in {dt:.1f}s")
    return {"value": n / dt, "unit": "tokens/s", "cores": 1, "kind": "oracle",
            "sample": f"prompt group {g0} of {w.name} (first non-zero-variance group): {G} "
                      f"rollouts x first {L} tokens = {n} "
                      f"tokens, V={V}, fwd (O1-O6) + dlogits (O7) of every row, numpy fp64, "
                      f"single thread; host has {len(os.sched_getaffinity(0))} cores",
            "seconds": dt}


def _oracle_worker(job):
    """One host process of cpu_baseline_parallel: builds its own seeded sample (one prompt
    group × L tokens per rollout, the espo_synth recipe), waits for the others, then times the
    oracle as it stands (fwd O1-O6 + dlogits O7 of every row) on one BLAS thread."""
    config, g, L, barrier = job
    from threadpoolctl import threadpool_limits
    from oracle import espo_oracle as O
    w = S.WORKLOADS[config]
    seed = S.config_seed(w.index) ^ (0x5151 + g)
    V, G = w.V, w.G
    rows = S.make_logit_rows(G * L, V, seed, dtype="bf16")
    tok = S.sample_tokens_gumbel(rows, seed)
    so = np.arange(G + 1, dtype=np.int64) * L
    cfg = O.OracleConfig(vocab=V, alpha=float(np.float32(0.4)), eps_min=float(np.float32(0.01)))
    with threadpool_limits(limits=1):
        lp = np.array([O.row_stats(rows[t], int(tok[t]))[1] for t in range(G * L)])
        old = S.drift_old_logp(lp, so, seed)
        rw = np.array([1.0, 0.0] * (G // 2) + [1.0] * (G % 2), np.float32)
        barrier.wait()
        t0 = time.perf_counter()
        res = O.espo_loss(rows, tok, old, None, rw, np.zeros(G, np.int32), so, cfg)
        for t in range(G * L):
            O.dlogits_row(res, t, rows[t], int(tok[t]), cfg)
        dt = time.perf_counter() - t0
    return G * L, dt


def cpu_baseline_parallel(config, L=48, max_procs=32):
    """The oracle on every host core: one process per core, each on its own prompt group
    (the pass is independent across groups up to the scalar normaliser), started together;
    throughput = all tokens ÷ the slowest process's time."""
    import multiprocessing as mp
    procs = max(1, min(max_procs, len(os.sched_getaffinity(0))))
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        barrier = m.Barrier(procs)
        with ctx.Pool(procs) as pool:
            out = pool.map(_oracle_worker, [(config, g, L, barrier) for g in range(procs)])
    n = sum(o[0] for o in out)
    dt = max(o[1] for o in out)
    w = S.WORKLOADS[config]
    return {"value": n / dt, "unit": "tokens/s", "cores": procs, "kind": "oracle",
            "sample": f"{procs} processes x one {w.name}-shaped prompt group each ({w.G} rollouts "
                      f"x {L} tokens, V={w.V}, seeded espo_synth rows), fwd (O1-O6) + dlogits "
                      f"(O7) of every row, numpy fp64, one BLAS thread per process, started on "
                      f"a barrier; tokens / slowest process time"}


# ------------------------------------------------------------------------------ main arms
def main_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2512_07710_b200.espo import (Espo, OPT_BLOCKS_PER_SM, OPT_BWD_IMPL,
                                            OPT_FACTORED_IMPL, OPT_FWD_IMPL, stats_to_dict)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.device_count() <= local:
        print(f"bench.py: rank {rank} needs cuda:{local}, {torch.cuda.device_count()} visible",
              file=sys.stderr)
        raise SystemExit(2)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # NCCL logs "nranks N" at init
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    log = (lambda m: print(f"[bench r{rank}] {m}", file=sys.stderr, flush=True))
    w = S.WORKLOADS[args.config]
    if args.emulate_ranks > 0:
        if world != 1:
            raise SystemExit("--emulate-ranks runs on one process")
        emulate_ranks(args, w, dev, log)
        return
    strong = args.scaling == "strong"
    if strong and (args.single_pass or args.vocab_shards > 1):
        raise SystemExit("--scaling strong runs the two-sweep (or --factored) path")
    # weak: every rank draws its own batch; strong: one global batch, the same seed everywhere
    seed = S.config_seed(w.index) ^ (0 if strong else rank * 0x9E3779B9)
    d = make_batch(w, seed, dev, args.buffer_rows, log, single_pass=args.single_pass,
                   shard=(world, rank) if strong else None, drift=(args.drift_seq, args.drift_tok))
    kw = dict(zero_fill_inactive_rows=not args.compact,
              zv_mode=1 if args.zv_mode == "rlzvp" else 0)
    S_ = args.vocab_shards
    if S_ > 1:
        if world > 1:
            raise SystemExit("--vocab-shards is a single-GPU leg")
        wd = [((w.V * (k + 1) // S_) // 8 * 8) - ((w.V * k // S_) // 8 * 8) for k in range(S_)]
        wd[-1] = w.V - sum(wd[:-1])
        shards = [(sum(wd[:k]), wd[k]) for k in range(S_)]
        ctxs = [Espo(w.V, logits_dtype=torch.bfloat16, device=local, vocab_shard=sh, **kw)
                for sh in shards]
        for c in ctxs:
            c.set_option(OPT_FWD_IMPL, args.fwd_impl)
            c.set_option(OPT_BWD_IMPL, args.bwd_impl)
        ctx = ShardedStep(ctxs, shards, d["Rc"], dev, p2p=args.tp_p2p)
        step_fn = run_step_sharded
    else:
        ctx = Espo(w.V, logits_dtype=torch.bfloat16, device=local, rank=rank, world=world, **kw)
        nranks = ctx.comm_size
        log(f"DP communicator: nranks={nranks} (world {world}, rank {rank}, cuda:{local})")
        if nranks != world:
            raise SystemExit(f"bench.py: NCCL communicator has {nranks} ranks, world is {world}")
        ctx.set_option(OPT_FWD_IMPL, args.fwd_impl)
        ctx.set_option(OPT_BWD_IMPL, args.bwd_impl)
        ctx.set_option(OPT_BLOCKS_PER_SM, args.blocks_per_sm)
        ctx.set_option(OPT_FACTORED_IMPL, args.factored_impl)
        step_fn = (run_step_factored if args.factored else
                   run_step_single if args.single_pass else run_step)
    dlog = torch.empty((d["Rc"], w.V), dtype=torch.bfloat16, device=dev)

    for _ in range(args.warmup):
        step_fn(ctx, d, dlog)
    ctx.get_error()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev = {"fwd": [], "bwd": [], "fwdbwd": []}
    launches0 = ctx.launch_count
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    start.record()
    for _ in range(args.steps):
        loss, stats = step_fn(ctx, d, dlog, ev)
    end.record()
    torch.cuda.synchronize(dev)
    launches = ctx.launch_count - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = start.elapsed_time(end)
    ctx.get_error()
    st = stats_to_dict(stats)
    t_ms = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_step = float(t_ms.item()) / args.steps
    t_all = torch.tensor([d["T"]], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t_all)
    T_total = int(t_all.item())             # tokens all ranks processed per step

    # algorithmic bytes (per rank, per step); SURVEY §8(d) per-row figures
    V, T = w.V, d["T"]
    n_act = st["n_active_tokens"] / world      # stats are global (all-reduced): per-rank mean
    n_clip = st["n_clipped_tokens"] / world
    fwd_bytes = n_act * (2 * V + 4 + 4 + 16) + T * (4 + 4 + 1 + 8)
    bwd_bytes = (n_act - n_clip) * 2 * V + (0 if args.compact else T) * 2 * V + T * 12
    if args.compact:
        bwd_bytes += (n_act - n_clip) * 2 * V      # swept rows are still written
    step_bytes = fwd_bytes + bwd_bytes
    if args.factored:          # one sweep: read valid rows once, write G (or zeros) per row
        step_bytes = n_act * (2 * V + 4 + 4 + 16) + T * (4 + 4 + 1 + 8 + 9) + \
            (n_act if args.compact else T) * 2 * V
        bwd_bytes = step_bytes
    fused = args.single_pass or args.factored
    peak, peak_src = measured_peaks()
    if fused:                  # one event pair per fused chunk: report the fused chunk
        fb_ms = statistics.mean(a.elapsed_time(b) for a, b in ev["fwdbwd"])
        n_chunks = len(ev["fwdbwd"]) // args.steps
        fwd_ms = bwd_ms = fb_ms
        fwd_gbs = bwd_gbs = step_bytes / n_chunks / (fb_ms * 1e-3) / 1e9
    else:
        fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in ev["fwd"])
        bwd_ms = statistics.mean(a.elapsed_time(b) for a, b in ev["bwd"])
        n_chunks = len(ev["bwd"]) // args.steps
        bwd_gbs = bwd_bytes / n_chunks / (bwd_ms * 1e-3) / 1e9
        fwd_gbs = fwd_bytes / n_chunks / (fwd_ms * 1e-3) / 1e9
    step_gbs = step_bytes / (ms_step * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    # ncu DRAM bytes of the dominant kernel, captured on the default C1 step (profiles/): only
    # for that workload; per launch for this run's chunking (the step's bytes do not depend
    # on how the rows are cut into calls)
    if os.path.exists(tpath) and args.config == "C1" and S_ == 1 and not args.compact and \
            args.zv_mode == "mask" and not args.single_pass:
        tr = json.load(open(tpath))
        key = "factored" if args.factored else "bwd"
        per, nl = tr.get(f"{key}_bytes_per_launch"), tr.get(f"{key}_launches")
        if per is not None and nl:
            traffic = per * nl / (n_chunks * world if strong else n_chunks)

    # the same workload through the factored-gradient API (one sweep per row; the consumer
    # applies the row scale), reported beside the headline — not in place of it
    factored = None
    if not (args.factored or args.single_pass or args.no_factored_leg) and S_ == 1:
        for _ in range(2):
            run_step_factored(ctx, d, dlog)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            run_step_factored(ctx, d, dlog)
        f1.record()
        torch.cuda.synchronize(dev)
        ctx.get_error()
        t_f = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_f, op=dist.ReduceOp.MAX)
        f_ms = float(t_f.item()) / args.steps
        f_bytes = n_act * (2 * V + 4 + 4 + 16) + T * (4 + 4 + 1 + 8 + 9) + \
            (n_act if args.compact else T) * 2 * V
        factored = {"value": T_total / (f_ms * 1e-3), "unit": "tokens/s", "ms_per_step": f_ms,
                    "achieved_hbm_gbs_step": f_bytes / (f_ms * 1e-3) / 1e9,
                    "api": "espo_loss_fwd_factored + espo_loss_row_scale (dlogits = scale_t * G_t, "
                           "G = onehot - softmax written by the statistics sweep; the consumer "
                           "applies scale_t)"}

    e2e = None
    if not args.no_e2e and S_ == 1:
        tps, h2d, d2h, dt = run_e2e(ctx, d, dlog, args, dev)
        if world > 1:       # whole-job rate: every rank's tokens over the slowest rank's time
            t_e2e = torch.tensor([dt, h2d, d2h], dtype=torch.float64, device=dev)
            red = t_e2e.clone()
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
            dist.all_reduce(red)
            dt, h2d, d2h = float(t_e2e[0].item()), int(red[1].item()), int(red[2].item())
        tps = T_total / dt
        e2e = {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "mode": args.e2e_mode,
               "note": "host-resident inputs incl. every logits chunk over PCIe from a pinned "
                       "host ring (" + ("once per step: espo_set_mask + espo_loss_fwd_bwd on "
                       "chunks of whole rollouts" if args.e2e_mode == "single-pass" else
                       "twice per step: fwd and bwd sweeps") + "); wall clock over "
                       f"{args.e2e_steps} step(s) after one warm-up; dlogits stay on the device "
                       "(a trainer consumes them there: they are the input of the LM-head "
                       "backward), d2h is the loss"}
    cpu = cpu_par = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(d, w, args.cpu_sample_tokens, log)
        cpu.pop("seconds", None)
        try:
            cpu_par = cpu_baseline_parallel(args.config)
            log(f"cpu oracle on {cpu_par['cores']} cores: {cpu_par['value']:.0f} tokens/s")
        except Exception as e:          # the single-core baseline above stands on its own
            cpu_par = {"unavailable": f"{type(e).__name__}: {e}"}

    digest = None
    if args.verify:
        dg, vloss, vstats = dlogits_digest(ctx, d, dlog, log)
        dgt = torch.tensor([dg - (1 << 64) if dg >= (1 << 63) else dg], dtype=torch.int64,
                           device=dev)
        if world > 1:
            dist.all_reduce(dgt)            # int64 sum wraps mod 2^64, like the digest
        digest = {"dlogits_digest": "%016x" % (int(dgt.item()) & ((1 << 64) - 1)),
                  "loss_f64": stats_to_dict(vstats)["loss"],
                  "note": "order-independent hash of every dlogits row (bits) with its global "
                          "row id, summed over ranks; strong scaling: must not depend on N"}

    gname = (f"{w.name} global batch: {w.n_prompts} prompts x {w.G} rollouts x {w.L} tokens "
             f"split over {world} GPU(s) by prompt group (LPT plan)") if strong else \
        f"{w.name}: {w.n_prompts} prompts x {w.G} rollouts x {w.L} tokens per GPU"
    out = {
        "metric": "ESPO loss fwd+bwd tokens/sec (achieved HBM GB/s vs 8 TB/s in config)",
        "value": T_total / (ms_step * 1e-3),
        "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (espo_synth recipe: 80/20 entropy logits, Gumbel-sampled tokens, "
                "Bernoulli rewards, drifted old log-probs)",
        "config": {
            "workload": gname + f", vocab {V}, bf16 logits/grads" + (", compact dlogits" if args.compact else "")
                        + (", RL-ZVP advantages for zero-variance groups" if args.zv_mode == "rlzvp" else "")
                        + (f", {S_} vocabulary shards back to back on one GPU (TP emulation, "
                           + ("partials exchanged by the fused peer-memory path)" if args.tp_p2p
                              else "partials gathered by device copy)") if S_ > 1 else "")
                        + (", single-pass (espo_loss_fwd_bwd per chunk of whole rollouts)" if args.single_pass else "")
                        + (", factored gradient (espo_loss_fwd_factored: one sweep writes G = onehot - p; "
                           "dlogits = row_scale * G applied by the consumer)" if args.factored else ""),
            "global_batch_tokens": T_total, "seq_len": w.L,
            "parallelism": f"dp{world} (prompt-group sharded" + (", LPT plan)" if strong else ")"),
            "nccl_nranks": ctx.comm_size if S_ == 1 else 1,
            "drift": {"seq_sigma": args.drift_seq, "tok_sigma": args.drift_tok,
                      "clip_frac": n_clip / n_act if n_act else 0.0,
                      "note": "old_logp = lp + b_i + tok_sigma*n_t, b_i ~ N(0, seq_sigma); clipped "
                              "tokens need no logits read in the backward (c_t = 0)"},
            "chunk_rows": d["Rc"],
            "l2": (f"inputs larger than L2 (chunk buffer {d['Rc'] * V * 2 / 1e9:.2f} GB > 126 MB)"
                   if d["Rc"] * V * 2 > 126e6 else
                   f"inputs fit in L2 ({d['Rc'] * V * 2 / 1e6:.1f} MB): a parity-size config, "
                   "not a bench line"),
            "fwd_impl": ["tma16x2x6k_s4_f32x2 (rows >= 64 KB; 16x3x4k below)", "ldg", "tma16x2x7k_s2_f32x2", "tma14x2x7k_s2_f32x2", "tma20x2x5k_s2_f32x2", "tma16x3x4k_s4_f32x2", "tma16x2x6k_s4_poly1", "tma18x2x6k_s4_f32x2", "tma16x2x6k_s4_scalar", "tile32k_b4", "tile32k_b3", "tile32k_b2"][args.fwd_impl],
            "bwd_impl": ["tile32k_f32x2", "ldg", "tma16x3x4k", "tma16x2x4k", "tma12x4x4k", "tma8x6x4k", "tma8x4x4k", "tile16k", "tile32k_scalar", "tlist32k_r4", "tlist32k_r8", "tlist32k_r16"][args.bwd_impl],
            "achieved_hbm_gbs_step": step_gbs, "frac_of_8TBs_step": step_gbs / NOMINAL_HBM_GBS,
            "frac_of_measured_step": step_gbs / peak,
            "fwd_sweep_gbs": fwd_gbs, "fwd_sweep_ms_per_chunk": fwd_ms,
            "bwd_sweep_ms_per_chunk": bwd_ms,
            "active_tokens": n_act, "clipped_tokens": n_clip,
            "zv_groups": st["n_zv_groups"], "groups": st["n_groups"],
        },
        "roofline": {"bound": "hbm", "kernel": ("espo_loss_fwd_factored chunk (k_fwd_rows + k_fwd_grad)" if args.factored
                                                else "espo_loss_fwd_bwd chunk (K2 + K3 + K5)" if args.single_pass
                                                else "espo_loss_bwd sweep (k_bwd_recs + k_dlogits_tile)"),
                     "achieved": bwd_gbs, "peak": peak, "unit": "GB/s",
                     "frac": bwd_gbs / peak, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": bwd_bytes / n_chunks},
        "cpu_baseline": cpu,
        "cpu_baseline_all_cores": cpu_par,
        "e2e": e2e,
        "gpu_launches": launches,
        "factored_gradient": factored,
        "verify": digest,
        "clocks": clk,
        "loss": st["loss"],
    }
    if args.factored:
        out["config"]["factored_impl"] = ["ring 20+1 warps x 5 x 40 KB", "cta1024 L2 re-read",
                                          "ring 16+1 x 6 x 32 KB", "ring 20+1 x 5 x 40 KB + TMEM stash",
                                          "ring 10+1 x 5 x 20 KB, 2 CTAs/SM",
                                          "ring 12+1 x 4 x 24 KB, 2 CTAs/SM",
                                          "rolling 20+1 x 5 x 40 KB"][args.factored_impl]
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main_reference(args):
    """The CPU oracle on bounded samples of the same workload (rank 0 only)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle import espo_oracle as O
    w = S.WORKLOADS[args.config]
    seed = S.config_seed(w.index)
    V, G = w.V, w.G
    L = 32
    cfg = O.OracleConfig(vocab=V, alpha=float(np.float32(0.4)), eps_min=float(np.float32(0.01)))
    rewards = S.make_rewards(w, seed)

    def sample(step):
        rows = S.make_logit_rows(G * L, V, seed ^ (step + 1), dtype="bf16")
        tok = S.sample_tokens_gumbel(rows, seed ^ (step + 1))
        so = np.arange(G + 1, dtype=np.int64) * L
        lp = np.array([O.row_stats(rows[t], int(tok[t]))[1] for t in range(G * L)])
        old = S.drift_old_logp(lp, so, seed)
        g = step % w.n_prompts
        return rows, tok, old, rewards[g * G:(g + 1) * G], np.zeros(G, np.int32), so

    def step(data):
        rows, tok, old, rw, gid, so = data
        res = O.espo_loss(rows, tok, old, None, rw, gid, so, cfg)
        for t in range(rows.shape[0]):
            O.dlogits_row(res, t, rows[t], int(tok[t]), cfg)

    samples = [sample(i) for i in range(args.warmup + args.steps)]
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):          # one core, as "cores" reports
        for i in range(args.warmup):
            step(samples[i])
        t0 = time.perf_counter()
        for i in range(args.steps):
            step(samples[args.warmup + i])
        dt = (time.perf_counter() - t0) / args.steps
    n = G * L
    out = {
        "impl": "reference",
        "metric": "ESPO loss fwd+bwd tokens/sec (achieved HBM GB/s vs 8 TB/s in config)",
        "value": n / dt, "unit": "tokens/s", "n_gpus": args.gpus or 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{w.name}: bounded sample per step: one prompt group "
                               f"({G} rollouts) x {L} tokens, vocab {V}"},
        "cpu_baseline": {"value": n / dt, "unit": "tokens/s", "cores": 1, "kind": "oracle",
                         "sample": f"{G} rollouts x {L} tokens of {w.name} per step, fwd+dlogits, "
                                   "numpy fp64 single thread"},
        "e2e": {"value": n / dt, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    resolve_world(a)
    if a.impl == "reference":
        main_reference(a)
    else:
        main_ours(a)
