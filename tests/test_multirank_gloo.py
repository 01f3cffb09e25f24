"""world_size-2 CPU tests (gloo) of the N > 1 host path: NCCL unique-id bootstrap over a
torch process group, deterministic prompt-group sharding, and sharding invariance of the one
all-reduce (loss and per-token gradient scale equal the single-rank oracle)."""
import multiprocessing as mp
import socket

import numpy as np
import pytest

from oracle import espo_oracle as O
from paper_2512_07710_b200.sharding import imbalance, plan_shards, shard_batch
from tests import mp_workers
from tests._instances import tiny_instance


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=180) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


def test_unique_id_bootstrap_over_gloo():
    out = run_world(mp_workers.worker_unique_id)
    assert all(n == 128 and same for _, n, same in out)


def test_sharded_reduction_matches_single_rank():
    out = run_world(mp_workers.worker_sharded_oracle)
    inst = tiny_instance(31, V=97, group_sizes=(4, 4, 3, 4, 2, 4, 1), L=9, mask_tail=3,
                         sigma_seq=0.1,
                         rewards=[1, 0, 0, 1, 1, 1, 1, 1, 0, 1, 0, 1, 0, 1, 1, 0.5, 0.5,
                                  0.25, 0.75, 0.2, 0, 1])
    ref = inst.run(O.OracleConfig(vocab=97))
    losses = [o[1] for o in out]
    assert losses[0] == losses[1]                     # every rank sees the same loss
    assert losses[0] == pytest.approx(ref.loss, rel=1e-12)
    v = np.array(out[0][2])
    assert v[1] == ref.stats["n_active_rollouts"] and v[2] == ref.stats["n_active_tokens"]
    assert v[3] == ref.stats["n_zv_groups"] and v[4] == ref.stats["n_groups"]
    # per-token gradient scale c_t / D on each rank == single-rank value, bitwise
    for _, _, _, toks, g, plans in out:
        assert np.array_equal(np.array(g), ref.coef[np.array(toks)] / ref.denom)
    assert out[0][5] == out[1][5]                     # identical plans on both ranks
    covered = sorted(sum(out[0][5][0], []))
    assert covered == list(range(7))


def test_plan_covers_groups_and_balances():
    rng = np.random.default_rng(3)
    G = 16
    lengths = np.clip(np.round(rng.lognormal(np.log(3000), 0.8, size=256 * G)), 64, 8192)
    so = np.zeros(256 * G + 1, np.int64)
    np.cumsum(lengths, out=so[1:])
    gid = np.repeat(np.arange(256, dtype=np.int32), G)
    rewards = (rng.uniform(size=256 * G) < 0.5).astype(np.float32)
    rewards[: 154 * G] = 1.0                          # 60 % eliminated groups, clustered
    for world in (2, 4, 8):
        lpt = plan_shards(gid, so, world, rewards=rewards)
        blk = plan_shards(gid, so, world, method="block")
        for plan in (lpt, blk):
            assert sorted(sum(plan, [])) == list(range(256))
        assert imbalance(lpt, gid, so, rewards) <= imbalance(blk, gid, so, rewards)
        assert imbalance(lpt, gid, so, rewards) < 1.02
        r, toks, lg, lso = shard_batch(lpt[0], gid, so)
        assert lso[-1] == len(toks) and len(lg) == len(r)
        assert np.all(np.diff(lg) >= 0)


def test_unique_id_bootstrap_over_subgroup():
    out = run_world(mp_workers.worker_subgroup_unique_id)
    assert out[1][1] == 128 and out[0][1] is None
    assert all(o[2] == 128 for o in out)


def _strong_rows(out):
    rows = {}
    for _, g, tok, old, bufrow, *_ in out:
        for t, y, o, b in zip(g, tok, old, bufrow):
            assert t not in rows                        # every global row on exactly one rank
            rows[t] = (y, o, b)
    return rows


def test_bench_strong_scaling_batch_is_independent_of_world():
    """bench.py --scaling strong, host side: the world-2 ranks together hold exactly the rows
    of the world-1 batch, each with the same token, old log-prob and logits buffer row — so
    the kernels see identical inputs per global row whatever N is."""
    one = _strong_rows(run_world(mp_workers.worker_bench_strong_batch, world=1))
    two_out = run_world(mp_workers.worker_bench_strong_batch, world=2)
    two = _strong_rows(two_out)
    assert sorted(two) == sorted(one) == list(range(len(one)))
    assert two == one
    for _, _, _, _, _, chunks, gid, so in two_out:    # chunks never cross a prompt group
        so = np.array(so)
        for b, e in chunks:
            r0 = int(np.searchsorted(so, b, side="right") - 1)
            r1 = int(np.searchsorted(so, e - 1, side="right") - 1)
            assert gid[r0] == gid[r1]
