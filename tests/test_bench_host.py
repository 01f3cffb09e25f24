"""Host-side pieces of bench.py (no GPU): rollout-aligned chunking for the single-pass and
e2e legs, and the all-cores oracle baseline (spawned processes, the oracle as it stands)."""
import numpy as np
import pytest

import bench


def test_rollout_chunks_cover_whole_rollouts():
    so = np.array([0, 5, 9, 20, 21, 30], dtype=np.int64)
    ch = bench.rollout_chunks(so, 12)
    assert ch[0][0] == 0 and ch[-1][1] == 30
    for (b0, e0), (b1, e1) in zip(ch, ch[1:]):
        assert e0 == b1                                   # contiguous, no overlap
    for b, e in ch:
        assert e - b <= 12 and b in so and e in so        # chunk borders are rollout borders
    with pytest.raises(SystemExit):
        bench.rollout_chunks(so, 8)                       # rollout 2 has 11 rows > 8


def test_cpu_baseline_all_cores_runs_the_oracle():
    r = bench.cpu_baseline_parallel("C0", L=4, max_procs=2)
    assert r["kind"] == "oracle" and r["unit"] == "tokens/s"
    assert 1 <= r["cores"] <= 2 and r["value"] > 0


def test_group_chunks_stay_inside_groups():
    gid = np.array([0, 0, 1, 1, 1, 2], dtype=np.int32)
    so = np.array([0, 7, 12, 20, 21, 33, 40], dtype=np.int64)
    ch = bench.group_chunks(so, gid, 8)
    assert ch == [(0, 8), (8, 12), (12, 20), (20, 28), (28, 33), (33, 40)]
    covered = np.zeros(40, int)
    for b, e in ch:
        covered[b:e] += 1
    assert np.all(covered == 1)


def test_resolve_world_rejects_mismatch(monkeypatch):
    from types import SimpleNamespace as NS
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.resolve_world(NS(gpus=4, impl="ours"))
    a = NS(gpus=None, impl="ours")
    assert bench.resolve_world(a) == 2 and a.gpus == 2
    monkeypatch.delenv("WORLD_SIZE")
    a = NS(gpus=None, impl="ours")
    assert bench.resolve_world(a) == 1 and a.gpus == 1


def test_launcher_spawns_ranks_for_gpus_n():
    """`bench.py --gpus 2` without torchrun re-executes itself under torch.distributed.run
    (the driver's launch); the reference arm prints one JSON line from rank 0 only, with
    n_gpus = 2 (CPU-only: that arm never touches a GPU)."""
    import json
    import os
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, bench.__file__, "--impl", "reference", "--gpus", "2",
                        "--config", "C0", "--steps", "1", "--warmup", "0"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2


def test_strong_plan_covers_every_group_once():
    import espo_synth as S
    w = S.WORKLOADS["C4"]
    seed = S.config_seed(w.index)
    for world in (1, 2, 4, 8):
        gid, so, rw, plan = bench.strong_plan(w, seed, world)
        assert sorted(sum(plan, [])) == list(range(w.n_prompts))
        loads = [sum(int(so[(g + 1) * w.G] - so[g * w.G]) for g in p) for p in plan]
        assert max(loads) - min(loads) <= 2 * w.G * w.L     # LPT: within two groups' rows


def test_chunk_digest_is_additive_over_row_splits():
    """--verify / --emulate-ranks: the digest of a row set is the mod-2^64 sum of the digests
    of any split of it (what makes rank digests comparable with the N = 1 digest), and it
    sees a one-ulp change in any row or a swapped pair of global ids."""
    import torch
    g = torch.Generator().manual_seed(3)
    z = torch.randn(37, 50, generator=g).to(torch.bfloat16)
    gid = np.arange(100, 137, dtype=np.int64)
    full = bench.chunk_digest(z, gid)
    perm = np.random.default_rng(0).permutation(37)
    a, b = perm[:11], perm[11:]
    parts = (bench.chunk_digest(z[torch.from_numpy(a)], gid[a]) +
             bench.chunk_digest(z[torch.from_numpy(b)], gid[b])) & ((1 << 64) - 1)
    assert parts == full
    z2 = z.clone()
    z2.view(torch.int16)[5, 7] += 1
    assert bench.chunk_digest(z2, gid) != full
    gid2 = gid.copy()
    gid2[[3, 4]] = gid2[[4, 3]]
    assert bench.chunk_digest(z, gid2) != full


def test_emulate_ranks_requires_strong_single_process(monkeypatch):
    monkeypatch.setattr("sys.argv", ["bench.py", "--emulate-ranks", "2"])
    with pytest.raises(SystemExit):
        bench.parse()                                     # weak scaling: rejected
    monkeypatch.setattr("sys.argv", ["bench.py", "--emulate-ranks", "2", "--scaling", "strong"])
    assert bench.parse().emulate_ranks == 2
