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
