"""bench.py's strong-scaling path on one GPU: the dlogits digest and the
loss of `--scaling strong --verify` must not depend on how many ranks the global batch is split
over. `--emulate-ranks N` runs the N ranks' shards one after another through the split
finalize (espo_loss_reduce_local → device-side sum → espo_loss_finalize_reduced), so its digest
must equal the N = 1 run's bit for bit (C0: variable group outcomes, a forced zero-variance
group, masked tails; C3: variable lengths, 60 % eliminated groups, bf16 at V = 151,936)."""
import json
import os
import subprocess
import sys

import pytest

from tests.gpu_common import require_cuda

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--scaling", "strong", "--verify",
           "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-factored-leg",
           *args]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("config,ranks", [("C0", (2, 3)), ("C3", (4,))])
def test_emulated_ranks_digest_equals_single_gpu(config, ranks):
    require_cuda()
    extra = ["--config", config] + (["--buffer-rows", "8192"] if config == "C3" else [])
    one = _bench(*extra)
    ref = one["verify"]["dlogits_digest"]
    for n in ranks:
        emu = _bench(*extra, "--emulate-ranks", str(n))
        assert emu["emulated_ranks"] == n and emu["n_gpus"] == 1
        assert emu["dlogits_digest"] == ref, (n, emu["dlogits_digest"], ref)
        assert emu["loss_f64"] == pytest.approx(one["verify"]["loss_f64"], rel=1e-12, abs=1e-15)
        assert sum(emu["rank_tokens"]) == one["config"]["global_batch_tokens"]
