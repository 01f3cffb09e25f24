"""K2 on one 1/S-vocabulary shard: does the layout of the shard's rows matter? Times
espo_loss_fwd_partial (shard s of S, Rc rows, bf16, V = 151,936) on (a) a column view of a
full-width buffer (the bench's TP emulation: row pitch 2V), (b) a contiguous [Rc, w] tensor
(a real TP rank's shard), (c) contiguous with the pitch padded to 128 B. Interleaved rounds,
CUDA events. usage: python tools/tp_layout_probe.py [S] [Rc] [rounds] [fwd_impl]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import espo_synth as S  # noqa: E402
from paper_2512_07710_b200.espo import OPT_FWD_IMPL, Espo  # noqa: E402


def main(nsh=8, Rc=32768, rounds=5, impl=0, V=151936):
    dev = torch.device("cuda", 0)
    full = S.make_logit_rows_torch(Rc, V, 7, dev, torch.bfloat16)
    w = (V // nsh) // 8 * 8 if nsh > 1 else V
    v0 = w if nsh > 1 else 0                         # shard 1 (no target for most rows)
    tok = torch.randint(0, V, (Rc,), device=dev, dtype=torch.int32)
    old = torch.full((Rc,), -2.0, device=dev)
    so = torch.arange(0, Rc + 1, Rc // 8, device=dev, dtype=torch.int64)
    gid = torch.zeros(8, dtype=torch.int32, device=dev)
    rw = torch.tensor([1.0, 0.0] * 4, device=dev)
    views = {"column_view": full[:, v0:v0 + w]}
    views["contiguous"] = views["column_view"].contiguous()
    pad = torch.empty((Rc, (w + 63) // 64 * 64), dtype=torch.bfloat16, device=dev)
    pad[:, :w] = views["column_view"]
    views["pitch128"] = pad[:, :w]
    ctx = Espo(V, logits_dtype=torch.bfloat16, device=0, vocab_shard=(v0, w))
    ctx.set_option(OPT_FWD_IMPL, impl)
    part = torch.empty((Rc, 4), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    times = {k: [] for k in views}
    outs = {}
    for _ in range(rounds):
        for k, z in views.items():
            ctx.prepare(rw, gid, so, n_tokens=Rc)
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ctx.loss_fwd_partial(z, tok, old, None, partial=part)
            b.record()
            torch.cuda.synchronize()
            times[k].append(a.elapsed_time(b))
            outs[k] = part.clone()
    ctx.get_error()
    res = {k: {"ms": statistics.median(v), "GBs": Rc * w * 2 / statistics.median(v) / 1e6}
           for k, v in times.items()}
    res["same_partials"] = all(torch.equal(outs["column_view"], o) for o in outs.values())
    res["config"] = dict(shards=nsh, rows=Rc, width=w, impl=impl)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
