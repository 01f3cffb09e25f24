"""Practical HBM ceilings on this B200 for the three traffic shapes of the pass: read-only
(torch.sum), write-only (zero_), copy (copy_), 10 GB bf16 buffers, CUDA events, best of 10."""
import json
import torch

n = 5 * 1024 ** 3  # elements (10 GiB bf16)
x = torch.randn(n // 4, device="cuda", dtype=torch.bfloat16).repeat(4)
y = torch.empty_like(x)
res = {}
for name, fn, nbytes in (("read_sum", lambda: x.sum(dtype=torch.float32), 2 * n),
                         ("write_zero", lambda: y.zero_(), 2 * n),
                         ("copy", lambda: y.copy_(x), 4 * n)):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    res[name] = nbytes / (best * 1e-3) / 1e9
print(json.dumps(res))
