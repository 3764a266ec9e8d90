"""Read-only HBM bandwidth on this B200, for context beside MEASURED_PEAKS.json's copy
figure (a copy moves 1 B read + 1 B written; the streaming passes are ~97 % reads).
torch reductions and a copy over 8 GB fp64 tensors, CUDA events, best of 10."""
import json

import torch

n = 1 << 30  # 8 GB of fp64
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)


def best(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    out = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out = max(out, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return out


res = {"sum_read_gbs": best(lambda: x.sum(), 8 * n),
       "amax_read_gbs": best(lambda: x.abs().max() if False else torch.amax(x), 8 * n),
       "copy_gbs": best(lambda: y.copy_(x), 16 * n)}
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
