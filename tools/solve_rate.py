"""Per-iteration cost of the device solve loop (bmg_solve: V-cycle, residual
b - A x, partition-invariant norm, host-side stopping test) against bare V-cycles."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, Vector, default_params  # noqa
from paper_2509_06744_b200 import problems as pr  # noqa

cfg = pr.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
A, T, b = pr.make_problem(cfg)
H = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                    default_params(t_max=1, nest=cfg.nest, coarse_dim_cap=1 << 30))
bv = Vector(ctx, b)
x = Vector(ctx, b.size)
H.solve(cfg.k, cfg.k, bv, x, 1e-30, iters)  # warm-up with the same shape (graph captured here)
torch.cuda.synchronize()
x = Vector(ctx, b.size)
t0 = time.perf_counter()
hist, it, st = H.solve(cfg.k, cfg.k, bv, x, 1e-30, iters)
dt = time.perf_counter() - t0
for _ in range(3):
    H.v_cycle(cfg.k, cfg.k, bv, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(iters):
    H.v_cycle(cfg.k, cfg.k, bv, x)
e1.record(stream)
torch.cuda.synchronize()
print(json.dumps(dict(config=cfg.name, iters=it, solve_ms_per_iter=round(dt * 1e3 / it, 4),
                      cycle_ms=round(e0.elapsed_time(e1) / iters, 4), rho_final=float(hist[-1] / hist[0]))))
