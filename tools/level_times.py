"""Where a V-cycle's time goes, level by level: v_cycle started on level l
(bmg_vcycle_level, graph-replayed) times the sub-cycle of levels <= l; the
difference between consecutive starts is level l's share (its smoothing, residual,
restriction and prolongation), set against its bytes at the in-run read-only peak."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, Vector, default_params  # noqa
from paper_2509_06744_b200 import problems as pr  # noqa

cfg = pr.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
if len(sys.argv) > 2:  # reduced grid (C3 / C5 do not fit one GPU at full size)
    cfg = cfg.scaled(int(sys.argv[2]))
ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
A, T, b = pr.make_problem(cfg)
H = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                    default_params(t_max=1, nest=cfg.nest, coarse_dim_cap=1 << 30))
k = cfg.k
out = []
prev = 0.0
for l in range(H.levels):
    nl = H.level(l)[0].info()["dim_r"]
    bv, xv = Vector(ctx, np.ones(nl)), Vector(ctx, nl)
    for _ in range(3):
        H.v_cycle_level(k, k, l, bv, xv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50 if l < H.levels - 1 else 20
    e0.record(stream)
    for _ in range(reps):
        H.v_cycle_level(k, k, l, bv, xv)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out.append(dict(start_level=l, rows=nl, ms=round(ms, 4), level_share_ms=round(ms - prev, 4)))
    prev = ms
for r in out:
    print(json.dumps(r))
