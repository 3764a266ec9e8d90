"""Batched V-cycles (bmg_vcycle_batch) on a BASELINE config: RHS-cycles/s and the
effective GB/s of the batch byte model at K = 1, 2, 4, 8 (CUDA events).

usage: python tools/batch_cycles.py [C2|C4|...] [steps]
"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = pr.CONFIGS[name]
ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
t0 = time.perf_counter()
A, T, b = pr.make_problem(cfg)
H = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                    default_params(t_max=1, nest=cfg.nest, coarse_dim_cap=1 << 30))
ctx.sync()
setup = time.perf_counter() - t0
del A, T
k = cfg.k
for K in (1, 2, 4, 8):
    B = np.stack([np.roll(b, 7 * v) for v in range(K)], axis=1).ravel().copy()
    bv, xv = Vector(ctx, B), Vector(ctx, B.size)
    for _ in range(3):
        H.v_cycle_batch(k, k, K, bv, xv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        H.v_cycle_batch(k, k, K, bv, xv)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    by = H.cycle_bytes(k, k, K)
    print(json.dumps(dict(config=name, K=K, ms_per_batch=round(ms, 3), rhs_cycles_s=round(K * 1e3 / ms, 2),
                          batch_gb=round(by / 1e9, 2), gbs=round(by / ms / 1e6, 1), setup_s=round(setup, 1))),
          flush=True)
    del bv, xv
