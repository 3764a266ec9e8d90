"""Device setup of a BASELINE config under `ncu --profile-from-start off` (the
host-side generation and upload run before the profiled range)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, default_params  # noqa
from paper_2509_06744_b200 import problems as pr  # noqa

cfg = pr.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
if len(sys.argv) > 2:
    cfg = cfg.scaled(int(sys.argv[2]))
ctx = Context(0)
A, T, b = pr.make_problem(cfg)
dA = BlockSparseMatrix(ctx, A)
dT = [BlockSparseMatrix(ctx, p) for p in T]
del A, T
ctx.sync()
torch.cuda.profiler.start()
H = Hierarchy.setup(dA, dT, default_params(t_max=1, nest=cfg.nest, coarse_dim_cap=1 << 30))
ctx.sync()
torch.cuda.profiler.stop()
print("done", H.levels)
