"""Profiling driver for ncu (run under `ncu --profile-from-start off`).

mode=cycle:    setup C2, then profile 2 V-cycles (launch list / shares)
mode=residual: profile 3 launches of the finest-level residual pass
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import Context, Hierarchy, BlockSparseMatrix, Vector, default_params, residual  # noqa
from paper_2509_06744_b200 import problems as pr  # noqa

mode = sys.argv[1] if len(sys.argv) > 1 else "cycle"
cfg = pr.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C2"]
if len(sys.argv) > 3:
    cfg = cfg.scaled(int(sys.argv[3]))
ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
A, T, b = pr.make_problem(cfg)
dA = BlockSparseMatrix(ctx, A)
dT = [BlockSparseMatrix(ctx, p) for p in T]
H = Hierarchy.setup(dA, dT, default_params(t_max=1, coarse_dim_cap=1 << 30))
bv, xv = Vector(ctx, b), Vector(ctx, A.dim_r)
for _ in range(3):
    H.v_cycle(cfg.k, cfg.k, bv, xv)
torch.cuda.synchronize()
if mode == "cycle":
    torch.cuda.profiler.start()
    for _ in range(1 if cfg.dim == 3 else 2):
        H.v_cycle(cfg.k, cfg.k, bv, xv)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
elif mode in ("gpass", "gtpass"):
    from paper_2509_06744_b200 import spmv
    Af, _, Mf = H.level(H.levels - 1)
    G = Mf.G if mode == "gpass" else Mf.G.transpose()
    rv = Vector(ctx, A.dim_r)
    spmv(G, bv, rv)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(3):
        spmv(G, bv, rv)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
elif mode.startswith("residual@"):  # residual pass of level l (residual@2)
    lvl = int(mode.split("@")[1])
    Al, _, _ = H.level(lvl)
    nl = Al.info()["dim_r"]
    xl, bl, rl = Vector(ctx, np.ones(nl)), Vector(ctx, np.ones(nl)), Vector(ctx, nl)
    residual(Al, bl, xl, rl)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(3):
        residual(Al, bl, xl, rl)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
else:
    rv = Vector(ctx, A.dim_r)
    Af, _, _ = H.level(H.levels - 1)
    residual(Af, bv, xv, rv)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(3):
        residual(Af, bv, xv, rv)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("done")
