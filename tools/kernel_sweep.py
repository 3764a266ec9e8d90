"""Residual-pass bandwidth of the streaming kernel on the fine-level operators of
every BASELINE config family (reduced grids where the full one would not fit):
bytes = nnzb * (8 m^2 + 4) + 24 N per launch, timed with CUDA events."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Vector, residual  # noqa
from paper_2509_06744_b200 import problems as pr  # noqa

cases = [("C1/C2 fine 2-D 13pt m=10", 2, 256, 2, 10), ("C5 fine 2-D 13pt m=15 (1024^2)", 2, 1024, 2, 15),
         ("C3 fine 2-D 25pt m=21 (512^2)", 2, 512, 3, 21), ("C4 fine 3-D 25pt m=20 (48^3)", 3, 48, 2, 20)]
ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
out = []
for name, dim, n, p, m in cases:
    A = pr.stencil_matrix(dim, n, p, m)
    dA = BlockSparseMatrix(ctx, A)
    x = Vector(ctx, pr.normal_vector(A.dim_r, 0, 1))
    b = Vector(ctx, pr.normal_vector(A.dim_r, 0, 2))
    r = Vector(ctx, A.dim_r)
    for _ in range(3):
        residual(dA, b, x, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record(stream)
    for _ in range(reps):
        residual(dA, b, x, r)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nbytes = dA.info()["pass_bytes"] + 24 * A.dim_r
    rec = dict(case=name, nnzb=A.nnzb, bytes=nbytes, ms=ms, gbs=nbytes / ms / 1e6)
    out.append(rec)
    print(json.dumps(rec), flush=True)
    del dA, x, b, r, A
