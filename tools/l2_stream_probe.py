"""Residual pass r = b - A x on 2-D 13-point m = 10 operators of growing size, 50
back-to-back launches: where the matrix fits the 126 MB L2 the stream is served from
L2, so the rate shows whether the SM side (TMA ingress) or HBM bounds the pass."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Vector, residual  # noqa
from paper_2509_06744_b200 import problems as pr  # noqa

ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
for n in (64, 80, 96, 112, 128, 192, 256):
    A = pr.stencil_matrix(2, n, 2, 10)
    dA = BlockSparseMatrix(ctx, A)
    x = Vector(ctx, pr.normal_vector(A.dim_r, 0, 1))
    b = Vector(ctx, pr.normal_vector(A.dim_r, 0, 2))
    r = Vector(ctx, A.dim_r)
    for _ in range(5):
        residual(dA, b, x, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record(stream)
    for _ in range(reps):
        residual(dA, b, x, r)
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    nbytes = dA.info()["pass_bytes"] + 24 * A.dim_r
    print(json.dumps(dict(n=n, mb=round(nbytes / 1e6, 1), us=round(us, 2), gbs=round(nbytes / us / 1e3, 1))), flush=True)
    del dA, x, b, r, A
