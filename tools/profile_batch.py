"""Batched streaming pass under ncu (`ncu --profile-from-start off`), and its
CUDA-event timing without ncu.

usage: python tools/profile_batch.py K [dim n p m] [reps]
Profiles 3 launches of y = A x on K right-hand sides (interleaved per scalar
row) for one fine-level stencil operator (default: C2's, 256^2, 13-point, m=10);
prints the CUDA-event GB/s (matrix once + K vectors) of 20 launches first.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Vector, spmv_batch  # noqa
from paper_2509_06744_b200 import problems as pr  # noqa

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dim, n, p, m = (int(v) for v in sys.argv[2:6]) if len(sys.argv) > 5 else (2, 256, 2, 10)
ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
A = pr.stencil_matrix(dim, n, p, m)
dA = BlockSparseMatrix(ctx, A)
x = Vector(ctx, pr.normal_vector(A.dim_r * K, 0, 1))
y = Vector(ctx, A.dim_r * K)
for _ in range(3):
    spmv_batch(dA, K, x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record(stream)
for _ in range(reps):
    spmv_batch(dA, K, x, y)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
nbytes = dA.info()["pass_bytes"] + 16 * K * A.dim_r
print(json.dumps(dict(dim=dim, n=n, m=m, K=K, us=round(ms * 1e3, 1), gbs=round(nbytes / ms / 1e6, 1))))
torch.cuda.profiler.start()
for _ in range(3):
    spmv_batch(dA, K, x, y)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
