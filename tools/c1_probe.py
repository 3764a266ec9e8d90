"""C1 (one k = 3 fourth-kind smoother application on the 64^2, m = 10 operator):
eager launches vs the same application replayed from a captured CUDA graph, to
separate host launch overhead from device time."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import (FSAI_STATIC_LOWER, BlockSparseMatrix, Context, Fsai, Vector,  # noqa
                                   cheb_fourth_apply, lanczos_lambda_max)
from paper_2509_06744_b200 import problems as pr  # noqa

c1 = pr.CONFIGS["C1"]
ctx = Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
A = pr.stencil_matrix(c1.dim, c1.n, c1.power, c1.m, c1.seed, c1.reg)
dA = BlockSparseMatrix(ctx, A)
M = Fsai.build(dA, FSAI_STATIC_LOWER)
beta = lanczos_lambda_max(dA, M, 100, 1.01, 42)
b = Vector(ctx, pr.normal_vector(A.dim_r, c1.seed, 0))
x = Vector(ctx, pr.normal_vector(A.dim_r, c1.seed, 3))


def timed(fn, reps=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


eager = timed(lambda: cheb_fourth_apply(dA, M, b, x, beta, c1.k))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for _ in range(10):
        cheb_fourth_apply(dA, M, b, x, beta, c1.k)
graph = timed(lambda: g.replay(), 50) / 10
print(json.dumps(dict(eager_us=round(eager, 2), graph_us=round(graph, 2))))
if len(sys.argv) > 1 and sys.argv[1] == "profile":  # 2 applications under `ncu --profile-from-start off`
    torch.cuda.profiler.start()
    for _ in range(2):
        cheb_fourth_apply(dA, M, b, x, beta, c1.k)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
