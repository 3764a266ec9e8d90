"""Randomized campaign: the NCCL code path (loopback transport: one thread per rank
on one GPU) for partitioned cycles and the distributed setup, random world sizes,
shapes, agglomeration and batch sizes -- bitwise against the single-device run.
Usage (on a B200): python tools/fuzz_transport.py SEED SECONDS"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2509_06744_b200 import (BlockSparseMatrix, Context, Hierarchy, LoopbackGroup, Vector,  # noqa: E402
                                   default_params)
from paper_2509_06744_b200 import problems as pr  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 120
ctx = Context(0)
t0 = time.time()
cases = fails = 0
while time.time() - t0 < budget:
    dim = int(rng.choice([2, 2, 3]))
    levels = int(rng.integers(2, 4))
    n = 32 if dim == 2 else 16
    m = int(rng.choice([3, 4, 10]))
    nest = int(rng.choice([0, 0, 1])) if dim == 2 else 0
    world = int(rng.integers(2, 5))
    agg = int(rng.integers(1, levels))
    K = int(rng.choice([1, 2, 4]))
    dist = bool(rng.integers(0, 2))
    cfg = pr.Config("t", dim, n, 2, m, levels, "adaptive", 3, nest=nest, seed=int(rng.integers(100)))
    params = default_params(t_max=1, nest=nest, coarse_dim_cap=1 << 30)
    A, T, b = pr.make_problem(cfg)
    gran = pr.level_grid(cfg)[2]
    h = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T], params)
    h.partition(1, gran)
    B = np.stack([np.roll(b, v) for v in range(K)], axis=1)
    X0 = rng.standard_normal(B.shape)
    xr = Vector(ctx, X0.ravel().copy())
    for _ in range(2):
        h.v_cycle_batch(2, 2, K, Vector(ctx, B.ravel().copy()), xr)
    want = xr.download().reshape(-1, K)
    group = LoopbackGroup(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            c = Context(0, loopback=(group, r))
            if dist:
                Ae, Te, _, _ = pr.dist_inputs(cfg, world, r, agg, params)
                hh = Hierarchy.setup_dist(c, BlockSparseMatrix(c, Ae), [BlockSparseMatrix(c, p) for p in Te], gran,
                                          pr.level_grid(cfg)[3], agg, params)
            else:
                hh = Hierarchy.setup(BlockSparseMatrix(c, A), [BlockSparseMatrix(c, p) for p in T], params)
                hh.partition(world, gran, agglomerate=agg, rank=r)
            lo, hi = hh.part_info(levels - 1, r)[:2]
            rows = slice(lo * m, hi * m)
            xv = Vector(c, X0[rows].ravel().copy())
            for _ in range(2):
                hh.v_cycle_batch(2, 2, K, Vector(c, B[rows].ravel().copy()), xv)
            out[r] = (rows, xv.download().reshape(-1, K))
        except Exception as e:  # noqa: BLE001
            errs.append(f"rank {r}: {type(e).__name__}: {e}")

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    cases += 1
    ok = not errs and all(o is not None and np.array_equal(o[1], want[o[0]]) for o in out)
    if not ok:
        fails += 1
        print("FAIL", dict(dim=dim, levels=levels, m=m, nest=nest, world=world, agg=agg, K=K, dist=dist), errs[:2],
              flush=True)
print("cases", cases, "fails", fails)
