"""Randomized campaign: device setup + V-cycle vs the oracle on small 2-D / 3-D
hierarchies (m, levels, nest, t_max, smoother kind, variable layouts, asymmetric
cycles) and batched cycles bitwise vs single ones.  Usage: python tools/fuzz_hierarchy.py SEED SECONDS"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as O
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, Vector, default_params
from paper_2509_06744_b200 import problems as pr
ctx = Context(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
t0 = time.time(); cases = 0; fails = 0
while time.time() - t0 < float(sys.argv[2] if len(sys.argv) > 2 else 120):
    dim = int(rng.choice([2, 2, 3]))
    levels = int(rng.integers(2, 4))
    n = int(rng.choice([8, 16])) if dim == 2 else 8
    # the BASELINE block sizes (C2 10, C5 15, C4 20, C3 21) and small ones
    m = int(rng.choice([3, 4, 6, 10, 15, 20, 21]))
    power = int(rng.choice([1, 2])) if dim == 3 else int(rng.choice([2, 3]))
    nest = int(rng.choice([0, 0, 1]))
    t_max = int(rng.choice([1, 2]))
    kind = int(rng.choice([0, 1, 2]))
    var = bool(rng.integers(0, 2)) and m == 10 and dim == 2
    cfg = pr.Config("f", dim, n, power, m, levels, "adaptive", 3, nest=nest, seed=int(rng.integers(100)))
    try:
        A, T, b = pr.make_variable_problem(cfg, 6) if var else pr.make_problem(cfg)
    except Exception as e:
        continue
    kpre, kpost = int(rng.integers(0, 4)), int(rng.integers(0, 4))
    if kpre + kpost == 0:
        kpost = 1
    try:
        oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=t_max, nest=nest, coarse_dim_cap=1 << 30, probe=False,
                         smoother_kind=kind)
        dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                             default_params(t_max=t_max, nest=nest, coarse_dim_cap=1 << 30, smoother_kind=kind))
    except Exception as e:
        print("SETUP-ERR", dim, n, m, levels, nest, t_max, kind, var, type(e).__name__, str(e)[:80], flush=True)
        fails += 1
        continue
    x0 = rng.standard_normal(b.size)
    xo = oh.v_cycle(kpre, kpost, b, x0.copy())
    xv = Vector(ctx, x0.copy())
    dh.v_cycle(kpre, kpost, Vector(ctx, b), xv)
    err = np.linalg.norm(xv.download() - xo) / max(np.linalg.norm(xo), 1e-300)
    ok = err <= 1e-9
    ok_tol = ok
    K = int(rng.choice([2, 4, 8]))
    B = np.stack([b * (v + 1) for v in range(K)], axis=1).ravel().copy()
    X0 = np.stack([x0] * K, axis=1).ravel().copy()
    xb = Vector(ctx, X0)
    dh.v_cycle_batch(kpre, kpost, K, Vector(ctx, B), xb)
    Xb = xb.download().reshape(-1, K)
    for v in range(K):
        xs = Vector(ctx, x0.copy())
        dh.v_cycle(kpre, kpost, Vector(ctx, b * (v + 1)), xs)
        ok &= np.array_equal(Xb[:, v], xs.download())
    cases += 1
    if not ok:
        fails += 1
        # tolerance vs the oracle (3-D 7-point operators, power 1, are
        # Lanczos-sensitive) or the batched-cycle bitwise identity (a kernel bug if it fails)
        what = "tol" if not ok_tol and ok == ok_tol else ("batch" if ok_tol else "tol+batch")
        print("FAIL", what, "dim", dim, "p", power, "n", n, "m", m, "L", levels, "nest", nest, "t", t_max, "kind", kind,
              "var", var, "k", kpre, kpost, "K", K, "err", f"{err:.2e}", flush=True)
print("cases", cases, "fails", fails)
