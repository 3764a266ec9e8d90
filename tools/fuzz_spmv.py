"""Randomized campaign: uniform-layout SpMV (K = 1 and batched) bitwise vs the oracle.
Usage (on a B200): python tools/fuzz_spmv.py SEED SECONDS"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as O
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Vector, spmv, spmv_batch, residual
from paper_2509_06744_b200.api import HostBsr
from tests.helpers import random_bsr
ctx = Context(0)
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
t0 = time.time(); cases = 0; fails = 0
while time.time() - t0 < float(sys.argv[2] if len(sys.argv) > 2 else 120):
    m = int(rng.choice([10, 15, 20, 21, 3, 6, 7]))
    nbr = int(rng.integers(1, 400)); nbc = int(rng.integers(1, 400))
    dens = float(rng.choice([0.002, 0.02, 0.1, 0.5]))
    h = random_bsr(rng, np.full(nbr, m, np.int32), np.full(nbc, m, np.int32), dens)
    # a few very long rows and empty rows
    A = BlockSparseMatrix(ctx, h)
    x = rng.standard_normal(h.dim_c)
    want = O.Mat(h).spmv(x)
    y = Vector(ctx, h.dim_r)
    spmv(A, Vector(ctx, x), y)
    ok = np.array_equal(y.download(), want)
    K = int(rng.choice([2, 4, 8]))
    X = rng.standard_normal((h.dim_c, K))
    Y = Vector(ctx, h.dim_r * K)
    spmv_batch(A, K, Vector(ctx, X.ravel().copy()), Y)
    Yg = Y.download().reshape(-1, K)
    for v in range(K):
        ok &= np.array_equal(Yg[:, v], O.Mat(h).spmv(X[:, v].copy()))
    cases += 1
    if not ok:
        fails += 1
        print("FAIL", m, nbr, nbc, dens, K, flush=True)
print("cases", cases, "fails", fails)
