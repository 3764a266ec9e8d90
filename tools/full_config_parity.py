"""One-off parity check at a WHOLE BASELINE config (default C4, the headline): the
oracle's setup + N V-cycles (residual history from x = 0) on all host threads,
then the device's, compared: beta per level (relative), |rho_gpu - rho_cpu| per
cycle and relative while rho >= 1e-2 (the north_star criterion, here over the
first N cycles of the full-size problem instead of a scaled fixture).
Usage: python tools/full_config_parity.py C4 [cycles]   (C4 needs ~130 GB host RAM)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import pyoracle as O  # noqa: E402
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, Vector, default_params  # noqa: E402
from paper_2509_06744_b200 import problems as pr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = pr.CONFIGS[name.split("@")[0]]
if "@" in name:  # the same shape on an N-per-side grid (e.g. C5@1024: a quarter of C5's rows)
    cfg = cfg.scaled(int(name.split("@")[1]))
O.set_threads(os.cpu_count() or 1)
A, T, b = pr.make_problem(cfg)
oA, oT = O.Mat(A), [O.Mat(p) for p in T]
del A, T
t0 = time.perf_counter()
oh = O.Hierarchy(oA, oT, t_max=1, tau=1.0, nest=cfg.nest, coarse_dim_cap=1 << 30, probe=False, consume=True)
o_setup = time.perf_counter() - t0
del oA, oT
beta_o = [oh.beta(l) for l in range(1, oh.levels())]
t0 = time.perf_counter()
hist_o, it_o, st_o, x_o = oh.solve(cfg.k, cfg.k, b, np.zeros_like(b), 1e-30, cycles)
o_solve = time.perf_counter() - t0
xn_o = float(np.linalg.norm(x_o))
del oh

ctx = Context(0)
A, T, b2 = pr.make_problem(cfg)
assert np.array_equal(b, b2)
dA, dT = BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T]
del A, T
t0 = time.perf_counter()
dh = Hierarchy.setup(dA, dT, default_params(t_max=1, tau=1.0, nest=cfg.nest, coarse_dim_cap=1 << 30))
ctx.sync()
d_setup = time.perf_counter() - t0
beta_g = [dh.beta(l) for l in range(1, dh.levels)]
xv = Vector(ctx, b.size)
hist_g, it_g, st_g = dh.solve(cfg.k, cfg.k, Vector(ctx, b), xv, 1e-30, cycles)
x_g = xv.download()
rho_o, rho_g = hist_o / hist_o[0], np.asarray(hist_g) / hist_g[0]
big = rho_o >= 1e-2
print(json.dumps({
    "config": name, "cycles": cycles, "unknowns": int(b.size), "levels": len(beta_o) + 1,
    "beta_rel_diff": [abs(g - o) / o for g, o in zip(beta_g, beta_o)],
    "rho_cpu": [float(v) for v in rho_o], "rho_gpu": [float(v) for v in rho_g],
    "max_abs_drho": float(np.max(np.abs(rho_g - rho_o))),
    "max_rel_drho_while_rho_ge_1e-2": float(np.max(np.abs(rho_g[big] - rho_o[big]) / rho_o[big])),
    "r0_equal": bool(hist_g[0] == hist_o[0]),
    "x_rel_diff": float(np.linalg.norm(x_g - x_o) / xn_o),
    "oracle_setup_s": round(o_setup, 1), "oracle_solve_s": round(o_solve, 1), "device_setup_s": round(d_setup, 1),
    "oracle_threads": O.get_threads()}), flush=True)
