"""The BASELINE configurations' shapes against the oracle, setup through the
stop-on-tolerance solve (VERDICT r01 "parity on the
untested BASELINE shapes").

Each case keeps its config's block size, stencil, FSAI kind / nesting, smoother
degree and depth at a reduced grid (tests/golden/make_solve_golden.py):

  * C4 shape: 3-D 25-point, m = 20, adaptive block-FSAI, V(3,3), 4 levels;
  * C5 shape: 2-D 13-point, m = 15, adaptive, V(3,3), 6 levels;
  * C3 shape: 2-D 25-point triharmonic, m = 21, nested FSAI (nest = 1), V(4,4), 5 levels.

Against the oracle fixtures (the reference's `setup` + `measure_rates` loop,
multilevel.cpp:36-75, experiments.cpp:46-58, restated in oracle/):

  * Galerkin operators A_l (galerkin_coarsen, multilevel.cpp:11-28): bitwise;
  * FSAI factors F_0..F_{nest-1} and G = L^-1 F_nest (fsai.cpp:106-253): bitwise;
  * beta_l (lanczos.hpp:16-58): 1e-10 relative;
  * residual history rho_n = ||r_n|| / ||r_0|| of the solve to 1e-8:
    |rho_gpu - rho_cpu| <= 1e-10 for every n, and relative 1e-10 while rho >= 1e-2
    (SURVEY.md App. C);
  * identical iteration counts and status -- unless the oracle's stopping rho lies
    within the measured history discrepancy of the tolerance,
    which the test reports instead of hiding.
"""
import os

import numpy as np
import pytest

from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy, Vector, default_params
from paper_2509_06744_b200 import problems as pr
from tests.golden.make_solve_golden import bsr_digest, case_config, load, path_for

pytestmark = pytest.mark.gpu

FAST = ["C4@16x4", "C5@128x6", "C3@128x5"]
LARGE = ["C5@256x6", "C4@32x4"]


def device_setup(ctx, cfg):
    A, T, b = pr.make_problem(cfg)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, tau=1.0, nest=cfg.nest, coarse_dim_cap=1 << 30,
                                        fsai_kind=0 if cfg.fsai == "static" else 3))
    return dh, b


def check_setup(dh, cfg, fx):
    assert dh.levels == fx["levels"] == cfg.levels
    for l in range(dh.levels):
        ent = fx["level"][l]
        A, _, M = dh.level(l)
        nb = A.info()["nbr"]
        sizes = np.full(nb, cfg.m, np.int32)
        assert bsr_digest(A.download(sizes, sizes, symmetric=True)) == ent["A"], f"A_{l} differs"
        if l == 0:
            continue
        assert M.chain_len == len(ent["factors"]) + 1
        for k, dg in enumerate(ent["factors"]):
            assert bsr_digest(M.factor(k).download(sizes, sizes)) == dg, f"F_{k} of level {l} differs"
        assert bsr_digest(M.G.download(sizes, sizes)) == ent["G"], f"G of level {l} differs"
        bo = float.fromhex(ent["beta"])
        assert abs(dh.beta(l) - bo) <= 1e-10 * bo, (l, dh.beta(l), bo)


def check_history(hist_g, it_g, st_g, fx):
    hist_o = fx["history_f"]
    it_o, st_o, tol = fx["iterations"], fx["status"], fx["tol"]
    rho_o, rho_g = hist_o / hist_o[0], hist_g / hist_g[0]
    n = min(rho_o.size, rho_g.size)
    d = np.abs(rho_g[:n] - rho_o[:n])
    assert np.all(d <= 1e-10), f"max |drho| {d.max():.3e} at n = {int(d.argmax())}"
    big = rho_o[:n] >= 1e-2
    rel = np.abs(rho_g[:n][big] / rho_o[:n][big] - 1)
    assert np.all(rel <= 1e-10), f"max relative drho {rel.max():.3e}"
    if it_g != it_o:
        # allowed only when the oracle's crossing of the tolerance is closer to
        # tol than the histories' measured disagreement
        margin = min(abs(rho_o[it_o] - tol), abs(rho_o[it_o - 1] - tol))
        assert abs(it_g - it_o) == 1 and margin <= d.max(), (it_g, it_o, margin, d.max())
        pytest.xfail(f"iteration count {it_g} vs {it_o}: the oracle's stopping rho is within "
                     f"{margin:.2e} of tol, below the measured discrepancy {d.max():.2e}")
    assert st_g == st_o
    return d.max()


def run_case(ctx, case):
    if not os.path.exists(path_for(case)):
        pytest.skip(f"fixture {path_for(case)} not generated")
    fx = load(case)
    cfg, max_iter = case_config(case)
    dh, b = device_setup(ctx, cfg)
    check_setup(dh, cfg, fx)
    bv, xv = Vector(ctx, b), Vector(ctx, np.zeros_like(b))
    hist_g, it_g, st_g = dh.solve(cfg.k, cfg.k, bv, xv, cfg.tol, fx["max_iter"])
    dmax = check_history(hist_g, it_g, st_g, fx)
    xn = np.linalg.norm(xv.download())
    xo = float.fromhex(fx["x_norm"])
    assert abs(xn - xo) <= 1e-8 * xo, (xn, xo)
    return it_g, dmax


@pytest.mark.parametrize("case", FAST)
def test_shape_setup_and_solve_to_1e8(ctx, case):
    run_case(ctx, case)


@pytest.mark.parametrize("case", LARGE)
def test_large_shape_setup_and_solve_to_1e8(ctx, case):
    run_case(ctx, case)
