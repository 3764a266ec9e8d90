"""Committed golden fixtures (tests/golden/, written by tests/golden/make_golden.py).

CPU: the oracle still reproduces its committed outputs bitwise and the
reference's asserted known answers.  GPU: the product matches the committed
numbers (bitwise for the streaming SpMV, 1e-12 / 1e-10 elsewhere, as in
tests/test_gpu_solver.py)."""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import problems as pr

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLD = json.load(open(os.path.join(HERE, "oracle_small.json")))
KA = json.load(open(os.path.join(HERE, "known_answers.json")))


def test_known_answers_against_oracle():
    l, _ = O.cholesky(np.array(KA["cholesky_4_2_5"]["b"], float))
    assert np.allclose(l, KA["cholesky_4_2_5"]["l"], rtol=0, atol=1e-15)
    with pytest.raises(O.OracleError) as e:
        O.cholesky(np.array(KA["cholesky_indefinite_pivot"]["b"], float))
    assert e.value.pivot == KA["cholesky_indefinite_pivot"]["pivot"]
    assert O.poly_eval(O.SCALED_FOURTH, 1, 1.0, beta=1.0) == pytest.approx(KA["cheb4_degree1_factor"]["value"])
    for k, v in zip(KA["fourth_kind_W_at_one"]["k"], KA["fourth_kind_W_at_one"]["value"]):
        assert O.poly_eval(O.FOURTH_W, k, 1.0) == pytest.approx(v, rel=1e-14)
    lam = O.lanczos_diag(np.arange(1.0, 51.0), 100, 1.0, 42)
    assert KA["lanczos_diag_1_50"]["lo"] <= lam <= KA["lanczos_diag_1_50"]["hi"] + 1e-10


def test_oracle_reproduces_committed_fixtures():
    g = GOLD["c1_16"]
    A = pr.stencil_matrix(2, g["grid"], 2, g["m"])
    om = O.Mat(A)
    of = O.Fsai(om, O.Fsai.STATIC)
    beta = O.lanczos_lambda_max(om, of, 100, 1.01, 42)
    assert beta == g["beta"]
    x0 = pr.normal_vector(A.dim_r, 0, 3)
    y = om.spmv(x0)
    assert np.array_equal(y[:64], np.array(g["spmv_x0_head"]))
    x = O.smoother_apply(om, of, O.CHEB_FOURTH, pr.normal_vector(A.dim_r, 0, 0), x0, 3, beta=beta)
    assert np.array_equal(x[:64], np.array(g["cheb4_k3_head"]))


@pytest.mark.gpu
def test_product_matches_committed_fixtures(ctx):
    from paper_2509_06744_b200 import (FSAI_STATIC_LOWER, BlockSparseMatrix, Fsai, Hierarchy, Vector,
                                       cheb_fourth_apply, default_params, lanczos_lambda_max, spmv)

    g = GOLD["c1_16"]
    A = pr.stencil_matrix(2, g["grid"], 2, g["m"])
    dA = BlockSparseMatrix(ctx, A)
    x0 = pr.normal_vector(A.dim_r, 0, 3)
    y = Vector(ctx, A.dim_r)
    spmv(dA, Vector(ctx, x0), y)
    assert np.array_equal(y.download()[:64], np.array(g["spmv_x0_head"]))
    M = Fsai.build(dA, FSAI_STATIC_LOWER)
    beta = lanczos_lambda_max(dA, M, 100, 1.01, 42)
    assert abs(beta - g["beta"]) <= 1e-10 * g["beta"]
    xv = Vector(ctx, x0)
    cheb_fourth_apply(dA, M, Vector(ctx, pr.normal_vector(A.dim_r, 0, 0)), xv, g["beta"], 3)
    x = xv.download()
    assert np.linalg.norm(x[:64] - np.array(g["cheb4_k3_head"])) <= 1e-12 * np.linalg.norm(g["cheb4_k3_head"])
    assert abs(np.linalg.norm(x) - g["cheb4_k3_norm"]) <= 1e-12 * g["cheb4_k3_norm"]
    c = GOLD["c2_32_3lev"]
    cfg = pr.CONFIGS["C2"].scaled(c["grid"], c["levels"])
    A, T, b = pr.make_problem(cfg)
    H = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                        default_params(t_max=1, coarse_dim_cap=1 << 30))
    for l, bt in enumerate(c["betas"], start=1):
        assert abs(H.beta(l) - bt) <= 1e-10 * bt
    hist, it, st = H.solve(3, 3, Vector(ctx, b), Vector(ctx, b.size), 1e-8, len(c["rho"]) - 1)
    rho = hist / hist[0]
    assert len(rho) == len(c["rho"])
    assert np.all(np.abs(rho - np.array(c["rho"])) <= 1e-10)
