"""Device twins of the reference's own test cases for this path
(proj/tests/test_multilevel.cpp, test_fsai.cpp, test_chebyshev.cpp), on the
synthetic problems (the same cases on the reference's FD biharmonic problem:
test_gpu_fd_problem.py; the PUM generator is out of scope)."""
import numpy as np
import pytest

from paper_2509_06744_b200 import (FSAI_ADAPTIVE, BlockSparseMatrix, Fsai, Hierarchy, Vector, apply_smoother,
                                   cheb_fourth_apply, default_params, lanczos_lambda_max, spmv)
from paper_2509_06744_b200 import problems as pr
from paper_2509_06744_b200.api import HostBsr
from paper_2509_06744_b200.native import FSAI_DIAGONAL, InvalidArgument
from tests.helpers import random_layout, random_spd

pytestmark = pytest.mark.gpu


def _hier(ctx, n, levels, t_max):
    cfg = pr.CONFIGS["C2"].scaled(n, levels)
    A, T, _ = pr.make_problem(cfg)
    dA = BlockSparseMatrix(ctx, A)
    h = Hierarchy.setup(dA, [BlockSparseMatrix(ctx, p) for p in T],
                        default_params(t_max=t_max, coarse_dim_cap=1 << 30))
    return h, dA, A


def _Av(ctx, dA, v):
    y = Vector(ctx, v.size)
    spmv(dA, Vector(ctx, v), y)
    return y.download()


def _cycle_err(ctx, h, e, k):
    ev = Vector(ctx, e.copy())
    h.v_cycle(k, k, Vector(ctx, np.zeros_like(e)), ev)
    return ev.download()


def test_symmetric_cycle_operator_is_A_self_adjoint(ctx, rng):
    # test_multilevel.cpp:151-171
    h, dA, A = _hier(ctx, 16, 2, 2)
    e1, e2 = rng.uniform(-1, 1, A.dim_r), rng.uniform(-1, 1, A.dim_r)
    ce1, ce2 = _cycle_err(ctx, h, e1, 3), _cycle_err(ctx, h, e2, 3)
    lhs = _Av(ctx, dA, ce1) @ e2
    rhs = _Av(ctx, dA, ce2) @ e1
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), 1.0)


def test_vcycle_error_contraction(ctx, rng):
    # test_multilevel.cpp:129-149 (energy-norm contraction of V(4,4), t_max = 4)
    h, dA, A = _hier(ctx, 32, 3, 4)
    e = rng.uniform(-1, 1, A.dim_r)
    prev = np.sqrt(e @ _Av(ctx, dA, e))
    rho_max = 0.0
    for _ in range(6):
        e = _cycle_err(ctx, h, e, 4)
        cur = np.sqrt(max(e @ _Av(ctx, dA, e), 0.0))
        rho_max = max(rho_max, cur / prev)
        prev = cur
    assert rho_max < 1.0


def test_setup_is_deterministic_and_levels_spd(ctx):
    # test_multilevel.cpp:173-189: two setups give identical levels and bounds
    h1, _, A = _hier(ctx, 16, 3, 3)
    h2, _, _ = _hier(ctx, 16, 3, 3)
    for l in range(h1.levels):
        if l:
            assert h1.beta(l) == h2.beta(l)
        a1, _, _ = h1.level(l)
        a2, _, _ = h2.level(l)
        info = a1.info()
        d1 = a1.download(np.full(info["nbr"], 10, np.int32), np.full(info["nbc"], 10, np.int32))
        d2 = a2.download(np.full(info["nbr"], 10, np.int32), np.full(info["nbc"], 10, np.int32))
        assert np.array_equal(d1.vals, d2.vals) and np.array_equal(d1.col_idx, d2.col_idx)
        if l == 0:  # the coarse operator is SPD (its Cholesky succeeded) -- check it directly
            assert np.linalg.eigvalsh(d1.to_dense()).min() > 0


def test_identity_transfer_chain_shares_the_spectral_bound(ctx, rng):
    # test_multilevel.cpp:191-202: P = I, so A_0 = A and both levels share beta
    sizes = random_layout(rng, 6, 3)
    a = random_spd(rng, sizes, 0.8)
    n = len(sizes)
    eye = HostBsr(sizes, sizes, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
                  np.concatenate([np.eye(int(m)).ravel() for m in sizes]), False)
    params = default_params(t_max=2, coarse_dim_cap=1 << 30)
    h = Hierarchy.setup(BlockSparseMatrix(ctx, a), [BlockSparseMatrix(ctx, eye)], params)
    a0, _, _ = h.level(0)
    M0 = Fsai.build(a0, FSAI_ADAPTIVE, t_max=2)
    beta_coarse = lanczos_lambda_max(a0, M0, 100, 1.01, 42)
    assert h.beta(1) == pytest.approx(beta_coarse, rel=0.011)


def test_fourth_kind_application_is_linear(ctx, rng):
    # test_chebyshev.cpp:200-217 on a block operator with its FSAI preconditioner
    host = pr.stencil_matrix(2, 12, 2, 10)
    A = BlockSparseMatrix(ctx, host)
    M = Fsai.build(A, FSAI_ADAPTIVE, t_max=1)
    beta = lanczos_lambda_max(A, M, 100, 1.01, 42)
    n = host.dim_r
    b1, b2, x1, x2 = (rng.uniform(-1, 1, n) for _ in range(4))
    c1, c2 = 0.7, -1.3

    def cheb(b, x, k):
        xv = Vector(ctx, x.copy())
        cheb_fourth_apply(A, M, Vector(ctx, b.copy()), xv, beta, k)
        return xv.download()

    for k in range(1, 6):
        lhs = cheb(c1 * b1 + c2 * b2, c1 * x1 + c2 * x2, k)
        rhs = c1 * cheb(b1, x1, k) + c2 * cheb(b2, x2, k)
        assert np.linalg.norm(lhs - rhs) <= 1e-12 * (1.0 + np.linalg.norm(rhs))


def test_full_lower_pattern_is_an_exact_inverse(ctx, rng):
    # test_fsai.cpp:79-92
    for _ in range(5):
        sizes = random_layout(rng, 10, 3)
        a = random_spd(rng, sizes, 1.0)
        n = len(sizes)
        M = Fsai.from_pattern(BlockSparseMatrix(ctx, a), [list(range(i + 1)) for i in range(n)])
        r = rng.uniform(-1, 1, a.dim_r)
        z = Vector(ctx, a.dim_r)
        M.apply(Vector(ctx, r), z)
        want = np.linalg.solve(a.to_dense(), r)
        assert np.linalg.norm(z.download() - want) <= 1e-9 * np.linalg.norm(want)


def test_diagonal_pattern_reduces_to_block_jacobi(ctx, rng):
    # test_fsai.cpp:57-69: M = blockdiag(A)^-1
    sizes = np.array([2, 3, 1, 2], np.int32)
    a = random_spd(rng, sizes, 0.7)
    M = Fsai.build(BlockSparseMatrix(ctx, a), FSAI_DIAGONAL)
    r = rng.uniform(-1, 1, a.dim_r)
    z = Vector(ctx, a.dim_r)
    M.apply(Vector(ctx, r), z)
    d = a.to_dense()
    off = np.concatenate([[0], np.cumsum(sizes)])
    want = np.concatenate([np.linalg.solve(d[off[i]:off[i + 1], off[i]:off[i + 1]], r[off[i]:off[i + 1]])
                           for i in range(len(sizes))])
    assert np.linalg.norm(z.download() - want) <= 1e-13 * np.linalg.norm(want)


def test_smoother_parameter_validation(ctx):
    # test_chebyshev.cpp:219-229: beta <= 0, alpha outside (0, beta), degree 0
    host = pr.stencil_matrix(2, 4, 2, 10)
    A = BlockSparseMatrix(ctx, host)
    M = Fsai.build(A, FSAI_DIAGONAL)
    b, x = Vector(ctx, host.dim_r), Vector(ctx, host.dim_r)
    with pytest.raises(InvalidArgument):
        cheb_fourth_apply(A, M, b, x, -1.0, 2)
    with pytest.raises(InvalidArgument):
        apply_smoother(A, M, 1, b, x, 2, alpha=0.0, beta=1.0)
    with pytest.raises(InvalidArgument):
        apply_smoother(A, M, 1, b, x, 2, alpha=1.5, beta=1.0)
    with pytest.raises(InvalidArgument):
        apply_smoother(A, M, 0, b, x, 0, omega=1.0)
