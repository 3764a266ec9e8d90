"""The FD biharmonic test problem (experiments.cpp:104-195) pinned by an
independent Kronecker formulation, and the oracle run through the reference's
own multilevel test cases on it (test_multilevel.cpp:99-186) -- CPU only."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import problems as pr


@pytest.mark.parametrize("ng", [4, 8, 16])
def test_fd_matrix_is_kronecker_bilaplacian(ng):
    # Delta_h^2 with clamped ends: (T^2 + D) (x) I + 2 T (x) T + I (x) (T^2 + D),
    # T = tridiag(-1, 2, -1), D = diag(2, 0, ..., 0, 2), times 1/h^4
    m = ng - 1
    T = 2 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)
    D = np.zeros((m, m))
    D[0, 0] += 2
    D[-1, -1] += 2
    I = np.eye(m)
    want = (np.kron(I, T @ T + D) + 2 * np.kron(T, T) + np.kron(T @ T + D, I)) * float(ng) ** 4
    A = pr.fd_biharmonic_matrix(ng)
    assert np.array_equal(A.to_dense(), want)
    assert all(np.all(np.diff(A.col_idx[A.row_ptr[r]:A.row_ptr[r + 1]]) > 0) for r in range(A.nbr))


@pytest.mark.parametrize("ng", [8, 16, 32])
def test_fd_prolongation_is_tensor_linear_interpolation(ng):
    mf, mc = ng - 1, ng // 2 - 1
    P1 = np.zeros((mf, mc))
    for c in range(mc):  # coarse node c sits at fine node 2c + 1
        P1[2 * c + 1, c] = 1.0
        P1[2 * c, c] = 0.5
        P1[2 * c + 2, c] = 0.5
    assert np.array_equal(pr.fd_prolongation(ng).to_dense(), np.kron(P1, P1))


def test_fd_problem_shapes_and_errors():
    fd = pr.fd_biharmonic(32, 3)
    assert [(p.dim_r, p.dim_c) for p in fd.transfers] == [(15 ** 2, 7 ** 2), (31 ** 2, 15 ** 2)]
    assert np.allclose(fd.mass.to_dense(), np.eye(31 ** 2) / 32 ** 2)
    assert np.linalg.norm(fd.b - fd.A.to_dense() @ fd.reference) <= 1e-14 * np.linalg.norm(fd.b)
    for bad in ((12, 2), (16, 0), (16, 4)):
        with pytest.raises(ValueError):
            pr.fd_biharmonic(*bad)


def _ohier(ng, levels, t_max):
    fd = pr.fd_biharmonic(ng, levels)
    return fd, O.Hierarchy(O.Mat(fd.A), [O.Mat(p) for p in fd.transfers], t_max=t_max, probe=False)


def test_oracle_one_level_fd_solves_directly():
    # test_multilevel.cpp:99-106
    fd, oh = _ohier(8, 1, 1)
    x = oh.v_cycle(2, 2, fd.b, np.zeros_like(fd.b))
    assert np.linalg.norm(x - fd.reference) <= 1e-9 * np.linalg.norm(fd.reference)


def test_oracle_fd_contraction_and_self_adjointness():
    # test_multilevel.cpp:129-171
    rng = np.random.default_rng(213)
    fd, oh = _ohier(32, 3, 4)
    A = fd.A.to_dense()
    n = A.shape[0]
    e = rng.standard_normal(n)
    prev, rho_max = np.sqrt(e @ A @ e), 0.0
    for _ in range(6):
        e = oh.v_cycle(4, 4, np.zeros(n), e)
        cur = np.sqrt(max(e @ A @ e, 0.0))
        rho_max, prev = max(rho_max, cur / prev), cur
    assert rho_max < 1.0
    fd, oh = _ohier(16, 2, 2)
    A = fd.A.to_dense()
    n = A.shape[0]
    e1, e2 = rng.standard_normal(n), rng.standard_normal(n)
    ce1, ce2 = (oh.v_cycle(3, 3, np.zeros(n), e.copy()) for e in (e1, e2))
    lhs, rhs = (A @ ce1) @ e2, (A @ ce2) @ e1
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), 1.0)
