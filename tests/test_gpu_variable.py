"""Variable block layouts through the whole hierarchy (the reference's general
BlockLayout, block_layout.hpp:8-28; the paper's PUM systems mix block sizes):
Galerkin and triple products bitwise, full device setup + solve against the
oracle with the BASELINE tolerances."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import (FSAI_ADAPTIVE, FSAI_STATIC_LOWER, BlockSparseMatrix, Fsai, Hierarchy, Vector,
                                   default_params, galerkin_coarsen)
from paper_2509_06744_b200 import problems as pr

pytestmark = pytest.mark.gpu


def _same(got, want):
    assert np.array_equal(got.row_ptr, want.row_ptr)
    assert np.array_equal(got.col_idx, want.col_idx)
    assert np.array_equal(got.vals, want.vals)


def _problem(n=16, levels=3, m=10, m_bnd=6, power=2):
    cfg = pr.Config("var", 2, n, power, m, levels, "adaptive", 3)
    return pr.make_variable_problem(cfg, m_bnd)


def test_variable_layout_is_spd_and_mixed():
    A, T, b = _problem(8, 2)
    assert set(np.unique(A.row_sizes)) == {6, 10}
    d = A.to_dense()
    assert np.array_equal(d, d.T)
    assert np.linalg.eigvalsh(d).min() > 0


def test_galerkin_variable_bitwise(ctx):
    A, T, _ = _problem(16, 2)
    got = galerkin_coarsen(BlockSparseMatrix(ctx, A), BlockSparseMatrix(ctx, T[0])).download(
        T[0].col_sizes, T[0].col_sizes)
    _same(got, O.galerkin(O.Mat(A), O.Mat(T[0])).export())


def test_triple_product_variable_bitwise(ctx):
    from paper_2509_06744_b200 import triple_product
    A, _, _ = _problem(10, 2)
    F = O.Fsai(O.Mat(A), O.Fsai.STATIC).factor(0).export()
    want = O.triple_product(O.Mat(F), O.Mat(A)).export(symmetric=True)
    got = triple_product(BlockSparseMatrix(ctx, F), BlockSparseMatrix(ctx, A)).download(A.row_sizes, A.col_sizes)
    _same(got, want)


@pytest.mark.parametrize("kind,okind", [(FSAI_STATIC_LOWER, O.Fsai.STATIC), (FSAI_ADAPTIVE, O.Fsai.NESTED)])
def test_fsai_variable_bitwise(ctx, kind, okind):
    A, _, _ = _problem(16, 2)
    M = Fsai.build(BlockSparseMatrix(ctx, A), kind, t_max=2)
    _same(M.G.download(A.row_sizes, A.col_sizes), O.Fsai(O.Mat(A), okind, t_max=2).G().export())


@pytest.mark.parametrize("nest,t_max", [(0, 1), (1, 1), (0, 2)])
def test_variable_hierarchy_history_matches_oracle(ctx, nest, t_max):
    # setup (multilevel.cpp:36-75: nested_build per level) on a mixed 6 / 10 layout
    A, T, b = _problem(16, 3)
    okw = dict(t_max=t_max, nest=nest, coarse_dim_cap=1 << 30, probe=False)
    kw = dict(t_max=t_max, nest=nest, coarse_dim_cap=1 << 30)
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], **okw)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T], default_params(**kw))
    for l in range(1, dh.levels):
        assert abs(dh.beta(l) - oh.beta(l)) <= 1e-10 * oh.beta(l)
    hist_o, it_o, st_o, _ = oh.solve(3, 3, b, np.zeros_like(b), 1e-8, 12)
    hist_g, it_g, st_g = dh.solve(3, 3, Vector(ctx, b), Vector(ctx, b.size), 1e-8, 12)
    assert it_g == it_o and st_g == st_o
    rho_o, rho_g = hist_o / hist_o[0], hist_g / hist_g[0]
    assert np.all(np.abs(rho_g - rho_o) <= 1e-10)
    big = rho_o >= 1e-2
    assert np.all(np.abs(rho_g[big] / rho_o[big] - 1) <= 1e-10)


def test_variable_hierarchy_rejects_partition(ctx):
    from paper_2509_06744_b200.native import InvalidArgument
    A, T, b = _problem(8, 2)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, coarse_dim_cap=1 << 30))
    with pytest.raises(InvalidArgument, match="variable"):
        dh.partition(2, [8, 4])


def test_matrix_io_variable_system_solves_identically(ctx, tmp_path):
    # a PUM-style export (matrix_io.cpp:39-58: scalar triplets + .blocks sidecar) read
    # straight into a device matrix, then setup + solve: same history, bitwise
    from paper_2509_06744_b200 import read_matrix, read_vector, write_matrix, write_vector
    A, T, b = _problem(16, 3)
    dA = BlockSparseMatrix(ctx, A)
    write_matrix(dA, str(tmp_path / "A.mtx"))
    write_vector(Vector(ctx, b), str(tmp_path / "b.vec"))
    rA, sym = read_matrix(ctx, str(tmp_path / "A.mtx"))
    assert sym
    rb = read_vector(ctx, str(tmp_path / "b.vec"))
    params = default_params(t_max=1, coarse_dim_cap=1 << 30)
    dT = [BlockSparseMatrix(ctx, p) for p in T]
    h1 = Hierarchy.setup(dA, dT, params)
    h2 = Hierarchy.setup(rA, dT, params)
    x1, x2 = Vector(ctx, b.size), Vector(ctx, b.size)
    r1 = h1.solve(3, 3, Vector(ctx, b), x1, 1e-8, 6)
    r2 = h2.solve(3, 3, rb, x2, 1e-8, 6)
    assert r1[1] == r2[1] and np.array_equal(r1[0], r2[0])
    assert np.array_equal(x1.download(), x2.download())
