"""GPU parity of the streaming kernels against the oracle (bitwise where the
arithmetic order is shared, see oracle/bmg_oracle.cpp header).

Reference behaviour: spmv / spmv_transpose (kernels.cpp:39-64), the residual
r = b - A x of cheb_fourth_apply (chebyshev.hpp:55-56) and the V-cycle
(multilevel.cpp:91-93), prolongation x += P e (multilevel.cpp:98-100).
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import BlockSparseMatrix, Vector, residual, spmv, spmv_transpose
from paper_2509_06744_b200 import problems as pr
from tests.helpers import random_bsr, random_layout

pytestmark = pytest.mark.gpu


def _dev_spmv(ctx, host, x):
    A = BlockSparseMatrix(ctx, host)
    xv = Vector(ctx, x)
    yv = Vector(ctx, host.dim_r)
    spmv(A, xv, yv)
    return yv.download()


@pytest.mark.parametrize("m", [3, 6, 10, 15, 20, 21])
@pytest.mark.parametrize("density", [0.05, 0.4, 1.0])
def test_spmv_uniform_bitwise(ctx, rng, m, density):
    # density 1.0 gives rows far longer than one chunk (carry across chunks)
    nbr, nbc = 37, 41
    host = random_bsr(rng, np.full(nbr, m, np.int32), np.full(nbc, m, np.int32), density)
    x = rng.standard_normal(host.dim_c)
    got = _dev_spmv(ctx, host, x)
    want = O.Mat(host).spmv(x)
    assert np.array_equal(got, want)


def test_spmv_empty_rows_and_matrix(ctx, rng):
    m = 10
    host = random_bsr(rng, np.full(50, m, np.int32), np.full(20, m, np.int32), 0.02)
    assert (np.diff(host.row_ptr) == 0).any()
    x = rng.standard_normal(host.dim_c)
    assert np.array_equal(_dev_spmv(ctx, host, x), O.Mat(host).spmv(x))
    empty = random_bsr(rng, np.full(5, m, np.int32), np.full(5, m, np.int32), 0.0)
    assert np.array_equal(_dev_spmv(ctx, empty, np.ones(50)), np.zeros(50))


def test_spmv_variable_layout_bitwise(ctx, rng):
    for rep in range(10):
        rs = random_layout(rng, 12, 4)
        cs = random_layout(rng, 12, 4)
        host = random_bsr(rng, rs, cs, 0.5)
        x = rng.standard_normal(host.dim_c)
        assert np.array_equal(_dev_spmv(ctx, host, x), O.Mat(host).spmv(x))


@pytest.mark.parametrize("m", [10, 15, 3, 6])
def test_spmv_transpose_and_residual_bitwise(ctx, rng, m):
    host = random_bsr(rng, np.full(29, m, np.int32), np.full(23, m, np.int32), 0.3)
    A = BlockSparseMatrix(ctx, host)
    o = O.Mat(host)
    x = rng.standard_normal(host.dim_r)
    xv, yv = Vector(ctx, x), Vector(ctx, host.dim_c)
    spmv_transpose(A, xv, yv)
    assert np.array_equal(yv.download(), o.spmv_t(x))
    xc = rng.standard_normal(host.dim_c)
    b = rng.standard_normal(host.dim_r)
    rv = Vector(ctx, host.dim_r)
    residual(A, Vector(ctx, b), Vector(ctx, xc), rv)
    assert np.array_equal(rv.download(), b - o.spmv(xc))


def test_spmv_baseline_stencil_bitwise(ctx):
    # C1's operator (64^2 patches, m = 10, 13-point block stencil)
    host = pr.stencil_matrix(2, 64, 2, 10)
    x = pr.normal_vector(host.dim_c, 0, 7)
    assert np.array_equal(_dev_spmv(ctx, host, x), O.Mat(host).spmv(x))


def test_spmv_length_validation(ctx, rng):
    from paper_2509_06744_b200 import InvalidArgument

    host = random_bsr(rng, np.full(4, 10, np.int32), np.full(4, 10, np.int32), 0.5)
    A = BlockSparseMatrix(ctx, host)
    with pytest.raises(InvalidArgument):
        spmv(A, Vector(ctx, 39), Vector(ctx, 40))


def test_objects_outlive_their_context_handle():
    # handles may be destroyed in any order (the C objects keep their context alive):
    # closing the context first must neither crash nor break the objects still in use
    import gc

    from paper_2509_06744_b200 import BlockSparseMatrix, Context, Vector, spmv
    from paper_2509_06744_b200 import problems as pr
    c = Context(0)
    host = pr.stencil_matrix(2, 8, 2, 10)
    A = BlockSparseMatrix(c, host)
    x = Vector(c, pr.normal_vector(host.dim_c, 0, 1))
    y = Vector(c, host.dim_r)
    c.close()
    spmv(A, x, y)
    assert np.isfinite(y.download()).all()
    del A, x
    gc.collect()
    y.close()
