"""The CUDA path against THE REFERENCE ITSELF (oracle/_ref/libblockmg_ref.so: the
reference's own sources, built in the container against oracle/eigen_shim and
shipped prebuilt -- see oracle/ref_driver.cpp), through the C ABI, without the
oracle in between.

  * spmv / spmv_transpose (kernels.cpp:39-64): bitwise;
  * setup (multilevel.cpp:36-75) on the C2 / C4 / C5 / C3 shapes: Galerkin operators
    and FSAI factors bitwise, beta_l to 1e-10;
  * the stop-on-tolerance solve around v_cycle (multilevel.cpp:77-103,
    experiments.cpp:46-58): |rho_gpu - rho_ref| <= 1e-10 per cycle, relative 1e-10
    while rho >= 1e-2, equal iteration counts;
  * measure_rates (experiments.cpp:15-67) on the reference's own fd_biharmonic
    problem (experiments.cpp:104-195), inputs produced by the reference.
"""
import numpy as np
import pytest

from oracle import pyref as R
from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy, Vector, default_params, spmv, spmv_transpose
from paper_2509_06744_b200 import problems as pr
from tests.golden.make_solve_golden import bsr_digest
from tests.helpers import random_bsr, random_layout

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="reference build (oracle/_ref) unavailable")]


def test_spmv_bitwise_against_the_reference(ctx, rng):
    for m in (10, 15, 20, 21):
        sizes = np.full(40, m, np.int32)
        h = random_bsr(rng, sizes, sizes, 0.2, min_per_row=1)
        x = rng.normal(size=h.dim_c)
        A, ref = BlockSparseMatrix(ctx, h), R.Mat(h)
        y = Vector(ctx, h.dim_r)
        spmv(A, Vector(ctx, x), y)
        assert np.array_equal(y.download(), ref.spmv(x))
        z = Vector(ctx, h.dim_c)
        spmv_transpose(A, Vector(ctx, x[:h.dim_r]), z)
        assert np.array_equal(z.download(), ref.spmv_t(x[:h.dim_r]))
    for rep in range(5):  # the reference's general layouts (variable m_i)
        h = random_bsr(rng, random_layout(rng, 12, 6), random_layout(rng, 12, 6), 0.5)
        x = rng.normal(size=h.dim_c)
        y = Vector(ctx, h.dim_r)
        spmv(BlockSparseMatrix(ctx, h), Vector(ctx, x), y)
        assert np.array_equal(y.download(), R.Mat(h).spmv(x))


SHAPES = [
    ("C2", (16, 3), 0, 3),
    ("C4", (8, 3), 0, 3),
    ("C5", (32, 4), 0, 3),
    ("C3", (32, 3), 1, 4),
]


@pytest.mark.parametrize("name,scaled,nest,k", SHAPES, ids=[s[0] for s in SHAPES])
def test_setup_and_solve_against_the_reference(ctx, name, scaled, nest, k):
    cfg = pr.CONFIGS[name].scaled(*scaled)
    A, T, b = pr.make_problem(cfg)
    rh = R.Hierarchy(R.Mat(A), [R.Mat(p) for p in T], t_max=1, tau=1.0, nest=nest, coarse_dim_cap=1 << 30)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, tau=1.0, nest=nest, coarse_dim_cap=1 << 30))
    assert dh.levels == rh.levels()
    for l in range(dh.levels):
        Al, _, M = dh.level(l)
        sizes = np.full(Al.info()["nbr"], cfg.m, np.int32)
        assert bsr_digest(Al.download(sizes, sizes, symmetric=True)) == bsr_digest(rh.A(l).export(symmetric=True))
        if l == 0:
            continue
        f = rh.fsai(l)
        assert M.chain_len == f.chain_len()
        for q in range(f.chain_len() - 1):
            assert bsr_digest(M.factor(q).download(sizes, sizes)) == bsr_digest(f.factor(q).export())
        assert bsr_digest(M.G.download(sizes, sizes)) == bsr_digest(f.G().export())
        assert abs(dh.beta(l) - rh.beta(l)) <= 1e-10 * rh.beta(l)
    want, it_r, st_r, x_r = rh.solve(k, k, b, np.zeros_like(b), tol=1e-8, max_iter=40)
    xg = Vector(ctx, b.size)
    got, it_g, st_g = dh.solve(k, k, Vector(ctx, b), xg, 1e-8, 40)
    assert (it_g, st_g) == (it_r, st_r)
    rho_g, rho_r = np.asarray(got) / got[0], want / want[0]
    assert np.max(np.abs(rho_g - rho_r)) <= 1e-10
    big = rho_r >= 1e-2
    assert np.max(np.abs(rho_g[big] - rho_r[big]) / rho_r[big]) <= 1e-10
    assert np.linalg.norm(xg.download() - x_r) <= 1e-10 * np.linalg.norm(x_r)


def test_measure_rates_on_the_references_fd_problem(ctx):
    fd = R.fd_biharmonic(32, 3)  # inputs made by the reference (experiments.cpp:104-195)
    A, mass = fd["A"].export(symmetric=True), fd["mass"].export(symmetric=True)
    T = [p.export() for p in fd["transfers"]]
    b, u = fd["b"], fd["reference"]
    rh = R.Hierarchy(fd["A"], fd["transfers"], t_max=2)
    want = rh.measure_rates(fd["mass"], b, u, 2, 2, seed=1, tol=1e-9, max_iter=60)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T], default_params(t_max=2))
    got = dh.measure_rates(BlockSparseMatrix(ctx, mass), Vector(ctx, b), Vector(ctx, u), 2, 2, seed=1, tol=1e-9,
                           max_iter=60)
    assert (got["iterations"], got["status"]) == (want["iterations"], want["status"])
    # histories in units of the field's own norm (tests/test_gpu_fd_problem.py: the
    # error is measured against an exact field, so rounding-level differences of the
    # iterates are relative differences of ~eps |u| / |e| in the tail)
    Ad = A.to_dense()
    it = got["iterations"]
    scales = {"l2_sq": np.sqrt(u @ (mass.to_dense() @ u)), "energy_sq": np.sqrt(u @ (Ad @ u)),
              "residual": np.linalg.norm(b)}
    for key, rate in (("l2_sq", "rho_l2"), ("energy_sq", "rho_a"), ("residual", "rho_r")):
        g, w = got[key], want[key]
        if key != "residual":
            g, w = np.sqrt(g), np.sqrt(w)
        delta = 1e-12 * scales[key] * (np.arange(g.size) + 1)
        assert np.all(np.abs(g - w) <= delta), key
        assert abs(got[rate] - want[rate]) <= (delta[-1] / (it * w[-1]) + 1e-12) * want[rate], rate


def test_matrix_io_files_cross_read(ctx, rng, tmp_path):
    """matrix_io.cpp: a file written by the reference is read by the product and
    the other way round, values and pattern exact; vectors likewise."""
    from paper_2509_06744_b200 import api
    from tests.helpers import random_spd

    sizes = random_layout(rng, 7, 5)
    a = random_spd(rng, sizes, 0.6)
    p_ref, p_dev = str(tmp_path / "ref.bmat"), str(tmp_path / "dev.bmat")
    R.write_matrix(p_ref, R.Mat(a))
    got, _ = api.read_matrix(ctx, p_ref)
    assert bsr_digest(got.download(sizes, sizes, symmetric=True)) == bsr_digest(a)
    api.write_matrix(BlockSparseMatrix(ctx, a), p_dev)
    back = R.read_matrix(p_dev)
    assert bsr_digest(back.export(symmetric=True)) == bsr_digest(a)
    assert np.array_equal(back.row_sizes, sizes)
    v = rng.normal(size=23)
    R.write_vector(str(tmp_path / "v_ref.txt"), v)
    assert np.array_equal(api.read_vector(ctx, str(tmp_path / "v_ref.txt")).download(), v)
    api.write_vector(Vector(ctx, v), str(tmp_path / "v_dev.txt"))
    assert np.array_equal(R.read_vector(str(tmp_path / "v_dev.txt")), v)
