"""GPU parity of FSAI setup/apply, Galerkin coarsening, Lanczos, the fourth-kind
smoother and the V-cycle against the oracle restatement of the reference.

Tolerances (written per test):
  * G (= L^{-1} F) and Galerkin operators: bitwise -- same arithmetic order;
  * M r = G^T G r vs the reference's F^T S^{-1} F r: 1e-12 relative (the
    per-row solves are folded into G at setup, a rounding-level change);
  * beta (Lanczos): 1e-10 relative;
  * residual histories: |rho_gpu - rho_cpu| <= 1e-10 and relative 1e-10 while
    rho >= 1e-2.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import (FSAI_ADAPTIVE, FSAI_STATIC_LOWER, BlockSparseMatrix, Fsai, Hierarchy,
                                   NotPositiveDefinite, Vector, cheb_fourth_apply, default_params,
                                   galerkin_coarsen, lanczos_lambda_max)
from paper_2509_06744_b200 import problems as pr
from tests.helpers import random_layout, random_spd

pytestmark = pytest.mark.gpu


def _download(mat, sizes_r, sizes_c):
    return mat.download(sizes_r, sizes_c)


def _assert_same_bsr(got, want):
    assert np.array_equal(got.row_ptr, want.row_ptr)
    assert np.array_equal(got.col_idx, want.col_idx)
    assert np.array_equal(got.vals, want.vals)


@pytest.mark.parametrize("kind,okind", [(FSAI_STATIC_LOWER, O.Fsai.STATIC), (FSAI_ADAPTIVE, O.Fsai.NESTED)])
def test_fsai_G_bitwise_on_stencil(ctx, kind, okind):
    host = pr.stencil_matrix(2, 16, 2, 10)
    A = BlockSparseMatrix(ctx, host)
    M = Fsai.build(A, kind, t_max=1, tau=1.0, nest=0)
    of = O.Fsai(O.Mat(host), okind, t_max=1, tau=1.0, nest=0)
    want = of.G().export()
    got = M.G.download(host.row_sizes, host.col_sizes)
    _assert_same_bsr(got, want)


def test_fsai_variable_layout_and_apply(ctx, rng):
    for rep in range(5):
        sizes = random_layout(rng, 10, 4)
        host = random_spd(rng, sizes, 0.6)
        A = BlockSparseMatrix(ctx, host)
        for kind, okind in [(FSAI_STATIC_LOWER, O.Fsai.STATIC), (FSAI_ADAPTIVE, O.Fsai.NESTED)]:
            M = Fsai.build(A, kind, t_max=1)
            of = O.Fsai(O.Mat(host), okind, t_max=1)
            _assert_same_bsr(M.G.download(sizes, sizes), of.G().export())
            r = rng.standard_normal(host.dim_r)
            z = Vector(ctx, host.dim_r)
            M.apply(Vector(ctx, r), z)
            want = of.apply(r)
            assert np.linalg.norm(z.download() - want) <= 1e-12 * np.linalg.norm(want)


def test_fsai_from_factors_matches_oracle_apply(ctx, rng):
    host = pr.stencil_matrix(2, 12, 2, 10)
    of = O.Fsai(O.Mat(host), O.Fsai.STATIC)
    F = of.factor(0).export()
    M = Fsai.from_factors(ctx, BlockSparseMatrix(ctx, F), of.shat())
    r = rng.standard_normal(host.dim_r)
    z = Vector(ctx, host.dim_r)
    M.apply(Vector(ctx, r), z)
    want = of.apply(r)
    assert np.linalg.norm(z.download() - want) <= 1e-12 * np.linalg.norm(want)
    _assert_same_bsr(M.G.download(host.row_sizes, host.col_sizes), of.G().export())


def test_fsai_not_spd_reports_pivot(ctx):
    from tests.helpers import from_dense_blocks

    blocks = {(0, 0): np.array([[1.0, 2.0], [2.0, 1.0]])}
    host = from_dense_blocks(np.array([2], np.int32), np.array([2], np.int32), blocks, symmetric=True)
    with pytest.raises(NotPositiveDefinite) as ei:
        Fsai.build(BlockSparseMatrix(ctx, host), FSAI_STATIC_LOWER)
    assert ei.value.pivot == 1


def test_galerkin_bitwise(ctx):
    cfg = pr.CONFIGS["C2"].scaled(16, 2)
    A, T, b = pr.make_problem(cfg)
    dA = BlockSparseMatrix(ctx, A)
    dP = BlockSparseMatrix(ctx, T[0])
    got = galerkin_coarsen(dA, dP).download(T[0].col_sizes, T[0].col_sizes)
    want = O.galerkin(O.Mat(A), O.Mat(T[0])).export()
    _assert_same_bsr(got, want)


def test_lanczos_matches_oracle(ctx):
    host = pr.stencil_matrix(2, 16, 2, 10)
    A = BlockSparseMatrix(ctx, host)
    M = Fsai.build(A, FSAI_ADAPTIVE, t_max=1)
    om, of = O.Mat(host), O.Fsai(O.Mat(host), O.Fsai.NESTED, t_max=1)
    got = lanczos_lambda_max(A, M, 100, 1.01, 42)
    want = O.lanczos_lambda_max(om, of, 100, 1.01, 42)
    assert abs(got - want) <= 1e-10 * want


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_cheb4_matches_oracle(ctx, k):
    host = pr.stencil_matrix(2, 32, 2, 10)
    A = BlockSparseMatrix(ctx, host)
    om = O.Mat(host)
    of = O.Fsai(om, O.Fsai.STATIC)
    M = Fsai.build(A, FSAI_STATIC_LOWER)
    beta = O.lanczos_lambda_max(om, of, 100, 1.01, 42)
    b = pr.normal_vector(host.dim_r, 0, 0)
    x0 = pr.normal_vector(host.dim_r, 0, 3)
    xv = Vector(ctx, x0)
    cheb_fourth_apply(A, M, Vector(ctx, b), xv, beta, k)
    want = O.smoother_apply(om, of, O.CHEB_FOURTH, b, x0, k, beta=beta)
    got = xv.download()
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def _small_hierarchies(ctx, n=32, levels=3):
    cfg = pr.CONFIGS["C2"].scaled(n, levels)
    A, T, b = pr.make_problem(cfg)
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, coarse_dim_cap=1 << 30, probe=False)
    dA = BlockSparseMatrix(ctx, A)
    dT = [BlockSparseMatrix(ctx, p) for p in T]
    dh = Hierarchy.setup(dA, dT, default_params(t_max=1, coarse_dim_cap=1 << 30))
    return A, T, b, oh, dh


def test_vcycle_setup_and_history_match_oracle(ctx):
    A, T, b, oh, dh = _small_hierarchies(ctx)
    for l in range(1, dh.levels):
        assert abs(dh.beta(l) - oh.beta(l)) <= 1e-10 * oh.beta(l)
    hist_o, it_o, st_o, _ = oh.solve(3, 3, b, np.zeros_like(b), 1e-8, 40)
    bv, xv = Vector(ctx, b), Vector(ctx, np.zeros_like(b))
    hist_g, it_g, st_g = dh.solve(3, 3, bv, xv, 1e-8, 40)
    assert it_g == it_o and st_g == st_o
    rho_o, rho_g = hist_o / hist_o[0], hist_g / hist_g[0]
    assert np.all(np.abs(rho_g - rho_o) <= 1e-10)
    big = rho_o >= 1e-2
    assert np.all(np.abs(rho_g[big] / rho_o[big] - 1) <= 1e-10)


def test_vcycle_injected_hierarchy_matches_oracle(ctx):
    # apply-phase parity isolated from setup: oracle-built
    # A_l, P_l, F/S-hat factors and beta_l injected into the device V-cycle
    A, T, b, oh, _ = _small_hierarchies(ctx)
    L = oh.levels()
    As = [BlockSparseMatrix(ctx, oh.A(l).export(symmetric=True)) for l in range(L)]
    Ps = [None] + [BlockSparseMatrix(ctx, oh.P(l).export()) for l in range(1, L)]
    Ms = [None]
    for l in range(1, L):
        f = oh.fsai(l)
        Ms.append(Fsai.from_factors(ctx, BlockSparseMatrix(ctx, f.factor(0).export()), f.shat()))
    betas = [0.0] + [oh.beta(l) for l in range(1, L)]
    dh = Hierarchy.create(ctx, As, Ps, Ms, betas)
    x_o = np.zeros_like(b)
    xv = Vector(ctx, x_o)
    bv = Vector(ctx, b)
    for it in range(5):
        x_o = oh.v_cycle(3, 3, b, x_o)
        dh.v_cycle(3, 3, bv, xv)
        x_g = xv.download()
        assert np.linalg.norm(x_g - x_o) <= 1e-11 * np.linalg.norm(x_o)


def test_vcycle_fixed_point_linearity_graph(ctx, rng):
    # test_multilevel.cpp:108-127: zero rhs keeps zero; superposition
    A, T, b, oh, dh = _small_hierarchies(ctx, 16, 2)
    n = A.dim_r
    x = Vector(ctx, n)
    dh.v_cycle(2, 2, Vector(ctx, np.zeros(n)), x)
    assert np.linalg.norm(x.download()) == 0.0
    b1, b2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    outs = []
    for rhs in (b1, b2, 0.5 * b1 - 2.0 * b2):
        xv = Vector(ctx, n)
        dh.v_cycle(2, 2, Vector(ctx, rhs), xv)
        outs.append(xv.download())
    xa, xb, xc = outs
    assert np.linalg.norm(xc - (0.5 * xa - 2.0 * xb)) <= 1e-12 * (1.0 + np.linalg.norm(xc))
    # graph replay == eager launch, bitwise
    x1, x2 = Vector(ctx, n), Vector(ctx, n)
    bv = Vector(ctx, b1)
    dh.use_graph(True)
    dh.v_cycle(3, 3, bv, x1)
    dh.v_cycle(3, 3, bv, x1)
    dh.use_graph(False)
    dh.v_cycle(3, 3, bv, x2)
    dh.v_cycle(3, 3, bv, x2)
    dh.use_graph(True)
    assert np.array_equal(x1.download(), x2.download())


def test_vcycle_host_e2e_equals_device(ctx):
    A, T, b, oh, dh = _small_hierarchies(ctx, 16, 2)
    x_host = np.zeros_like(b)
    dh.v_cycle_host(3, 3, b, x_host)
    xv = Vector(ctx, b.size)
    dh.v_cycle(3, 3, Vector(ctx, b), xv)
    assert np.array_equal(x_host, xv.download())


def test_single_level_hierarchy_direct_solve(ctx):
    # test_multilevel.cpp:99-106: one level -> x = A^{-1} b
    host = pr.stencil_matrix(2, 8, 2, 10)
    A = BlockSparseMatrix(ctx, host)
    dh = Hierarchy.setup(A, [], default_params(t_max=1, coarse_dim_cap=1 << 30))
    b = pr.normal_vector(host.dim_r, 0, 0)
    xv = Vector(ctx, host.dim_r)
    dh.v_cycle(2, 2, Vector(ctx, b), xv)
    want = np.linalg.solve(host.to_dense(), b)
    assert np.linalg.norm(xv.download() - want) <= 1e-9 * np.linalg.norm(want)


@pytest.mark.parametrize("world,agg", [(2, 1), (3, 2), (4, 1)])
def test_partitioned_vcycle_bitwise_equal_to_single(ctx, world, agg):
    # row strips + halo exchange; per-row arithmetic is partition
    # independent, so emulated ranks (in-process halos) match the 1-GPU cycle bitwise
    cfg = pr.CONFIGS["C2"].scaled(32, 3)
    A, T, b = pr.make_problem(cfg)
    params = default_params(t_max=1, coarse_dim_cap=1 << 30)
    dA = BlockSparseMatrix(ctx, A)
    dT = [BlockSparseMatrix(ctx, p) for p in T]
    h1 = Hierarchy.setup(dA, dT, params)
    h2 = Hierarchy.setup(dA, dT, params)
    granule = [cfg.n >> (cfg.levels - 1 - l) for l in range(cfg.levels)]
    h1.partition(1, granule)  # same residual-norm segmentation (one segment per grid row)
    h2.partition(world, granule, agglomerate=agg)
    for l in range(cfg.levels):
        spans = [h2.part_info(l, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == A.nbr >> (2 * (cfg.levels - 1 - l))
        if l < agg:
            assert all(s[1] == s[0] for s in spans[1:])
    x1, x2 = Vector(ctx, b.size), Vector(ctx, b.size)
    bv = Vector(ctx, b)
    for it in range(3):
        h1.v_cycle(3, 3, bv, x1)
        h2.v_cycle(3, 3, bv, x2)
        assert np.array_equal(x1.download(), x2.download())
    x1, x2 = Vector(ctx, b.size), Vector(ctx, b.size)
    hist1, it1, _ = h1.solve(3, 3, bv, x1, 1e-8, 6)
    hist2, it2, _ = h2.solve(3, 3, bv, x2, 1e-8, 6)
    assert it1 == it2 and np.array_equal(hist1, hist2)


@pytest.mark.parametrize("t_max", [2, 3])
def test_adaptive_fsai_general_tmax_bitwise(ctx, rng, t_max):
    # adaptive_build with t_max > 1 (fsai.cpp:132-198): same pattern, bitwise G
    host = pr.stencil_matrix(2, 12, 2, 10)
    M = Fsai.build(BlockSparseMatrix(ctx, host), FSAI_ADAPTIVE, t_max=t_max)
    of = O.Fsai(O.Mat(host), O.Fsai.NESTED, t_max=t_max)
    _assert_same_bsr(M.G.download(host.row_sizes, host.col_sizes), of.G().export())
    for rep in range(3):
        sizes = random_layout(rng, 9, 3)
        h2 = random_spd(rng, sizes, 0.7)
        M2 = Fsai.build(BlockSparseMatrix(ctx, h2), FSAI_ADAPTIVE, t_max=t_max)
        of2 = O.Fsai(O.Mat(h2), O.Fsai.NESTED, t_max=t_max)
        _assert_same_bsr(M2.G.download(sizes, sizes), of2.G().export())


def test_triple_product_bitwise(ctx, rng):
    # kernels.cpp:88-119 on the device (F from a static FSAI of a stencil)
    host = pr.stencil_matrix(2, 10, 2, 10)
    of = O.Fsai(O.Mat(host), O.Fsai.STATIC)
    F = of.factor(0).export()
    want = O.triple_product(O.Mat(F), O.Mat(host)).export(symmetric=True)
    from paper_2509_06744_b200 import triple_product

    got = triple_product(BlockSparseMatrix(ctx, F), BlockSparseMatrix(ctx, host)).download(
        host.row_sizes, host.col_sizes)
    _assert_same_bsr(got, want)


@pytest.mark.parametrize("t_max,nest", [(1, 1), (2, 1), (1, 2)])
def test_nested_fsai_chain_matches_oracle(ctx, rng, t_max, nest):
    # nested_build (fsai.cpp:243-253): F_0 .. F_{n-1} bitwise, G_n = L^-1 F_n bitwise,
    # M r (chain apply, fsai.cpp:200-217) and beta within rounding
    host = pr.stencil_matrix(2, 12, 2, 10)
    A = BlockSparseMatrix(ctx, host)
    M = Fsai.build(A, FSAI_ADAPTIVE, t_max=t_max, nest=nest)
    om = O.Mat(host)
    of = O.Fsai(om, O.Fsai.NESTED, t_max=t_max, nest=nest)
    assert M.chain_len == of.chain_len() == nest + 1
    for k in range(nest):
        _assert_same_bsr(M.factor(k).download(host.row_sizes, host.col_sizes), of.factor(k).export())
    _assert_same_bsr(M.G.download(host.row_sizes, host.col_sizes), of.G().export())
    r = rng.standard_normal(host.dim_r)
    z = Vector(ctx, host.dim_r)
    M.apply(Vector(ctx, r), z)
    want = of.apply(r)
    assert np.linalg.norm(z.download() - want) <= 1e-12 * np.linalg.norm(want)
    beta = lanczos_lambda_max(A, M, 100, 1.01, 42)
    assert abs(beta - O.lanczos_lambda_max(om, of, 100, 1.01, 42)) <= 1e-10 * beta


def test_nested_hierarchy_history_matches_oracle(ctx):
    # C3's smoother (nest = 1) inside the V-cycle, small 2-D triharmonic-like problem
    cfg = pr.CONFIGS["C3"].scaled(16, 2)
    cfg.m = 10
    A, T, b = pr.make_problem(cfg)
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, nest=1, coarse_dim_cap=1 << 30, probe=False)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, nest=1, coarse_dim_cap=1 << 30))
    hist_o, it_o, st_o, _ = oh.solve(4, 4, b, np.zeros_like(b), 1e-8, 15)
    hist_g, it_g, st_g = dh.solve(4, 4, Vector(ctx, b), Vector(ctx, b.size), 1e-8, 15)
    assert it_o == it_g
    assert np.all(np.abs(hist_g / hist_g[0] - hist_o / hist_o[0]) <= 1e-10)


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_apply_smoother_kinds_match_oracle(ctx, kind):
    # apply_smoother (chebyshev.hpp:117-129): Richardson, first kind on [beta/30, beta], fourth kind
    from paper_2509_06744_b200 import apply_smoother

    host = pr.stencil_matrix(2, 16, 2, 10)
    A = BlockSparseMatrix(ctx, host)
    om = O.Mat(host)
    of = O.Fsai(om, O.Fsai.STATIC)
    M = Fsai.build(A, FSAI_STATIC_LOWER)
    beta = O.lanczos_lambda_max(om, of, 100, 1.01, 42)
    alpha, omega = beta / 30.0, 1.0 / beta
    b = pr.normal_vector(host.dim_r, 0, 0)
    x0 = pr.normal_vector(host.dim_r, 0, 3)
    for k in (1, 3, 4):
        xv = Vector(ctx, x0)
        apply_smoother(A, M, kind, Vector(ctx, b), xv, k, alpha=alpha, beta=beta, omega=omega)
        want = O.smoother_apply(om, of, kind, b, x0, k, alpha=alpha, beta=beta, omega=omega)
        assert np.linalg.norm(xv.download() - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("kind,kpre,kpost", [(1, 2, 2), (0, 3, 3), (2, 6, 0), (2, 0, 4), (2, 1, 5)])
def test_vcycle_smoother_kinds_and_v2k0(ctx, kind, kpre, kpost):
    # SetupParams::kind / first_kind_fraction / richardson_omega (multilevel.hpp:39-42,
    # multilevel.cpp:62-65) and CycleSpec::v2k0 (multilevel.hpp:18)
    cfg = pr.CONFIGS["C2"].scaled(16, 3)
    A, T, b = pr.make_problem(cfg)
    omega = 0.3
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, coarse_dim_cap=1 << 30, probe=False,
                     smoother_kind=kind, richardson_omega=omega)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, coarse_dim_cap=1 << 30, smoother_kind=kind,
                                        richardson_omega=omega))
    hist_o, it_o, _, _ = oh.solve(kpre, kpost, b, np.zeros_like(b), 1e-8, 8)
    hist_g, it_g, _ = dh.solve(kpre, kpost, Vector(ctx, b), Vector(ctx, b.size), 1e-8, 8)
    assert it_o == it_g
    assert np.all(np.abs(hist_g / hist_g[0] - hist_o / hist_o[0]) <= 1e-10)


def _block_diag(host):
    # the diagonal blocks of an s.p.d. block matrix: an s.p.d. stand-in for the PUM mass matrix
    m = int(host.row_sizes[0])
    n = host.nbr
    vals = []
    for i in range(n):
        for p in range(host.row_ptr[i], host.row_ptr[i + 1]):
            if host.col_idx[p] == i:
                vals.append(host.vals[p * m * m:(p + 1) * m * m])
    from paper_2509_06744_b200.api import HostBsr
    return HostBsr(host.row_sizes, host.col_sizes, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
                   np.concatenate(vals), True)


@pytest.mark.parametrize("tol,max_iter", [(1e-3, 30), (1e-30, 6), (10.0, 5)])
def test_measure_rates_matches_oracle(ctx, tol, max_iter):
    # measure_rates (experiments.cpp:15-67): error histories in the M- and A-norms,
    # residual history, iteration count, status and the three rates
    cfg = pr.CONFIGS["C2"].scaled(16, 3)
    A, T, _ = pr.make_problem(cfg)
    Mh = _block_diag(A)
    u = pr.normal_vector(A.dim_r, 0, 7)
    b = O.Mat(A).spmv(u)
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, coarse_dim_cap=1 << 30, probe=False)
    want = oh.measure_rates(O.Mat(Mh), b, u, 3, 3, seed=11, tol=tol, max_iter=max_iter)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, coarse_dim_cap=1 << 30))
    got = dh.measure_rates(BlockSparseMatrix(ctx, Mh), Vector(ctx, b), Vector(ctx, u), 3, 3, seed=11, tol=tol,
                           max_iter=max_iter)
    assert got["iterations"] == want["iterations"] and got["status"] == want["status"]
    assert got["blowup_iteration"] == want["blowup_iteration"]
    for key in ("l2_sq", "energy_sq", "residual"):
        g, w = got[key], want[key]
        assert np.all(np.abs(g / w[0] - w / w[0]) <= 1e-10), key
    for key in ("rho_l2", "rho_a", "rho_r"):
        assert abs(got[key] - want[key]) <= 1e-9 * max(abs(want[key]), 1e-300), key
    if tol == 10.0:
        assert got["iterations"] == 0 and got["status"] == 0 and got["rho_l2"] == 0.0


def test_vcycle_from_every_level_matches_oracle(ctx, rng):
    # v_cycle(h, spec, level, b, x) (multilevel.cpp:77-103) from each level, with a
    # nonzero initial guess; level 0 is the dense direct solve
    A, T, b, oh, dh = _small_hierarchies(ctx, 16, 3)
    for level in range(dh.levels):
        n = oh.A(level).export(symmetric=True).dim_r
        bl = rng.standard_normal(n)
        x0 = rng.standard_normal(n)
        want = oh.v_cycle(2, 1, bl, x0.copy(), level=level)
        xv = Vector(ctx, x0.copy())
        dh.v_cycle_level(2, 1, level, Vector(ctx, bl), xv)
        got = xv.download()
        assert np.linalg.norm(got - want) <= 1e-11 * np.linalg.norm(want), level
    from paper_2509_06744_b200.native import OutOfRange
    with pytest.raises(OutOfRange):
        dh.v_cycle_level(2, 2, dh.levels, Vector(ctx, 4), Vector(ctx, 4))


@pytest.mark.parametrize("layout", ["stencil", "variable"])
def test_fsai_user_pattern_bitwise(ctx, rng, layout):
    # build_fsai(A, LowerPattern p) (fsai.hpp:25) with a caller's pattern: G bitwise
    if layout == "stencil":
        host = pr.stencil_matrix(2, 12, 2, 10)
    else:
        host = random_spd(rng, random_layout(rng, 14, 5), 0.5)
    n = host.nbr
    pattern = []
    for i in range(n):
        lower = [int(j) for j in host.col_idx[host.row_ptr[i]:host.row_ptr[i + 1]] if j < i]
        extra = [int(j) for j in rng.integers(0, i + 1, size=2)] if i > 0 else []
        pattern.append(sorted(set(lower[::2] + extra + [i])))
    M = Fsai.from_pattern(BlockSparseMatrix(ctx, host), pattern)
    want = O.fsai_with_pattern(O.Mat(host), [[j for j in row if j < i] for i, row in enumerate(pattern)])
    _assert_same_bsr(M.G.download(host.row_sizes, host.col_sizes), want.G().export())
    from paper_2509_06744_b200.native import InvalidArgument
    with pytest.raises(InvalidArgument):
        Fsai.from_pattern(BlockSparseMatrix(ctx, host), [[i + 1] if i + 1 < n else [] for i in range(n)])


def test_hierarchy_keeps_its_inputs_alive(ctx):
    # setup (multilevel.hpp:59) has value semantics: destroying the caller's A and
    # transfers (and, for create, the FSAI objects) afterwards must not affect cycles
    cfg = pr.CONFIGS["C2"].scaled(16, 3)
    A, T, b = pr.make_problem(cfg)
    ref = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                          default_params(t_max=1, coarse_dim_cap=1 << 30))
    x_ref = Vector(ctx, b.size)
    ref.v_cycle(3, 3, Vector(ctx, b), x_ref)
    dA = BlockSparseMatrix(ctx, A)
    dT = [BlockSparseMatrix(ctx, p) for p in T]
    h = Hierarchy.setup(dA, dT, default_params(t_max=1, coarse_dim_cap=1 << 30))
    dA.close()
    for p in dT:
        p.close()
    h._keep.clear()
    x = Vector(ctx, b.size)
    h.v_cycle(3, 3, Vector(ctx, b), x)
    assert np.array_equal(x.download(), x_ref.download())
    # create(): levels, transfers and preconditioners taken from another hierarchy
    L = ref.levels
    As, Ps, Ms = [], [None], [None]
    for l in range(L):
        a, p, m = ref.level(l)
        As.append(a)
        if l:
            Ps.append(p)
            Ms.append(m)
    betas = [0.0] + [ref.beta(l) for l in range(1, L)]
    hc = Hierarchy.create(ctx, As, Ps, Ms, betas)
    hc._keep.clear()
    x2 = Vector(ctx, b.size)
    hc.v_cycle(3, 3, Vector(ctx, b), x2)
    ref.close()  # the level objects hc points to belonged to ref
    x3 = Vector(ctx, b.size)
    hc.v_cycle(3, 3, Vector(ctx, b), x3)
    assert np.array_equal(x2.download(), x3.download())


@pytest.mark.parametrize("n,levels,kpre,kpost", [(32, 3, 3, 3), (16, 2, 2, 1), (32, 3, 0, 2), (64, 3, 1, 0)])
def test_vcycle_pinned_host_pipelined_equals_device(ctx, n, levels, kpre, kpost):
    """Pinned host buffers take the pipelined path (sliced upload overlapped with the
    first residual, copies inside the captured graph); kpre = 0 falls back."""
    import torch

    cfg = pr.CONFIGS["C2"].scaled(n, levels)
    A, T, b = pr.make_problem(cfg)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, coarse_dim_cap=1 << 30))
    x0 = pr.normal_vector(b.size, 0, 9)
    hb = torch.from_numpy(b.copy()).pin_memory()
    hx = torch.from_numpy(x0.copy()).pin_memory()
    xv, bv = Vector(ctx, x0), Vector(ctx, b)
    for _ in range(3):
        dh.v_cycle_host_ptr(kpre, kpost, hb.data_ptr(), hx.data_ptr())
        dh.v_cycle(kpre, kpost, bv, xv)
        assert np.array_equal(hx.numpy(), xv.download())
    # the caller's b is untouched
    assert np.array_equal(hb.numpy(), b)


def test_solve_stopping_edge_cases_match_oracle(ctx):
    """tol above 1 (converged before any cycle), zero right-hand side (zero residual),
    max_iter 0: iteration counts, status and histories as the oracle's loop."""
    A, T, b, oh, dh = _small_hierarchies(ctx, 16, 2)
    for bb, tol, mi in ((b, 2.0, 10), (np.zeros_like(b), 1e-8, 10), (b, 1e-8, 0)):
        hist_o, it_o, st_o, _ = oh.solve(3, 3, bb, np.zeros_like(bb), tol, mi)
        hist_g, it_g, st_g = dh.solve(3, 3, Vector(ctx, bb), Vector(ctx, np.zeros_like(bb)), tol, mi)
        assert (it_g, st_g) == (it_o, st_o), (tol, mi, it_g, st_g, it_o, st_o)
        assert np.allclose(hist_g, hist_o, rtol=1e-12, atol=0.0)


@pytest.mark.parametrize("tol,max_iter", [(1e-8, 25), (1e-2, 200), (1e-30, 0), (5.0, 10)])
def test_graph_solve_loop_equals_eager_loop(ctx, tol, max_iter):
    """bmg_solve with one graph launch per iteration (cycle, residual, segment sums
    to pinned memory) against the eager loop (use_graph off): bitwise histories and
    iterates, iteration counts and status as the oracle's."""
    A, T, b, oh, dh = _small_hierarchies(ctx, 32, 3)
    out = []
    for graph in (False, True, True):  # eager loop, graph loop, graph loop from its cache
        dh.use_graph(graph)
        x = Vector(ctx, np.zeros_like(b))
        hist, it, st = dh.solve(3, 3, Vector(ctx, b), x, tol, max_iter)
        out.append((hist.copy(), it, st, x.download()))
    dh.use_graph(True)
    for o in out[1:]:
        assert o[1:3] == out[0][1:3]
        assert np.array_equal(o[0], out[0][0]) and np.array_equal(o[3], out[0][3])
    hist_o, it_o, st_o, _ = oh.solve(3, 3, b, np.zeros_like(b), tol, max_iter)
    assert (out[1][1], out[1][2]) == (it_o, st_o)


@pytest.mark.parametrize("m", [3, 6])
def test_small_uniform_blocks_stream_and_match_oracle(ctx, m):
    """Uniform linear / quadratic PUM-size blocks (m = 3, 6) on the streaming kernel:
    setup, cycles (graph), batched cycles and the solve loop against the oracle."""
    import dataclasses

    cfg = dataclasses.replace(pr.CONFIGS["C2"].scaled(32, 3), m=m)
    A, T, b = pr.make_problem(cfg)
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, coarse_dim_cap=1 << 30, probe=False)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, coarse_dim_cap=1 << 30))
    for l in range(1, dh.levels):
        assert abs(dh.beta(l) - oh.beta(l)) <= 1e-10 * oh.beta(l)
    hist_o, it_o, st_o, x_o = oh.solve(3, 3, b, np.zeros_like(b), 1e-8, 20)
    xv = Vector(ctx, np.zeros_like(b))
    hist_g, it_g, st_g = dh.solve(3, 3, Vector(ctx, b), xv, 1e-8, 20)
    assert (it_g, st_g) == (it_o, st_o)
    rho_o, rho_g = hist_o / hist_o[0], hist_g / hist_g[0]
    assert np.all(np.abs(rho_g - rho_o) <= 1e-10)
    # K = 4 batched cycle, each RHS bitwise the single cycle
    K = 4
    B = np.stack([np.roll(b, 5 * v) for v in range(K)], axis=1).ravel().copy()
    xb = Vector(ctx, B.size)
    dh.v_cycle_batch(3, 3, K, Vector(ctx, B), xb)
    xbk = xb.download().reshape(-1, K)
    for v in range(K):
        xs = Vector(ctx, b.size)
        dh.v_cycle(3, 3, Vector(ctx, np.ascontiguousarray(B.reshape(-1, K)[:, v])), xs)
        assert np.array_equal(xbk[:, v], xs.download())
