"""The reference's multilevel test cases on its own test problem
(proj/tests/test_multilevel.cpp:20-186 with fd_biharmonic, experiments.cpp:104-195),
run through the device hierarchy: scalar blocks (m = 1, the generic variable-layout
kernels), bilinear transfers, plus parity with the oracle on the same inputs.

Tolerances are the reference's own (written per test); oracle parity: betas
1e-10 relative, cycle iterates 1e-11 relative."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy, Vector, default_params
from paper_2509_06744_b200 import problems as pr

pytestmark = pytest.mark.gpu


def _fd_hier(ctx, n_grid, levels, t_max):
    # test_multilevel.cpp:20-23
    fd = pr.fd_biharmonic(n_grid, levels)
    dA = BlockSparseMatrix(ctx, fd.A)
    h = Hierarchy.setup(dA, [BlockSparseMatrix(ctx, p) for p in fd.transfers], default_params(t_max=t_max))
    return fd, h, dA


def _energy(A, e):
    return float(e @ (A @ e))


def test_one_level_fd_solves_directly(ctx):
    # test_multilevel.cpp:99-106
    fd = pr.fd_biharmonic(8, 1)
    assert fd.transfers == []
    h = Hierarchy.setup(BlockSparseMatrix(ctx, fd.A), [], default_params())
    x = Vector(ctx, fd.b.size)
    h.v_cycle(2, 2, Vector(ctx, fd.b), x)
    assert np.linalg.norm(x.download() - fd.reference) <= 1e-9 * np.linalg.norm(fd.reference)


def test_fd_fixed_point_and_linearity(ctx, rng):
    # test_multilevel.cpp:108-127
    fd, h, _ = _fd_hier(ctx, 16, 2, 3)
    n = fd.A.dim_r
    x = Vector(ctx, n)
    h.v_cycle(2, 2, Vector(ctx, np.zeros(n)), x)
    assert np.linalg.norm(x.download()) == 0.0
    b1, b2 = rng.standard_normal(n), rng.standard_normal(n)
    outs = []
    for rhs in (b1, b2, 0.5 * b1 - 2.0 * b2):
        xv = Vector(ctx, n)
        h.v_cycle(2, 2, Vector(ctx, rhs), xv)
        outs.append(xv.download())
    xa, xb, xc = outs
    assert np.linalg.norm(xc - (0.5 * xa - 2.0 * xb)) <= 1e-12 * (1.0 + np.linalg.norm(xc))


def test_fd_error_contraction(ctx, rng):
    # test_multilevel.cpp:129-149: V(4,4) on the homogeneous problem, t_max = 4
    fd, h, _ = _fd_hier(ctx, 32, 3, 4)
    A = fd.A.to_dense()
    n = fd.A.dim_r
    e = rng.standard_normal(n)
    ev, zero = Vector(ctx, e), Vector(ctx, np.zeros(n))
    prev = np.sqrt(_energy(A, e))
    rho_max = 0.0
    for _ in range(6):
        h.v_cycle(4, 4, zero, ev)
        cur = np.sqrt(max(_energy(A, ev.download()), 0.0))
        rho_max = max(rho_max, cur / prev)
        prev = cur
    assert rho_max < 1.0


def test_fd_cycle_operator_is_A_self_adjoint(ctx, rng):
    # test_multilevel.cpp:151-171
    fd, h, _ = _fd_hier(ctx, 16, 2, 2)
    A = fd.A.to_dense()
    n = fd.A.dim_r
    e1, e2 = rng.standard_normal(n), rng.standard_normal(n)

    def cycle_err(e):
        ev = Vector(ctx, e.copy())
        h.v_cycle(3, 3, Vector(ctx, np.zeros(n)), ev)
        return ev.download()

    ce1, ce2 = cycle_err(e1), cycle_err(e2)
    lhs, rhs = (A @ ce1) @ e2, (A @ ce2) @ e1
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), 1.0)


def test_fd_setup_deterministic_and_levels_spd(ctx):
    # test_multilevel.cpp:173-186
    fd, h1, _ = _fd_hier(ctx, 16, 3, 3)
    _, h2, _ = _fd_hier(ctx, 16, 3, 3)
    for l in range(h1.levels):
        if l > 0:
            assert h1.beta(l) == h2.beta(l)
        a1, a2 = h1.level(l)[0], h2.level(l)[0]
        n_l = (16 >> (h1.levels - 1 - l)) - 1
        ones = np.ones(n_l * n_l, np.int32)
        d1 = a1.download(ones, ones, symmetric=True)
        d2 = a2.download(ones, ones, symmetric=True)
        assert np.array_equal(d1.vals, d2.vals) and np.array_equal(d1.col_idx, d2.col_idx)
        assert np.linalg.eigvalsh(d1.to_dense()).min() > 0.0


@pytest.mark.parametrize("n_grid,levels,t_max", [(16, 3, 1), (32, 3, 2), (32, 4, 3)])
def test_fd_hierarchy_matches_oracle(ctx, n_grid, levels, t_max):
    fd = pr.fd_biharmonic(n_grid, levels)
    oh = O.Hierarchy(O.Mat(fd.A), [O.Mat(p) for p in fd.transfers], t_max=t_max, probe=False)
    dA = BlockSparseMatrix(ctx, fd.A)
    dh = Hierarchy.setup(dA, [BlockSparseMatrix(ctx, p) for p in fd.transfers], default_params(t_max=t_max))
    for l in range(1, dh.levels):
        assert abs(dh.beta(l) - oh.beta(l)) <= 1e-10 * oh.beta(l)
    x_o = np.zeros_like(fd.b)
    xv, bv = Vector(ctx, x_o), Vector(ctx, fd.b)
    for _ in range(4):
        x_o = oh.v_cycle(3, 3, fd.b, x_o)
        dh.v_cycle(3, 3, bv, xv)
        assert np.linalg.norm(xv.download() - x_o) <= 1e-11 * np.linalg.norm(x_o)
    # the cycle converges to the manufactured field
    hist, it, st = dh.solve(3, 3, bv, Vector(ctx, np.zeros_like(fd.b)), 1e-10, 60)
    assert st == 0 and hist[-1] <= 1e-10 * hist[0]


@pytest.mark.parametrize("k", [1, 3])
def test_fd_measure_rates_matches_oracle(ctx, k):
    # the reference CLI's `--problem fd` run (blockmg_cli.cpp:108-116): rates of
    # the V(k,k) cycle on fd_biharmonic(2^hi, hi - lo + 1) against its
    # manufactured field, in the mass (h^2 I), energy and residual norms
    fd = pr.fd_biharmonic(32, 4)
    oh = O.Hierarchy(O.Mat(fd.A), [O.Mat(p) for p in fd.transfers], t_max=2, probe=False)
    want = oh.measure_rates(O.Mat(fd.mass), fd.b, fd.reference, k, k, seed=5, tol=1e-8, max_iter=40)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, fd.A), [BlockSparseMatrix(ctx, p) for p in fd.transfers],
                         default_params(t_max=2))
    got = dh.measure_rates(BlockSparseMatrix(ctx, fd.mass), Vector(ctx, fd.b), Vector(ctx, fd.reference), k, k,
                           seed=5, tol=1e-8, max_iter=40)
    assert got["iterations"] == want["iterations"] and got["status"] == want["status"]
    # e = x - u is measured against an exact field (b = A u): rounding-level
    # differences of the iterates (~eps |u| per cycle) are relative differences
    # of ~eps |u| / |e| in the tail, so the histories are compared in units of
    # the field's own norm, and the rates (|e_it| / |e_0|)^(1/it) within
    # delta / (it |e_it|), delta = 1e-12 |u| (it + 1)
    A = fd.A.to_dense()
    it = got["iterations"]
    scales = {"l2_sq": np.sqrt(fd.reference @ (fd.mass.to_dense() @ fd.reference)),
              "energy_sq": np.sqrt(fd.reference @ (A @ fd.reference)), "residual": np.linalg.norm(fd.b)}
    for key, rate in (("l2_sq", "rho_l2"), ("energy_sq", "rho_a"), ("residual", "rho_r")):
        g, w = got[key], want[key]
        if key != "residual":
            g, w = np.sqrt(g), np.sqrt(w)
        delta = 1e-12 * scales[key] * (np.arange(g.size) + 1)
        assert np.all(np.abs(g - w) <= delta), key
        assert abs(got[rate] - want[rate]) <= (delta[-1] / (it * w[-1]) + 1e-12) * want[rate], rate
    assert 0.0 < got["rho_a"] < 1.0
