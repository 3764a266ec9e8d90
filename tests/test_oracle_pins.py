"""Pins the CPU oracle against every known-answer and property test the reference
holds for the hot path (proj/tests/*.cpp).  The reference ships no golden
vectors and cannot be built here (Eigen3 absent), so these are the pins
(SURVEY.md §8c).  Each test cites the reference test it restates.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import problems as pr
from tests.helpers import from_dense_blocks, random_bsr, random_layout, random_spd


def scalar22():
    # test_fsai.cpp:22-28 / test_blockcore.cpp two_by_two_scalar: [[4,1],[1,3]]
    return from_dense_blocks(np.array([1, 1], np.int32), np.array([1, 1], np.int32),
                             {(0, 0): [[4.0]], (1, 1): [[3.0]], (1, 0): [[1.0]], (0, 1): [[1.0]]}, symmetric=True)


def dense(m):
    return m.export().to_dense() if isinstance(m, O.Mat) else m.to_dense()


# ---------------------------------------------------------------- blockcore
def test_spmv_and_transpose_match_dense(rng):
    # test_blockcore.cpp:55-85 (1e-14)
    for rep in range(20):
        rs, cs = random_layout(rng, 8, 4), random_layout(rng, 8, 4)
        h = random_bsr(rng, rs, cs, 0.5)
        d = h.to_dense()
        m = O.Mat(h)
        x = rng.uniform(-1, 1, h.dim_c)
        y = rng.uniform(-1, 1, h.dim_r)
        assert np.linalg.norm(m.spmv(x) - d @ x) <= 1e-14 * (1 + np.linalg.norm(d @ x))
        assert np.linalg.norm(m.spmv_t(y) - d.T @ y) <= 1e-14 * (1 + np.linalg.norm(d.T @ y))


def test_multiply_matches_dense(rng):
    # test_blockcore.cpp:230-249
    for rep in range(10):
        a_l, b_l, c_l = random_layout(rng, 5, 3), random_layout(rng, 5, 3), random_layout(rng, 5, 3)
        a = random_bsr(rng, a_l, b_l, 0.6)
        b = random_bsr(rng, b_l, c_l, 0.6)
        c = O.multiply(O.Mat(a), O.Mat(b))
        want = a.to_dense() @ b.to_dense()
        assert np.linalg.norm(dense(c) - want) <= 1e-13 * (1 + np.linalg.norm(want))


def test_triple_product_identity_and_hand_case(rng):
    # test_blockcore.cpp:87-102: I A I^T = A; F = [[1,0],[-1/4,1]] on [[4,1],[1,3]]
    sizes = np.array([2, 3], np.int32)
    a = random_spd(rng, sizes, 1.0)
    eye = from_dense_blocks(sizes, sizes, {(0, 0): np.eye(2), (1, 1): np.eye(3)})
    c = O.triple_product(O.Mat(eye), O.Mat(a))
    assert np.linalg.norm(dense(c) - a.to_dense()) <= 1e-15
    f = from_dense_blocks(np.array([1, 1], np.int32), np.array([1, 1], np.int32),
                          {(0, 0): [[1.0]], (1, 1): [[1.0]], (1, 0): [[-0.25]]})
    p = O.triple_product(O.Mat(f), O.Mat(scalar22())).export()
    d = p.to_dense()
    assert d[0, 0] == pytest.approx(4.0, rel=1e-15)
    assert d[1, 1] == pytest.approx(11.0 / 4.0, rel=1e-15)
    assert p.nnzb == 2  # the exactly-zero (1,0) block is dropped


def test_triple_product_random(rng):
    # test_blockcore.cpp:104-122
    for rep in range(10):
        sizes = random_layout(rng, 6, 4)
        a = random_spd(rng, sizes, 0.6)
        blocks = {}
        for i in range(len(sizes)):
            blocks[(i, i)] = np.eye(sizes[i])
            for j in range(i):
                if rng.uniform() < 0.4:
                    blocks[(i, j)] = rng.uniform(-1, 1, (sizes[i], sizes[j]))
        f = from_dense_blocks(sizes, sizes, blocks)
        c = dense(O.triple_product(O.Mat(f), O.Mat(a)))
        fd, ad = f.to_dense(), a.to_dense()
        want = fd @ ad @ fd.T
        assert np.linalg.norm(c - want) <= 1e-13 * np.linalg.norm(want)
        assert np.array_equal(c, c.T)


def test_small_cholesky_hand_case_and_pivot():
    # test_blockcore.cpp:124-159
    l, ld = O.cholesky(np.eye(3))
    assert np.array_equal(l, np.eye(3)) and ld == 0.0
    b = np.array([[4.0, 2.0], [2.0, 5.0]])
    l, ld = O.cholesky(b)
    assert np.linalg.norm(l - np.array([[2.0, 0.0], [1.0, 2.0]])) <= 1e-15
    with pytest.raises(O.OracleError) as ei:
        O.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert ei.value.pivot == 1


def test_small_cholesky_random(rng):
    # test_blockcore.cpp:161-173 (logdet 1e-9)
    for rep in range(25):
        n = 1 + int(rng.integers(8))
        r = rng.uniform(-1, 1, (n, n))
        b = r @ r.T + n * np.eye(n)
        l, ld = O.cholesky(b)
        assert np.linalg.norm(l @ l.T - b) <= 1e-12 * np.linalg.norm(b)
        assert ld == pytest.approx(np.log(np.linalg.det(b)), rel=1e-9)


# ---------------------------------------------------------------- FSAI
def test_fsai_diagonal_pattern_is_block_jacobi(rng):
    # test_fsai.cpp:57-69
    sizes = np.array([2, 3, 1, 2], np.int32)
    a = random_spd(rng, sizes, 0.7)
    f = O.Fsai(O.Mat(a), O.Fsai.DIAGONAL)
    assert np.array_equal(dense(f.factor(0)), np.eye(a.dim_r))
    shat = f.shat()
    off = 0
    for i, m in enumerate(sizes):
        l = shat[off:off + m * m].reshape(m, m)
        blk = a.to_dense()[sum(sizes[:i]):sum(sizes[:i]) + m, sum(sizes[:i]):sum(sizes[:i]) + m]
        assert np.linalg.norm(l @ l.T - blk) <= 1e-13 * np.linalg.norm(blk)
        off += m * m


def test_fsai_scalar_2x2_hand_case():
    # test_fsai.cpp:71-77: F21 = -1/4, S = diag(4, 11/4)
    f = O.Fsai(O.Mat(scalar22()), O.Fsai.FULL)
    fd = dense(f.factor(0))
    assert fd[1, 0] == pytest.approx(-0.25, rel=1e-15)
    s = f.shat()
    assert s[0] ** 2 == pytest.approx(4.0, rel=1e-15)
    assert s[1] ** 2 == pytest.approx(11.0 / 4.0, rel=1e-14)


def test_fsai_full_pattern_is_exact_inverse(rng):
    # test_fsai.cpp:79-92
    for rep in range(5):
        sizes = random_layout(rng, 10, 3)
        a = random_spd(rng, sizes, 1.0)
        f = O.Fsai(O.Mat(a), O.Fsai.FULL)
        r = rng.uniform(-1, 1, a.dim_r)
        want = np.linalg.solve(a.to_dense(), r)
        assert np.linalg.norm(f.apply(r) - want) <= 1e-9 * np.linalg.norm(want)
        n = a.dim_r
        g = np.column_stack([f.apply_transformed(O.Mat(a), e) for e in np.eye(n)])
        assert np.linalg.norm(g - np.eye(n)) <= 1e-10


def test_fsai_apply_symmetric_positive(rng):
    # test_fsai.cpp:94-115
    sizes = np.array([2, 2, 3], np.int32)
    a = random_spd(rng, sizes, 0.8)
    pattern = [[j for j in range(i) if rng.uniform() < 0.8] for i in range(3)]
    f = O.fsai_with_pattern(O.Mat(a), pattern)
    r1, r2 = rng.uniform(-1, 1, a.dim_r), rng.uniform(-1, 1, a.dim_r)
    assert f.apply(r1) @ r2 == pytest.approx(r1 @ f.apply(r2), rel=1e-13)
    assert f.apply(r1) @ r1 > 0


def test_fsai_lemma_diag_fa_equals_s(rng):
    # test_fsai.cpp:117-137 (Lemma 2.4): diag(F A) = S = diag(F A F^T), (F A)_kj = 0 on the pattern
    for rep in range(10):
        sizes = random_layout(rng, 8, 4)
        a = random_spd(rng, sizes, 0.8)
        n = len(sizes)
        pattern = [[j for j in range(i) if rng.uniform() < 0.6] for i in range(n)]
        f = O.fsai_with_pattern(O.Mat(a), pattern)
        F = dense(f.factor(0))
        A = a.to_dense()
        H = F @ A
        FAF = F @ A @ F.T
        offs = np.concatenate([[0], np.cumsum(sizes)])
        shat = f.shat()
        so = 0
        for k in range(n):
            m = sizes[k]
            l = shat[so:so + m * m].reshape(m, m)
            so += m * m
            s = l @ l.T
            sl = slice(offs[k], offs[k + 1])
            assert np.linalg.norm(H[sl, sl] - s) <= 1e-12 * np.linalg.norm(s)
            assert np.linalg.norm(FAF[sl, sl] - s) <= 1e-12 * np.linalg.norm(s)
            for j in pattern[k]:
                assert np.linalg.norm(H[sl, offs[j]:offs[j + 1]]) <= 1e-10 * np.linalg.norm(A[sl, sl])


def test_delta_ratio_zero_block_and_brute_force(rng):
    # test_fsai.cpp:139-185
    z = from_dense_blocks(np.array([1, 1], np.int32), np.array([1, 1], np.int32),
                          {(0, 0): [[2.0]], (1, 1): [[5.0]], (1, 0): [[0.0]], (0, 1): [[0.0]]}, symmetric=True)
    assert O.delta_ratio(O.Mat(z), [[], []], 1, 0) == pytest.approx(1.0, rel=1e-15)
    for rep in range(6):
        sizes = random_layout(rng, 6, 3)
        n = len(sizes)
        a = random_spd(rng, sizes, 0.9)
        am = O.Mat(a)
        pattern = [[j for j in range(i) if rng.uniform() < 0.3] for i in range(n)]
        offs = np.concatenate([[0], np.cumsum(sizes)])
        A = a.to_dense()
        for k in range(1, n):
            for c in range(k):
                if c in pattern[k]:
                    continue
                F = dense(O.fsai_with_pattern(am, pattern).factor(0))
                F_H = F @ A
                if np.linalg.norm(F_H[offs[k]:offs[k + 1], offs[c]:offs[c + 1]]) == 0.0:
                    continue
                try:
                    got = O.delta_ratio(am, pattern, k, c)
                except O.OracleError:
                    continue
                pc = [list(p) for p in pattern]
                pc[k] = sorted(pc[k] + [c])
                Fc = dense(O.fsai_with_pattern(am, pc).factor(0))
                sl = slice(offs[k], offs[k + 1])
                det = np.linalg.det((F @ A @ F.T)[sl, sl])
                det_c = np.linalg.det((Fc @ A @ Fc.T)[sl, sl])
                assert 0 < got <= 1
                assert got == pytest.approx(det_c / det, rel=1e-10)


def test_adaptive_block_diagonal_input_stays_jacobi(rng):
    # test_fsai.cpp:187-199
    sizes = np.array([2, 3, 2], np.int32)
    blocks = {}
    for i in range(3):
        r = rng.uniform(-1, 1, (sizes[i], sizes[i]))
        blocks[(i, i)] = r @ r.T + 2 * np.eye(sizes[i])
    a = from_dense_blocks(sizes, sizes, blocks, symmetric=True)
    f = O.Fsai(O.Mat(a), O.Fsai.NESTED, t_max=3)
    assert np.array_equal(dense(f.factor(0)), np.eye(a.dim_r))


def test_adaptive_exhausts_to_exact_inverse(rng):
    # test_fsai.cpp:201-209
    n = 6
    a = random_spd(rng, np.ones(n, np.int32), 1.0)
    f = O.Fsai(O.Mat(a), O.Fsai.NESTED, t_max=n - 1)
    assert f.factor(0).info()["nnzb"] == n * (n + 1) // 2
    g = np.column_stack([f.apply_transformed(O.Mat(a), e) for e in np.eye(n)])
    assert np.linalg.norm(g - np.eye(n)) <= 1e-10


def test_nested_level1_equals_dense_composition(rng):
    # test_fsai.cpp:226-257
    sizes = random_layout(rng, 6, 3)
    a = random_spd(rng, sizes, 0.8)
    f = O.Fsai(O.Mat(a), O.Fsai.NESTED, t_max=2, nest=1)
    assert f.chain_len() == 2
    f0, f1 = dense(f.factor(0)), dense(f.factor(1))
    shat = f.shat()
    S = np.zeros((a.dim_r, a.dim_r))
    o = so = 0
    for m in sizes:
        l = shat[so:so + m * m].reshape(m, m)
        S[o:o + m, o:o + m] = l @ l.T
        o += m
        so += m * m
    M = f0.T @ f1.T @ np.linalg.inv(S) @ f1 @ f0
    r = rng.uniform(-1, 1, a.dim_r)
    assert np.linalg.norm(f.apply(r) - M @ r) <= 1e-12 * np.linalg.norm(M @ r)


# ---------------------------------------------------------------- Chebyshev
def test_fourth_kind_values_at_one():
    # test_chebyshev.cpp:22-27
    for k in range(7):
        assert O.poly_eval(O.FOURTH_W, k, 1.0) == pytest.approx(2 * k + 1, rel=1e-14)


def test_scaled_fourth_degree_one_closed_form(rng):
    # test_chebyshev.cpp:29-41
    beta = 3.7
    assert O.poly_eval(O.SCALED_FOURTH, 1, 0.0, beta=beta) == pytest.approx(1.0, rel=1e-15)
    for z in beta * rng.uniform(size=50):
        assert O.poly_eval(O.SCALED_FOURTH, 1, z, beta=beta) == pytest.approx(1 - 4 / (3 * beta) * z, rel=1e-14, abs=1e-15)
    for k in range(1, 11):
        assert O.poly_eval(O.SCALED_FOURTH, k, 0.0, beta=beta) == pytest.approx(1.0, rel=1e-13)


def test_fourth_kind_degree_one_closed_form():
    # test_chebyshev.cpp:83-89: W-hat_1(1) = -1/3
    e = np.array([1.0, -2.0, 1.0, 1.0])
    x = O.smoother_apply_diag(np.ones(4), O.CHEB_FOURTH, np.zeros(4), e, 1, beta=1.0)
    assert np.linalg.norm(x + e / 3.0) <= 1e-15


def test_fourth_kind_per_mode_error(rng):
    # test_chebyshev.cpp:91-106 (1e-12)
    n = 12
    lam = 0.05 + 2.0 * rng.uniform(size=n)
    beta = lam.max()
    for k in range(1, 11):
        e0 = rng.uniform(-1, 1, n)
        x = O.smoother_apply_diag(lam, O.CHEB_FOURTH, np.zeros(n), e0, k, beta=beta)
        want = np.array([O.poly_eval(O.SCALED_FOURTH, k, l, beta=beta) for l in lam]) * e0
        assert np.allclose(x, want, rtol=1e-12, atol=1e-15)


def test_mu_closed_form_exact():
    # test_chebyshev.cpp:108-110
    for n in range(21):
        assert O.lib().orc_fourth_kind_mu(n) == (2.0 * n + 1.0) / (2.0 * n + 3.0)


def test_first_kind_and_richardson(rng):
    # test_chebyshev.cpp:112-167
    n = 6
    lam = 1.0 + rng.uniform(size=n)
    b, x0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    x = O.smoother_apply_diag(lam, O.CHEB_FIRST, b, x0, 1, alpha=1.0, beta=2.0)
    want = x0 + 2.0 / 3.0 * (b - lam * x0)
    assert np.linalg.norm(x - want) <= 1e-14 * np.linalg.norm(want)
    lam = 0.1 + rng.uniform(size=8)
    sol = rng.uniform(-1, 1, 8)
    fixed = O.smoother_apply_diag(lam, O.RICHARDSON, lam * sol, sol, 3, omega=1.0)
    assert np.linalg.norm(fixed - sol) <= 1e-14 * np.linalg.norm(sol)
    x0 = rng.uniform(-1, 1, 8)
    for k in range(1, 6):
        xk = O.smoother_apply_diag(lam, O.RICHARDSON, np.zeros(8), x0, k, omega=0.7)
        assert np.allclose(xk, (1 - 0.7 * lam) ** k * x0, rtol=1e-12, atol=1e-15)


def test_weighted_minimax_and_smoothing_bound(rng):
    # test_chebyshev.cpp:169-198
    beta = 2.3
    z = beta * np.linspace(0, 1, 20001)
    for k in range(1, 9):
        vals = np.array([O.poly_eval(O.SCALED_FOURTH, k, t, beta=beta) for t in z])
        assert np.max(np.sqrt(z) * np.abs(vals)) == pytest.approx(np.sqrt(beta) / (2 * k + 1), rel=1e-3)
    lam = 2.5 * rng.uniform(size=30)
    beta = lam.max()
    for k in range(1, 7):
        bound = max(l * abs(O.poly_eval(O.SCALED_FOURTH, k, l, beta=beta)) for l in lam)
        v = rng.uniform(-1, 1, 30)
        e = O.smoother_apply_diag(lam, O.CHEB_FOURTH, np.zeros(30), v, k, beta=beta)
        assert np.linalg.norm(lam * e) <= bound * np.linalg.norm(v) * (1 + 1e-12)


def test_fourth_kind_linear_and_validates(rng):
    # test_chebyshev.cpp:200-229
    n = 9
    lam = 0.2 + rng.uniform(size=n)
    beta = lam.max() * 1.05
    b1, b2, x1, x2 = (rng.uniform(-1, 1, n) for _ in range(4))
    for k in range(1, 6):
        lhs = O.smoother_apply_diag(lam, O.CHEB_FOURTH, 0.7 * b1 - 1.3 * b2, 0.7 * x1 - 1.3 * x2, k, beta=beta)
        rhs = 0.7 * O.smoother_apply_diag(lam, O.CHEB_FOURTH, b1, x1, k, beta=beta) \
            - 1.3 * O.smoother_apply_diag(lam, O.CHEB_FOURTH, b2, x2, k, beta=beta)
        assert np.linalg.norm(lhs - rhs) <= 1e-13 * (1 + np.linalg.norm(rhs))
    with pytest.raises(O.OracleError):
        O.smoother_apply_diag(np.ones(2), O.CHEB_FOURTH, np.zeros(2), np.zeros(2), 2, beta=-1.0)
    with pytest.raises(O.OracleError):
        O.smoother_apply_diag(np.ones(2), O.RICHARDSON, np.zeros(2), np.zeros(2), 0)


# ---------------------------------------------------------------- multilevel / Lanczos
def test_lanczos_known_spectra(rng):
    # test_multilevel.cpp:60-83
    raw = O.lanczos_diag(np.arange(1.0, 51.0), 100, 1.0, 42)
    assert 49.5 <= raw <= 50.0 + 1e-10
    assert O.lanczos_diag(np.arange(1.0, 51.0), 100, 1.01, 42) >= 50.0
    assert O.lanczos_diag(np.full(20, 7.5), 100, 1.0, 1) == pytest.approx(7.5, rel=1e-12)
    sizes = random_layout(rng, 8, 3)
    a = random_spd(rng, sizes, 1.0)
    f = O.Fsai(O.Mat(a), O.Fsai.FULL)
    assert O.lanczos_lambda_max(O.Mat(a), f, 100, 1.0, 42) == pytest.approx(1.0, rel=1e-9)


def test_lanczos_bound_dominates_dense_spectrum(rng):
    # test_multilevel.cpp:85-97
    for rep in range(5):
        sizes = random_layout(rng, 8, 4)
        a = random_spd(rng, sizes, 0.6)
        am = O.Mat(a)
        f = O.Fsai(am, O.Fsai.NESTED, t_max=2)
        beta = O.lanczos_lambda_max(am, f, 100, 1.01, 42)
        n = a.dim_r
        g = np.column_stack([f.apply_transformed(am, e) for e in np.eye(n)])
        assert beta >= 0.99 * np.linalg.eigvalsh(0.5 * (g + g.T)).max()


def test_tridiagonal_eigs_match_numpy(rng):
    for n in (1, 2, 5, 40, 100):
        d, e = rng.standard_normal(n), rng.standard_normal(max(n - 1, 0))
        T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        assert np.allclose(O.tridiag_eigs(d, e), np.linalg.eigvalsh(T), rtol=1e-12, atol=1e-12)


def test_galerkin_identities(rng):
    # test_multilevel.cpp:27-58
    sizes = np.array([2, 1, 3], np.int32)
    a = random_spd(rng, sizes, 0.8)
    eye = from_dense_blocks(sizes, sizes, {(i, i): np.eye(s) for i, s in enumerate(sizes)})
    assert np.linalg.norm(dense(O.galerkin(O.Mat(a), O.Mat(eye))) - a.to_dense()) <= 1e-15
    p = from_dense_blocks(np.array([1, 1], np.int32), np.array([1], np.int32), {(0, 0): [[1.0]], (1, 0): [[1.0]]})
    i2 = from_dense_blocks(np.array([1, 1], np.int32), np.array([1, 1], np.int32),
                           {(0, 0): [[1.0]], (1, 1): [[1.0]]}, symmetric=True)
    assert dense(O.galerkin(O.Mat(i2), O.Mat(p)))[0, 0] == pytest.approx(2.0, rel=1e-15)
    for rep in range(10):
        fine, coarse = random_layout(rng, 6, 3), random_layout(rng, 3, 3)
        pr_ = random_bsr(rng, fine, coarse, 0.6)
        af = random_spd(rng, fine, 0.7)
        c = dense(O.galerkin(O.Mat(af), O.Mat(pr_)))
        want = pr_.to_dense().T @ af.to_dense() @ pr_.to_dense()
        assert np.linalg.norm(c - want) <= 1e-13 * (1 + np.linalg.norm(want))
        assert np.array_equal(c, c.T)


def _hier(n=16, levels=2, t_max=1):
    cfg = pr.CONFIGS["C2"].scaled(n, levels)
    A, T, b = pr.make_problem(cfg)
    return A, T, b, O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=t_max, coarse_dim_cap=1 << 30)


def test_vcycle_fixed_point_linearity_self_adjoint(rng):
    # test_multilevel.cpp:108-127, 151-171
    A, T, b, h = _hier()
    n = A.dim_r
    assert np.linalg.norm(h.v_cycle(2, 2, np.zeros(n), np.zeros(n))) == 0.0
    b1, b2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    xa, xb = h.v_cycle(2, 2, b1, np.zeros(n)), h.v_cycle(2, 2, b2, np.zeros(n))
    xc = h.v_cycle(2, 2, 0.5 * b1 - 2.0 * b2, np.zeros(n))
    assert np.linalg.norm(xc - (0.5 * xa - 2.0 * xb)) <= 1e-12 * (1 + np.linalg.norm(xc))
    am = O.Mat(A)
    e1, e2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    c1, c2 = h.v_cycle(3, 3, np.zeros(n), e1), h.v_cycle(3, 3, np.zeros(n), e2)
    lhs, rhs = am.spmv(c1) @ e2, am.spmv(c2) @ e1
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), 1.0)


def test_vcycle_contracts_and_setup_deterministic():
    # test_multilevel.cpp:129-149, 173-187
    A, T, b, h = _hier(16, 3)
    _, _, _, h2 = _hier(16, 3)
    for l in range(1, h.levels()):
        assert h.beta(l) == h2.beta(l)
    am = O.Mat(A)
    e = np.random.default_rng(213).uniform(-1, 1, A.dim_r)
    prev = np.sqrt(e @ am.spmv(e))
    for it in range(4):
        e = h.v_cycle(4, 4, np.zeros(A.dim_r), e)
        cur = np.sqrt(max(e @ am.spmv(e), 0.0))
        assert cur / prev < 1.0
        prev = cur


def test_one_level_direct_solve():
    # test_multilevel.cpp:99-106
    A = pr.stencil_matrix(2, 6, 2, 3)
    h = O.Hierarchy(O.Mat(A), [], t_max=1, coarse_dim_cap=1 << 30)
    b = pr.normal_vector(A.dim_r)
    x = h.v_cycle(2, 2, b, np.zeros_like(b), level=0)
    want = np.linalg.solve(A.to_dense(), b)
    assert np.linalg.norm(x - want) <= 1e-9 * np.linalg.norm(want)


def test_setup_cap_and_validation():
    # multilevel.cpp:68-70 (cap), multilevel.cpp:78-80 (cycle validation)
    A = pr.stencil_matrix(2, 6, 2, 3)
    with pytest.raises(O.OracleError):
        O.Hierarchy(O.Mat(A), [], t_max=1, coarse_dim_cap=10)
    h = O.Hierarchy(O.Mat(A), [], t_max=1, coarse_dim_cap=1 << 30)
    with pytest.raises(O.OracleError):
        h.v_cycle(0, 0, np.zeros(A.dim_r), np.zeros(A.dim_r))


def test_rng_counter_stream():
    # rng.hpp:12-36: uniform in (0,1), entry i depends only on (seed, i)
    lib = O.lib()
    u = [lib.orc_rng_uniform(42, i) for i in range(1000)]
    assert all(0.0 < v < 1.0 for v in u)
    assert lib.orc_rng_uniform(42, 17) == u[17]
    assert lib.orc_mix64(0) == 0


def test_measure_rates_semantics():
    # experiments.cpp:15-67: e normalised to unit M-norm (l2_sq[0] = 1), rates are
    # (q_n / q_0)^(1/2n) for the quadratic forms and (r_n / r_0)^(1/n) for the residual
    from paper_2509_06744_b200 import problems as pr
    cfg = pr.CONFIGS["C2"].scaled(8, 2)
    A, T, _ = pr.make_problem(cfg)
    u = pr.normal_vector(A.dim_r, 0, 7)
    om = O.Mat(A)
    b = om.spmv(u)
    oh = O.Hierarchy(om, [O.Mat(p) for p in T], t_max=1, coarse_dim_cap=1 << 30, probe=False)
    r = oh.measure_rates(om, b, u, 2, 2, seed=3, tol=1e-30, max_iter=4)
    assert abs(r["l2_sq"][0] - 1.0) < 1e-14
    assert r["l2_sq"][0] == r["energy_sq"][0]  # M = A here
    n = r["iterations"]
    assert n == 4 and r["status"] == 1 and r["blowup_iteration"] == -1
    assert abs(r["rho_l2"] - (r["l2_sq"][n] / r["l2_sq"][0]) ** (1 / (2 * n))) < 1e-15
    assert abs(r["rho_r"] - (r["residual"][n] / r["residual"][0]) ** (1 / n)) < 1e-15
    r0 = oh.measure_rates(om, b, u, 2, 2, seed=3, tol=2.0, max_iter=4)
    assert r0["iterations"] == 0 and r0["status"] == 0 and r0["rho_a"] == 0.0
