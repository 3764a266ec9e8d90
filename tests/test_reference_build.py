"""The oracle against THE REFERENCE ITSELF -- CPU only.

oracle/_ref/libblockmg_ref.so is the reference's own unmodified sources
(/root/reference/proj/src/*.cpp compiled where they lie, `make -C oracle ref`)
behind the same C API as the oracle (oracle/ref_driver.cpp, oracle/pyref.py).
Eigen3 is not installed, so they are built against oracle/eigen_shim, which fixes
the summation order inside a dense primitive (the order the oracle documents);
everything above the primitives is the reference's code.  Every comparison below
is BITWISE: it shows that the oracle restates the reference's algorithms exactly
-- block order of every accumulation, patterns, thresholds, recurrences, the
recursion -- on the BASELINE shapes and on the lower-level entry points.

The library is built in the container (where /root/reference exists) and travels
prebuilt; without it these tests skip.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from oracle import pyref as R
from paper_2509_06744_b200 import problems as pr
from tests.helpers import from_dense_blocks, random_bsr, random_layout, random_spd

pytestmark = pytest.mark.skipif(not R.available(), reason="reference build (oracle/_ref) unavailable")


@pytest.fixture(autouse=True, scope="module")
def _few_oracle_threads():
    """The cases are small: two OpenMP threads keep the oracle's barriers cheap on a
    loaded host (results do not depend on the thread count)."""
    n = O.get_threads()
    O.set_threads(2)
    yield
    O.set_threads(n)


def digest(m):
    e = m.export()
    d = hashlib.sha256()
    for a in (e.row_ptr, e.col_idx, e.vals):
        d.update(np.ascontiguousarray(a).tobytes())
    return d.hexdigest()


def test_library_is_the_reference_and_maps_no_oracle_code():
    assert R._xlib().orc_is_reference() == 1
    assert R.lib() is not O.lib()
    assert os.path.realpath(R.REF_LIB_PATH) != os.path.realpath(O.LIB_PATH)


# ------------------------------------------------------------------ kernels.cpp
def test_spmv_spmv_t_bitwise_variable_layouts(rng):
    for rep in range(20):
        rs, cs = random_layout(rng, 9, 5), random_layout(rng, 9, 5)
        h = random_bsr(rng, rs, cs, 0.5)
        x, y = rng.uniform(-1, 1, h.dim_c), rng.uniform(-1, 1, h.dim_r)
        assert np.array_equal(O.Mat(h).spmv(x), R.Mat(h).spmv(x))
        assert np.array_equal(O.Mat(h).spmv_t(y), R.Mat(h).spmv_t(y))


def test_products_bitwise(rng):
    for rep in range(8):
        al, bl, cl = random_layout(rng, 6, 4), random_layout(rng, 6, 4), random_layout(rng, 6, 4)
        a, b = random_bsr(rng, al, bl, 0.6), random_bsr(rng, bl, cl, 0.6)
        assert digest(O.multiply(O.Mat(a), O.Mat(b))) == digest(R.multiply(R.Mat(a), R.Mat(b)))
        p, q = random_bsr(rng, al, bl, 0.6), random_bsr(rng, al, cl, 0.6)
        assert digest(O.transpose_multiply(O.Mat(p), O.Mat(q))) == digest(R.transpose_multiply(R.Mat(p), R.Mat(q)))
        sizes = random_layout(rng, 6, 4)
        s = random_spd(rng, sizes, 0.6)
        blocks = {(i, i): np.eye(sizes[i]) for i in range(len(sizes))}
        for i in range(len(sizes)):
            for j in range(i):
                if rng.uniform() < 0.4:
                    blocks[(i, j)] = rng.uniform(-1, 1, (sizes[i], sizes[j]))
        f = from_dense_blocks(sizes, sizes, blocks)
        assert digest(O.triple_product(O.Mat(f), O.Mat(s))) == digest(R.triple_product(R.Mat(f), R.Mat(s)))
        pr_ = random_bsr(rng, sizes, random_layout(rng, 4, 3), 0.7)
        assert digest(O.galerkin(O.Mat(s), O.Mat(pr_))) == digest(R.galerkin(R.Mat(s), R.Mat(pr_)))


def test_small_cholesky_bitwise(rng):
    for n in (1, 3, 10, 21):
        q = rng.normal(size=(n, n))
        b = q @ q.T + n * np.eye(n)
        lo, ldo = O.cholesky(b)
        lr, ldr = R.cholesky(b)
        assert np.array_equal(lo, lr) and ldo == ldr
        rhs = rng.normal(size=n)
        x = R.chol_solve_spd(b, rhs)
        assert np.linalg.norm(b @ x - rhs) <= 1e-12 * np.linalg.norm(rhs)
    with pytest.raises(R.OracleError) as e:
        R.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.status == -3 and e.value.pivot == 1  # NotPositiveDefinite{pivot}


# --------------------------------------------------------------------- fsai.cpp
def _same_fsai(fo, fr):
    assert fo.chain_len() == fr.chain_len()
    for k in range(fo.chain_len()):
        assert digest(fo.factor(k)) == digest(fr.factor(k))
    assert np.array_equal(fo.shat(), fr.shat())
    assert digest(fo.G()) == digest(fr.G())


def test_fsai_builds_bitwise(rng):
    for rep in range(6):
        sizes = random_layout(rng, 8, 4)
        a = random_spd(rng, sizes, 0.5)
        ao, ar = O.Mat(a), R.Mat(a)
        for kind in (O.Fsai.STATIC, O.Fsai.DIAGONAL, O.Fsai.FULL):
            _same_fsai(O.Fsai(ao, kind), R.Fsai(ar, kind))
        for t_max, nest in ((1, 0), (3, 0), (2, 1), (1, 2)):
            fo, fr = O.Fsai(ao, O.Fsai.NESTED, t_max, 1.0, nest), R.Fsai(ar, R.Fsai.NESTED, t_max, 1.0, nest)
            _same_fsai(fo, fr)
            r = rng.normal(size=a.dim_r)
            assert np.array_equal(fo.apply(r), fr.apply(r))
            assert np.array_equal(fo.apply_transformed(ao, r), fr.apply_transformed(ar, r))
            assert O.lanczos_lambda_max(ao, fo, 30, 1.01, 42) == R.lanczos_lambda_max(ar, fr, 30, 1.01, 42)


def test_delta_ratio_bitwise(rng):
    sizes = random_layout(rng, 7, 3)
    a = random_spd(rng, sizes, 0.9)
    n = len(sizes)
    pat = [[] for _ in range(n)]
    pat[n - 1] = [0]
    ao, ar = O.Mat(a), R.Mat(a)
    checked = 0
    for k in range(2, n):
        for c in range(1 if k == n - 1 else 0, k):
            try:
                want = R.delta_ratio(ar, pat, k, c)
            except R.OracleError:
                with pytest.raises(O.OracleError):
                    O.delta_ratio(ao, pat, k, c)
                continue
            assert O.delta_ratio(ao, pat, k, c) == want
            checked += 1
    assert checked > 0


# ------------------------------------------------- chebyshev.hpp / lanczos.hpp
def test_smoothers_poly_lanczos_bitwise(rng):
    cfg = pr.CONFIGS["C1"].scaled(8, 1)
    host = pr.stencil_matrix(cfg.dim, cfg.n, cfg.power, cfg.m)
    ao, ar = O.Mat(host), R.Mat(host)
    fo, fr = O.Fsai(ao, O.Fsai.STATIC), R.Fsai(ar, R.Fsai.STATIC)
    beta = O.lanczos_lambda_max(ao, fo)
    assert beta == R.lanczos_lambda_max(ar, fr)
    b, x = rng.normal(size=host.dim_r), rng.normal(size=host.dim_r)
    for kind, kw in ((O.CHEB_FOURTH, dict(beta=beta)), (O.CHEB_FIRST, dict(alpha=beta / 30, beta=beta)),
                     (O.RICHARDSON, dict(omega=0.7))):
        for k in (1, 2, 3, 5):
            assert np.array_equal(O.smoother_apply(ao, fo, kind, b, x, k, **kw),
                                  R.smoother_apply(ar, fr, kind, b, x, k, **kw))
    lam = np.arange(1.0, 51.0)
    assert O.lanczos_diag(lam) == R.lanczos_diag(lam)
    assert O.lanczos_diag(lam, iters=30, smallest=True) == R.lanczos_diag(lam, iters=30, smallest=True)
    for kind in (O.FIRST_T, O.FOURTH_W, O.SCALED_FIRST, O.SCALED_FOURTH):
        for deg in range(6):
            for t in (0.0, 0.3, 1.7):
                assert O.poly_eval(kind, deg, t, 0.5, 2.0) == R.poly_eval(kind, deg, t, 0.5, 2.0)
    with pytest.raises(R.OracleError) as e:
        R.smoother_apply(ar, fr, R.CHEB_FOURTH, b, x, 0, beta=beta)
    assert e.value.status == -1  # std::invalid_argument, as the oracle


# ---------------------------------------------------------------- multilevel.cpp
SHAPES = [
    ("C2", (16, 3), dict(t_max=1), 3),            # m = 10, 13-pt
    ("C4", (8, 3), dict(t_max=1), 3),             # 3-D, m = 20, 25-pt
    ("C5", (32, 4), dict(t_max=1), 3),            # m = 15, 4 levels
    ("C3", (16, 3), dict(t_max=1, nest=1), 4),    # m = 21, 25-pt triharmonic, nested, V(4,4)
]


@pytest.mark.parametrize("name,scaled,kw,k", SHAPES, ids=[s[0] for s in SHAPES])
def test_setup_and_solve_bitwise_on_baseline_shapes(name, scaled, kw, k):
    """setup (multilevel.cpp:36-75) and the V-cycle (:77-103) inside the
    stop-on-tolerance loop: every Galerkin operator, FSAI factor, S-hat, beta_l,
    the coarse factor, the residual history and the iterate are bitwise equal."""
    cfg = pr.CONFIGS[name].scaled(*scaled)
    A, T, b = pr.make_problem(cfg)
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], coarse_dim_cap=1 << 30, probe=False, **kw)
    rh = R.Hierarchy(R.Mat(A), [R.Mat(p) for p in T], coarse_dim_cap=1 << 30, **kw)
    assert oh.levels() == rh.levels() == cfg.levels
    for l in range(oh.levels()):
        assert digest(oh.A(l)) == digest(rh.A(l)), f"A[{l}]"
        if l >= 1:
            _same_fsai(oh.fsai(l), rh.fsai(l))
            assert oh.beta(l) == rh.beta(l), f"beta[{l}]"
    ho, io, so, xo = oh.solve(k, k, b, np.zeros_like(b), tol=1e-8, max_iter=12)
    hr, ir, sr, xr = rh.solve(k, k, b, np.zeros_like(b), tol=1e-8, max_iter=12)
    assert (io, so) == (ir, sr)
    assert np.array_equal(ho, hr) and np.array_equal(xo, xr)
    # cycles started on every level, V(2k, 0)
    for l in range(oh.levels()):
        n = oh.A(l).info()["dim_r"]
        bl = np.cos(np.arange(n, dtype=np.float64))
        assert np.array_equal(oh.v_cycle(2 * k, 0, bl, np.zeros(n), level=l), rh.v_cycle(2 * k, 0, bl, np.zeros(n), level=l))


def test_setup_errors_match():
    cfg = pr.CONFIGS["C2"].scaled(8, 2)
    A, T, b = pr.make_problem(cfg)
    for mod in (O, R):
        with pytest.raises(mod.OracleError) as e:
            mod.Hierarchy(mod.Mat(A), [mod.Mat(p) for p in T], t_max=1, coarse_dim_cap=10)
        assert e.value.status == -1
        h = mod.Hierarchy(mod.Mat(A), [mod.Mat(p) for p in T], t_max=1, coarse_dim_cap=1 << 30)
        with pytest.raises(mod.OracleError) as e:
            h.v_cycle(0, 0, b, np.zeros_like(b))
        assert e.value.status == -1
        with pytest.raises(mod.OracleError) as e:
            h.v_cycle(1, 1, b, np.zeros_like(b), level=5)
        assert e.value.status == -2


# --------------------------------------------------------------- experiments.cpp
@pytest.mark.parametrize("ng,levels", [(8, 1), (16, 2), (32, 3)])
def test_fd_biharmonic_is_the_references(ng, levels):
    """problems.fd_biharmonic (the restatement the GPU tests use) against the
    reference's own fd_biharmonic (experiments.cpp:104-195): bitwise."""
    want = R.fd_biharmonic(ng, levels)
    got = pr.fd_biharmonic(ng, levels)
    assert digest(R.Mat(got.A)) == digest(want["A"])
    assert digest(R.Mat(got.mass)) == digest(want["mass"])
    assert len(got.transfers) == len(want["transfers"])
    for p, q in zip(got.transfers, want["transfers"]):
        assert digest(R.Mat(p)) == digest(q)
    assert np.array_equal(got.reference, want["reference"])
    assert np.array_equal(got.b, want["b"])
    assert got.h == want["h"]


def test_measure_rates_is_the_references():
    """The reference's measure_rates (experiments.cpp:15-67) on its own FD problem
    against the oracle's restatement: histories, status, iterations, rates."""
    fd = pr.fd_biharmonic(32, 3)
    oh = O.Hierarchy(O.Mat(fd.A), [O.Mat(p) for p in fd.transfers], t_max=2, probe=False)
    rh = R.Hierarchy(R.Mat(fd.A), [R.Mat(p) for p in fd.transfers], t_max=2)
    for k_pre, k_post in ((2, 2), (4, 0)):
        o = oh.measure_rates(O.Mat(fd.mass), fd.b, fd.reference, k_pre, k_post, seed=1, tol=1e-9, max_iter=40)
        r = rh.measure_rates(R.Mat(fd.mass), fd.b, fd.reference, k_pre, k_post, seed=1, tol=1e-9, max_iter=40)
        assert (o["iterations"], o["status"], o["blowup_iteration"]) == (r["iterations"], r["status"], r["blowup_iteration"])
        for key in ("l2_sq", "energy_sq", "residual"):
            assert np.array_equal(o[key], r[key]), key
        for key in ("rho_l2", "rho_a", "rho_r"):
            assert o[key] == r[key], key


# ----------------------------------------------------------------- matrix_io.cpp
def test_reference_matrix_io_round_trip(tmp_path, rng):
    sizes = random_layout(rng, 6, 4)
    a = random_spd(rng, sizes, 0.6)
    path = str(tmp_path / "a.bmat")
    R.write_matrix(path, R.Mat(a))
    back = R.read_matrix(path)
    assert digest(back) == digest(R.Mat(a))
    assert np.array_equal(back.row_sizes, sizes)
    v = rng.normal(size=17)
    R.write_vector(str(tmp_path / "v.txt"), v)
    assert np.array_equal(R.read_vector(str(tmp_path / "v.txt")), v)
    with open(path) as f:
        lines = f.read().splitlines()
    lines[2] = "1 x 3.0"
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    with pytest.raises(R.IoError) as e:
        R.read_matrix(path)
    assert e.value.line == 3
