"""ctypes wrapper of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

The oracle restates the reference's CPU algorithms (see bmg_oracle.h).  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this
module, as the checker or the CPU baseline; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_PD = C.POINTER(C.c_double)
_PI32 = C.POINTER(C.c_int32)
_PI64 = C.POINTER(C.c_int64)
_I = C.c_int
_D = C.c_double
_U64 = C.c_uint64

_SIGS = {
    "orc_last_error": (C.c_char_p, []),
    "orc_last_pivot": (_I, []),
    "orc_set_threads": (_I, [_I]),
    "orc_get_threads": (_I, []),
    "orc_mat_create": (_I, [_I, _PI32, _I, _PI32, _PI64, _PI32, _PD, _I, _PP]),
    "orc_mat_destroy": (None, [_P]),
    "orc_mat_info": (_I, [_P, C.POINTER(_I), C.POINTER(_I), _PI64, _PI64, C.POINTER(_I), C.POINTER(_I)]),
    "orc_mat_export": (_I, [_P, _PI64, _PI32, _PD]),
    "orc_spmv": (_I, [_P, _PD, _PD]),
    "orc_spmv_t": (_I, [_P, _PD, _PD]),
    "orc_multiply": (_I, [_P, _P, _PP]),
    "orc_transpose_multiply": (_I, [_P, _P, _PP]),
    "orc_triple_product": (_I, [_P, _P, _PP]),
    "orc_galerkin": (_I, [_P, _P, _PP]),
    "orc_cholesky": (_I, [_I, _PD, _PD, _PD]),
    "orc_chol_solve": (_I, [_I, _PD, _PD, _PD]),
    "orc_fsai_build": (_I, [_P, _I, _I, _D, _I, _PP]),
    "orc_fsai_destroy": (None, [_P]),
    "orc_fsai_build_pattern": (_I, [_P, _PI64, _PI32, _PP]),
    "orc_delta_ratio": (_I, [_P, _PI64, _PI32, _I, _I, _PD]),
    "orc_fsai_apply": (_I, [_P, _PD, _PD]),
    "orc_fsai_apply_transformed": (_I, [_P, _P, _PD, _PD]),
    "orc_fsai_chain_len": (_I, [_P]),
    "orc_fsai_factor": (_I, [_P, _I, _PP]),
    "orc_fsai_shat": (_I, [_P, _PD]),
    "orc_fsai_G": (_I, [_P, _PP]),
    "orc_lanczos_lambda_max": (_I, [_P, _P, _I, _D, _U64, _PD]),
    "orc_lanczos_diag": (_I, [_I, _PD, _I, _D, _U64, _I, _PD]),
    "orc_tridiag_eigs": (_I, [_I, _PD, _PD, _PD]),
    "orc_smoother_apply": (_I, [_P, _P, _I, _D, _D, _D, _I, _PD, _PD]),
    "orc_smoother_apply_diag": (_I, [_I, _PD, _I, _D, _D, _D, _I, _PD, _PD]),
    "orc_poly_eval": (_I, [_I, _I, _D, _D, _D, _PD]),
    "orc_fourth_kind_mu": (_D, [_I]),
    "orc_set_consume": (_I, [_I]),
    "orc_setup": (_I, [_P, _I, _PP, _I, _D, _I, _I, _I, _D, _U64, _I, _I, _I, _D, _D, _PP]),
    "orc_hier_destroy": (None, [_P]),
    "orc_hier_levels": (_I, [_P]),
    "orc_hier_level_A": (_I, [_P, _I, _PP]),
    "orc_hier_level_P": (_I, [_P, _I, _PP]),
    "orc_hier_level_fsai": (_I, [_P, _I, _PP]),
    "orc_hier_beta": (_I, [_P, _I, _PD]),
    "orc_hier_coarse_l": (_I, [_P, _PD]),
    "orc_vcycle": (_I, [_P, _I, _I, _I, _PD, _PD]),
    "orc_solve": (_I, [_P, _I, _I, _PD, _PD, _D, _I, _PD, C.POINTER(_I), C.POINTER(_I)]),
    "orc_measure_rates": (_I, [_P, _P, _PD, _PD, _I, _I, C.c_uint64, _D, _I, _PD, _PD, _PD, C.POINTER(_I),
                               C.POINTER(_I), C.POINTER(_I), _PD]),
    "orc_mix64": (_U64, [_U64]),
    "orc_rng_uniform": (_D, [_U64, _U64]),
}

_lib = None


class OracleError(RuntimeError):
    def __init__(self, status, msg, pivot=-1):
        super().__init__(msg)
        self.status = status
        self.pivot = pivot


def build():
    cmd = ["make", "-s", "-C", _HERE]
    subprocess.run(cmd, check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(st):
    if st != 0:
        raise OracleError(st, lib().orc_last_error().decode(), lib().orc_last_pivot())


def _d(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_PD)


def _i32(a):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_PI32)


def _i64(a):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_PI64)


class Mat:
    def __init__(self, host=None, _handle=None, _owned=True, row_sizes=None, col_sizes=None):
        self._owned = _owned
        if _handle is not None:
            self.h = _handle
            self.row_sizes = np.asarray(row_sizes, np.int32) if row_sizes is not None else None
            self.col_sizes = np.asarray(col_sizes, np.int32) if col_sizes is not None else None
            return
        h = C.c_void_p()
        check(lib().orc_mat_create(host.nbr, _i32(host.row_sizes), host.nbc, _i32(host.col_sizes),
                                   _i64(host.row_ptr), _i32(host.col_idx), _d(host.vals),
                                   1 if host.symmetric else 0, C.byref(h)))
        self.h = h
        self.row_sizes = host.row_sizes
        self.col_sizes = host.col_sizes

    def info(self):
        a, b, e, f = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        nnzb, nv = C.c_int64(), C.c_int64()
        check(lib().orc_mat_info(self.h, C.byref(a), C.byref(b), C.byref(nnzb), C.byref(nv), C.byref(e),
                                 C.byref(f)))
        return dict(nbr=a.value, nbc=b.value, nnzb=nnzb.value, nvals=nv.value, dim_r=e.value, dim_c=f.value)

    def export(self, symmetric=False):
        from paper_2509_06744_b200.api import HostBsr

        inf = self.info()
        rp = np.zeros(inf["nbr"] + 1, np.int64)
        ci = np.zeros(max(inf["nnzb"], 1), np.int32)
        vals = np.zeros(max(inf["nvals"], 1))
        check(lib().orc_mat_export(self.h, _i64(rp), _i32(ci), _d(vals)))
        rs = self.row_sizes if self.row_sizes is not None else None
        cs = self.col_sizes if self.col_sizes is not None else None
        return HostBsr(rs, cs, rp, ci[:inf["nnzb"]], vals[:inf["nvals"]], symmetric)

    def spmv(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.info()["dim_r"])
        check(lib().orc_spmv(self.h, _d(x), _d(y)))
        return y

    def spmv_t(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.info()["dim_c"])
        check(lib().orc_spmv_t(self.h, _d(x), _d(y)))
        return y

    def __del__(self):
        try:
            if self.h and self._owned:
                lib().orc_mat_destroy(self.h)
        except Exception:
            pass


def _newmat(fn, *args, row_sizes=None, col_sizes=None):
    h = C.c_void_p()
    check(fn(*args, C.byref(h)))
    return Mat(_handle=h, row_sizes=row_sizes, col_sizes=col_sizes)


def multiply(a, b):
    return _newmat(lib().orc_multiply, a.h, b.h, row_sizes=a.row_sizes, col_sizes=b.col_sizes)


def transpose_multiply(p, b):
    return _newmat(lib().orc_transpose_multiply, p.h, b.h, row_sizes=p.col_sizes, col_sizes=b.col_sizes)


def triple_product(f, a):
    return _newmat(lib().orc_triple_product, f.h, a.h, row_sizes=f.row_sizes, col_sizes=f.row_sizes)


def galerkin(a, p):
    return _newmat(lib().orc_galerkin, a.h, p.h, row_sizes=p.col_sizes, col_sizes=p.col_sizes)


def cholesky(b):
    b = np.ascontiguousarray(b, np.float64)
    n = b.shape[0]
    l = np.zeros((n, n))
    ld = C.c_double()
    check(lib().orc_cholesky(n, _d(b), _d(l), C.byref(ld)))
    return l, ld.value


class Fsai:
    STATIC, DIAGONAL, FULL, NESTED = 0, 1, 2, 3

    def __init__(self, a, kind, t_max=1, tau=1.0, nest=0, _handle=None, _owned=True):
        self._owned = _owned
        self.row_sizes = a.row_sizes if a is not None else None
        if _handle is not None:
            self.h = _handle
            return
        h = C.c_void_p()
        check(lib().orc_fsai_build(a.h, kind, t_max, tau, nest, C.byref(h)))
        self.h = h

    def apply(self, r):
        r = np.ascontiguousarray(r, np.float64)
        out = np.zeros_like(r)
        check(lib().orc_fsai_apply(self.h, _d(r), _d(out)))
        return out

    def apply_transformed(self, a, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros_like(x)
        check(lib().orc_fsai_apply_transformed(self.h, a.h, _d(x), _d(out)))
        return out

    def chain_len(self):
        return lib().orc_fsai_chain_len(self.h)

    def factor(self, k):
        return _newmat(lib().orc_fsai_factor, self.h, k, row_sizes=self.row_sizes, col_sizes=self.row_sizes)

    def shat(self):
        n = int(np.sum(np.asarray(self.row_sizes, np.int64) ** 2))
        out = np.zeros(n)
        check(lib().orc_fsai_shat(self.h, _d(out)))
        return out

    def G(self):
        return _newmat(lib().orc_fsai_G, self.h, row_sizes=self.row_sizes, col_sizes=self.row_sizes)

    def __del__(self):
        try:
            if self.h and self._owned:
                lib().orc_fsai_destroy(self.h)
        except Exception:
            pass


def _pattern_csr(n, pattern):
    """pattern: list of strict-lower column lists per block row."""
    pp = np.zeros(n + 1, np.int64)
    cols = []
    for i in range(n):
        cols.extend(sorted(pattern[i]))
        pp[i + 1] = len(cols)
    return pp, np.asarray(cols if cols else [0], np.int32)


def fsai_with_pattern(a, pattern):
    n = a.info()["nbr"]
    pp, pc = _pattern_csr(n, pattern)
    h = C.c_void_p()
    check(lib().orc_fsai_build_pattern(a.h, _i64(pp), _i32(pc), C.byref(h)))
    f = Fsai(None, 0, _handle=h)
    f.row_sizes = a.row_sizes
    return f


def delta_ratio(a, pattern, k, c):
    n = a.info()["nbr"]
    pp, pc = _pattern_csr(n, pattern)
    out = C.c_double()
    check(lib().orc_delta_ratio(a.h, _i64(pp), _i32(pc), k, c, C.byref(out)))
    return out.value


def lanczos_lambda_max(a, f, iters=100, safety=1.01, seed=42):
    out = C.c_double()
    check(lib().orc_lanczos_lambda_max(a.h, f.h, iters, safety, seed, C.byref(out)))
    return out.value


def lanczos_diag(lam, iters=100, safety=1.01, seed=42, smallest=False):
    lam = np.ascontiguousarray(lam, np.float64)
    out = C.c_double()
    check(lib().orc_lanczos_diag(len(lam), _d(lam), iters, safety, seed, 1 if smallest else 0, C.byref(out)))
    return out.value


def tridiag_eigs(d, e):
    d = np.ascontiguousarray(d, np.float64)
    e = np.ascontiguousarray(e, np.float64)
    out = np.zeros(len(d))
    check(lib().orc_tridiag_eigs(len(d), _d(d), _d(e) if len(e) else None, _d(out)))
    return out


RICHARDSON, CHEB_FIRST, CHEB_FOURTH = 0, 1, 2


def smoother_apply(a, f, kind, b, x, k, alpha=0.0, beta=1.0, omega=1.0):
    b = np.ascontiguousarray(b, np.float64)
    x = np.array(x, np.float64, copy=True)
    check(lib().orc_smoother_apply(a.h, f.h if f is not None else None, kind, alpha, beta, omega, k, _d(b), _d(x)))
    return x


def smoother_apply_diag(lam, kind, b, x, k, alpha=0.0, beta=1.0, omega=1.0):
    lam = np.ascontiguousarray(lam, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    x = np.array(x, np.float64, copy=True)
    check(lib().orc_smoother_apply_diag(len(lam), _d(lam), kind, alpha, beta, omega, k, _d(b), _d(x)))
    return x


def poly_eval(kind, degree, t, alpha=0.0, beta=1.0):
    out = C.c_double()
    check(lib().orc_poly_eval(kind, degree, alpha, beta, t, C.byref(out)))
    return out.value


FIRST_T, FOURTH_W, SCALED_FIRST, SCALED_FOURTH = 0, 1, 2, 3


class Hierarchy:
    def __init__(self, a, transfers, t_max=1, tau=1.0, nest=0, fsai_kind=3, lanczos_iters=100,
                 lanczos_safety=1.01, seed=42, coarse_dim_cap=5000, probe=True, smoother_kind=2,
                 richardson_omega=1.0, first_kind_fraction=1.0 / 30.0, consume=False):
        """consume=True moves a and the transfers into the hierarchy (they are
        left empty): large configs are not held twice in host memory."""
        arr = (C.c_void_p * max(len(transfers), 1))(*[t.h.value for t in transfers])
        h = C.c_void_p()
        lib().orc_set_consume(1 if consume else 0)
        try:
            check(lib().orc_setup(a.h, len(transfers), arr, t_max, tau, nest, fsai_kind, lanczos_iters,
                                  lanczos_safety, seed, coarse_dim_cap, 1 if probe else 0, smoother_kind,
                                  richardson_omega, first_kind_fraction, C.byref(h)))
        finally:
            lib().orc_set_consume(0)
        self.h = h
        self.sizes = [a.row_sizes] + []
        self._transfers = transfers
        self._a = a

    def levels(self):
        return lib().orc_hier_levels(self.h)

    def level_sizes(self, l):
        L = self.levels()
        if l == L - 1:
            return self._a.row_sizes
        return self._transfers[l].col_sizes

    def A(self, l):
        h = C.c_void_p()
        check(lib().orc_hier_level_A(self.h, l, C.byref(h)))
        s = self.level_sizes(l)
        return Mat(_handle=h, _owned=False, row_sizes=s, col_sizes=s)

    def P(self, l):
        h = C.c_void_p()
        check(lib().orc_hier_level_P(self.h, l, C.byref(h)))
        return Mat(_handle=h, _owned=False, row_sizes=self.level_sizes(l), col_sizes=self.level_sizes(l - 1))

    def fsai(self, l):
        h = C.c_void_p()
        check(lib().orc_hier_level_fsai(self.h, l, C.byref(h)))
        f = Fsai(None, 0, _handle=h, _owned=False)
        f.row_sizes = self.level_sizes(l)
        return f

    def beta(self, l):
        out = C.c_double()
        check(lib().orc_hier_beta(self.h, l, C.byref(out)))
        return out.value

    def v_cycle(self, k_pre, k_post, b, x, level=None):
        if level is None:
            level = self.levels() - 1
        b = np.ascontiguousarray(b, np.float64)
        x = np.array(x, np.float64, copy=True)
        check(lib().orc_vcycle(self.h, k_pre, k_post, level, _d(b), _d(x)))
        return x

    def solve(self, k_pre, k_post, b, x, tol=1e-8, max_iter=50):
        b = np.ascontiguousarray(b, np.float64)
        x = np.array(x, np.float64, copy=True)
        hist = np.zeros(max_iter + 1)
        it, st = C.c_int(), C.c_int()
        check(lib().orc_solve(self.h, k_pre, k_post, _d(b), _d(x), tol, max_iter, _d(hist), C.byref(it),
                              C.byref(st)))
        return hist[:it.value + 1], it.value, st.value, x

    def measure_rates(self, mass, b, u_ref, k_pre, k_post, seed=0, tol=1e-8, max_iter=50):
        """measure_rates (experiments.cpp:15-67) -> dict of histories and rates."""
        b = np.ascontiguousarray(b, np.float64)
        u = np.ascontiguousarray(u_ref, np.float64)
        l2, en, rs = np.zeros(max_iter + 1), np.zeros(max_iter + 1), np.zeros(max_iter + 1)
        rates = np.zeros(3)
        it, st, bl = C.c_int(), C.c_int(), C.c_int()
        check(lib().orc_measure_rates(self.h, mass.h, _d(b), _d(u), k_pre, k_post, seed, tol, max_iter, _d(l2),
                                      _d(en), _d(rs), C.byref(it), C.byref(st), C.byref(bl), _d(rates)))
        n = it.value + 1
        return dict(l2_sq=l2[:n], energy_sq=en[:n], residual=rs[:n], iterations=it.value, status=st.value,
                    blowup_iteration=bl.value, rho_l2=rates[0], rho_a=rates[1], rho_r=rates[2])

    def __del__(self):
        try:
            if self.h:
                lib().orc_hier_destroy(self.h)
        except Exception:
            pass


def set_threads(n):
    lib().orc_set_threads(n)


def get_threads():
    return lib().orc_get_threads()
