"""The REFERENCE ITSELF behind the pyoracle wrappers -- TEST INFRASTRUCTURE ONLY.

oracle/_ref/libblockmg_ref.so holds the reference's own unmodified sources
(/root/reference/proj/src/*.cpp, compiled where they lie by `make -C oracle ref`
against oracle/eigen_shim -- Eigen3 is not installed) and exports the same C API
as liboracle.so (bmg_oracle.h).  This module is a second instance of pyoracle
bound to that library, so a test can run `O.<f>(...)` and `R.<f>(...)` on the same
inputs and compare bitwise.  /root/reference is absent on the GPU box: the library
is built here and travels prebuilt; `available()` says whether it can be loaded.
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB_PATH = os.path.join(_HERE, "_ref", "libblockmg_ref.so")
REF_TREE = "/root/reference/proj"

_spec = importlib.util.spec_from_file_location("oracle._pyref_impl", os.path.join(_HERE, "pyoracle.py"))
_m = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_m)
_m.LIB_PATH = REF_LIB_PATH


def _build():
    if not os.path.isdir(REF_TREE):
        raise RuntimeError("the reference tree is absent and oracle/_ref/libblockmg_ref.so was not prebuilt")
    subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)


_m.build = _build


def available() -> bool:
    return os.path.exists(REF_LIB_PATH) or os.path.isdir(REF_TREE)


# the pyoracle surface, bound to the reference library
for _k in ("Mat", "Fsai", "Hierarchy", "OracleError", "multiply", "transpose_multiply", "triple_product", "galerkin",
           "cholesky", "fsai_with_pattern", "delta_ratio", "lanczos_lambda_max", "lanczos_diag", "tridiag_eigs",
           "smoother_apply", "smoother_apply_diag", "poly_eval", "RICHARDSON", "CHEB_FIRST", "CHEB_FOURTH",
           "FIRST_T", "FOURTH_W", "SCALED_FIRST", "SCALED_FOURTH", "check", "lib"):
    globals()[_k] = getattr(_m, _k)

_PD, _PI32, _PP, _I = _m._PD, _m._PI32, _m._PP, _m._I
_EXTRA = {
    "orc_is_reference": (_I, []),
    "orc_mat_layouts": (_I, [C.c_void_p, _PI32, _PI32]),
    "orc_chol_solve_spd": (_I, [_I, _PD, _PD, _PD]),
    "orc_fd_biharmonic": (_I, [_I, _I, _PP, _PP, _PP, _PD, _PD, _PD]),
    "orc_read_matrix": (_I, [C.c_char_p, _PP]),
    "orc_write_matrix": (_I, [C.c_char_p, C.c_void_p]),
    "orc_write_vector": (_I, [C.c_char_p, _I, _PD]),
    "orc_read_vector": (_I, [C.c_char_p, _I, _PD, C.POINTER(_I)]),
}
_extra_bound = False


def _xlib():
    global _extra_bound
    h = _m.lib()
    if not _extra_bound:
        for name, (res, args) in _EXTRA.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        assert h.orc_is_reference() == 1
        _extra_bound = True
    return h


def _wrap(handle):
    """Mat over a library-made matrix, with its layouts read back."""
    mat = _m.Mat(_handle=handle)
    inf = mat.info()
    rs, cs = np.zeros(inf["nbr"], np.int32), np.zeros(inf["nbc"], np.int32)
    _m.check(_xlib().orc_mat_layouts(handle, _m._i32(rs), _m._i32(cs)))
    mat.row_sizes, mat.col_sizes = rs, cs
    return mat


def chol_solve_spd(b, rhs):
    """SmallCholesky(B).solve(rhs) (small_cholesky.cpp:32-34)."""
    b = np.ascontiguousarray(b, np.float64)
    rhs = np.ascontiguousarray(rhs, np.float64)
    x = np.zeros_like(rhs)
    _m.check(_xlib().orc_chol_solve_spd(b.shape[0], _m._d(b), _m._d(rhs), _m._d(x)))
    return x


def fd_biharmonic(n_grid: int, levels: int):
    """The reference's fd_biharmonic (experiments.cpp:104-195): dict with A, mass
    (Mat), transfers (list of Mat, coarsest first), b, reference, h."""
    n = (n_grid - 1) ** 2
    a, mass = C.c_void_p(), C.c_void_p()
    tr = (C.c_void_p * max(levels - 1, 1))()
    b, u = np.zeros(n), np.zeros(n)
    h = C.c_double()
    _m.check(_xlib().orc_fd_biharmonic(n_grid, levels, C.byref(a), C.byref(mass), tr, _m._d(b), _m._d(u), C.byref(h)))
    return dict(A=_wrap(a), mass=_wrap(mass), transfers=[_wrap(C.c_void_p(tr[l])) for l in range(levels - 1)], b=b,
                reference=u, h=h.value)


class IoError(RuntimeError):
    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


def _io(st):
    if st == -5:
        raise IoError(_m.lib().orc_last_error().decode(), _m.lib().orc_last_pivot())
    _m.check(st)


def read_matrix(path: str):
    h = C.c_void_p()
    _io(_xlib().orc_read_matrix(path.encode(), C.byref(h)))
    return _wrap(h)


def write_matrix(path: str, mat):
    _io(_xlib().orc_write_matrix(path.encode(), mat.h))


def write_vector(path: str, v):
    v = np.ascontiguousarray(v, np.float64)
    _io(_xlib().orc_write_vector(path.encode(), len(v), _m._d(v)))


def read_vector(path: str, cap: int = 1 << 24):
    v = np.zeros(cap)
    n = C.c_int()
    _io(_xlib().orc_read_vector(path.encode(), cap, _m._d(v), C.byref(n)))
    return v[:n.value].copy()
