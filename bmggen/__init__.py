"""ctypes loader of bmggen/libbmggen.so, the synthetic BASELINE input generator
(include/bmg_gen.h).  Input data only: both benchmark arms and the tests build
their inputs through it; it is neither the product (libbmgcuda.so) nor the
oracle."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbmggen.so")

_P64 = C.POINTER(C.c_int64)
_P32 = C.POINTER(C.c_int32)
_PD = C.POINTER(C.c_double)
_SIGS = {
    "bmg_gen_last_error": (C.c_char_p, []),
    "bmg_gen_stencil": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_int64,
                                  C.c_int64, _P64, _P64, _P32, _PD]),
    "bmg_gen_prolongation": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int64, C.c_int64,
                                       _P64, _P64, _P32, _PD]),
    "bmg_gen_normal": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, _PD]),
}
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


class GeneratorError(ValueError):
    pass


def check(status: int):
    if status != 0:
        raise GeneratorError(lib().bmg_gen_last_error().decode())
