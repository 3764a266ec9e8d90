"""ctypes binding of libbmgcuda.so (the C ABI in include/bmg_cuda.h).

This is plumbing: the compute lives in the CUDA library.  Loading fails loudly
when the in-tree library is missing; there is no Python or CPU fallback.
Status codes are mapped back onto the reference's exception types
(kernels.cpp:9-11 invalid_argument, block_matrix.cpp:98-101 out_of_range,
small_cholesky.hpp:10-13 NotPositiveDefinite, multilevel.cpp:72-73 runtime_error).
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbmgcuda.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "bmg_cuda.h")

BMG_OK, BMG_EINVAL, BMG_ERANGE, BMG_ENOTSPD, BMG_ERUNTIME, BMG_ECUDA, BMG_ENCCL, BMG_EIO = 0, -1, -2, -3, -4, -5, -6, -7
BMG_SYMMETRIC = 1
FSAI_STATIC_LOWER, FSAI_DIAGONAL, FSAI_ADAPTIVE = 0, 1, 3
RICHARDSON, CHEB_FIRST, CHEB_FOURTH = 0, 1, 2  # SmootherKind (chebyshev.hpp:10)


class BmgError(RuntimeError):
    status = BMG_ERUNTIME


class InvalidArgument(BmgError, ValueError):
    status = BMG_EINVAL


class OutOfRange(BmgError, IndexError):
    status = BMG_ERANGE


class NotPositiveDefinite(BmgError):
    status = BMG_ENOTSPD

    def __init__(self, msg, pivot):
        super().__init__(msg)
        self.pivot = pivot


class CudaError(BmgError):
    status = BMG_ECUDA


class NcclError(BmgError):
    status = BMG_ENCCL


class IoError(BmgError):
    """IoError{line} (matrix_io.hpp:10-13)."""

    status = BMG_EIO

    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


class SetupParams(C.Structure):
    """SetupParams (multilevel.hpp:35-47)."""

    _fields_ = [
        ("t_max", C.c_int),
        ("tau", C.c_double),
        ("nest", C.c_int),
        ("fsai_kind", C.c_int),
        ("lanczos_iters", C.c_int),
        ("lanczos_safety", C.c_double),
        ("seed", C.c_uint64),
        ("coarse_dim_cap", C.c_int),
        ("smoother_kind", C.c_int),
        ("richardson_omega", C.c_double),
        ("first_kind_fraction", C.c_double),
    ]


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.c_double
_U64 = C.c_uint64
_PD = C.POINTER(C.c_double)
_PI32 = C.POINTER(C.c_int32)
_PI64 = C.POINTER(C.c_int64)
_PP = C.POINTER(C.c_void_p)

_SIGS = {
    "bmg_last_error": (C.c_char_p, []),
    "bmg_last_pivot": (_I, []),
    "bmg_version": (C.c_char_p, []),
    "bmg_setup_params_default": (None, [C.POINTER(SetupParams)]),
    "bmg_ctx_create": (_I, [_I, _PP]),
    "bmg_ctx_destroy": (_I, [_P]),
    "bmg_ctx_set_stream": (_I, [_P, _P]),
    "bmg_ctx_sync": (_I, [_P]),
    "bmg_ctx_launch_count": (_I64, [_P]),
    "bmg_bsr_create": (_I, [_P, _I, _PI32, _I, _PI32, _PI64, _PI32, _PD, _I, _PP]),
    "bmg_bsr_destroy": (_I, [_P]),
    "bmg_bsr_info": (_I, [_P, C.POINTER(_I), C.POINTER(_I), _PI64, C.POINTER(_I), C.POINTER(_I), _PI64, _PI64]),
    "bmg_bsr_sym_info": (_I, [_P, C.POINTER(_I), _PI64, _PD, _PD]),
    "bmg_bsr_download": (_I, [_P, _PI64, _PI32, _PD]),
    "bmg_bsr_transpose": (_I, [_P, _PP]),
    "bmg_vec_create": (_I, [_P, _I64, _PP]),
    "bmg_vec_destroy": (_I, [_P]),
    "bmg_vec_upload": (_I, [_P, _PD]),
    "bmg_vec_download": (_I, [_P, _PD]),
    "bmg_vec_fill": (_I, [_P, _D]),
    "bmg_vec_create_like": (_I, [_P, _PP]),
    "bmg_vec_copy": (_I, [_P, _P]),
    "bmg_vec_axpby": (_I, [_D, _P, _D, _P, _P]),
    "bmg_vec_device_ptr": (_P, [_P]),
    "bmg_vec_size": (_I64, [_P]),
    "bmg_spmv": (_I, [_P, _P, _P]),
    "bmg_spmv_batch": (_I, [_P, _I, _P, _P]),
    "bmg_spmv_t": (_I, [_P, _P, _P]),
    "bmg_residual": (_I, [_P, _P, _P, _P]),
    "bmg_dot": (_I, [_P, _P, _PD]),
    "bmg_galerkin": (_I, [_P, _P, _PP]),
    "bmg_fsai_build": (_I, [_P, _I, _I, _D, _I, _PP]),
    "bmg_fsai_build_pattern": (_I, [_P, _PI64, _PI32, _PP]),
    "bmg_fsai_from_factors": (_I, [_P, _P, _PD, _PP]),
    "bmg_fsai_destroy": (_I, [_P]),
    "bmg_fsai_apply": (_I, [_P, _P, _P]),
    "bmg_fsai_apply_transformed": (_I, [_P, _P, _P, _P]),
    "bmg_fsai_G": (_I, [_P, _PP]),
    "bmg_fsai_chain_len": (_I, [_P]),
    "bmg_fsai_factor": (_I, [_P, _I, _PP]),
    "bmg_triple_product": (_I, [_P, _P, _PP]),
    "bmg_cheb4_apply": (_I, [_P, _P, _P, _P, _D, _I]),
    "bmg_lanczos_lambda_max": (_I, [_P, _P, _I, _D, _U64, _PD]),
    "bmg_smoother_apply": (_I, [_P, _P, _I, _D, _D, _D, _I, _P, _P]),
    "bmg_hier_set_smoother": (_I, [_P, _I, _I, _D, _D, _D]),
    "bmg_hier_setup": (_I, [_P, _I, _PP, C.POINTER(SetupParams), _PP]),
    "bmg_hier_create": (_I, [_P, _I, _PP, _PP, _PP, _PD, _I, _PP]),
    "bmg_hier_destroy": (_I, [_P]),
    "bmg_hier_info": (_I, [_P, C.POINTER(_I), _PI64]),
    "bmg_hier_beta": (_I, [_P, _I, _PD]),
    "bmg_hier_level": (_I, [_P, _I, _PP, _PP, _PP]),
    "bmg_hier_cycle_bytes": (_I, [_P, _I, _I, _PI64]),
    "bmg_hier_cycle_bytes_batch": (_I, [_P, _I, _I, _I, _PI64]),
    "bmg_hier_cycle_bytes_ref": (_I, [_P, _I, _I, _PI64]),
    "bmg_vcycle_batch": (_I, [_P, _I, _I, _I, _P, _P]),
    "bmg_vcycle_batch_host": (_I, [_P, _I, _I, _I, _PD, _PD]),
    "bmg_hier_use_graph": (_I, [_P, _I]),
    "bmg_vcycle": (_I, [_P, _I, _I, _P, _P]),
    "bmg_vcycle_level": (_I, [_P, _I, _I, _I, _P, _P]),
    "bmg_vcycle_host": (_I, [_P, _I, _I, _PD, _PD]),
    "bmg_solve": (_I, [_P, _I, _I, _P, _P, _D, _I, _PD, C.POINTER(_I), C.POINTER(_I)]),
    "bmg_measure_rates": (_I, [_P, _P, _P, _P, _I, _I, C.c_uint64, _D, _I, _PD, _PD, _PD, C.POINTER(_I),
                               C.POINTER(_I), C.POINTER(_I), _PD]),
    "bmg_time_residual": (_I, [_P, _P, _P, _P, _I, _PD]),
    "bmg_nccl_unique_id": (_I, [C.c_char_p]),
    "bmg_ctx_create_nccl": (_I, [_I, _I, _I, C.c_char_p, _PP]),
    "bmg_ctx_transport_selftest": (_I, [_P, C.c_int64, _I, C.POINTER(C.c_int64)]),
    "bmg_loopback_create": (_I, [_I, _PP]),
    "bmg_loopback_destroy": (_I, [_P]),
    "bmg_ctx_create_loopback": (_I, [_I, _P, _I, _PP]),
    "bmg_hier_partition": (_I, [_P, _I, _I, _PI32, _I]),
    "bmg_dist_plan": (_I, [_I, _PI32, _PI32, _PI32, _I, _I, C.POINTER(SetupParams), _PI32, _PI32, _PI32, _PI32]),
    "bmg_hier_setup_dist": (_I, [_P, _I, _PI32, _PI32, _I, _P, _PP, C.POINTER(SetupParams), _PP]),
    "bmg_hier_setup_dist_emulated": (_I, [_P, _I, _I, _PI32, _PI32, _I, _PP, _PP, C.POINTER(SetupParams), _PP]),
    "bmg_hier_part_info": (_I, [_P, _I, _I, _PI32, _PI32, _PI32, _PI32]),
    "bmg_partition_rows": (_I, [_I, _PI64, _I, _I, _I, _PI32]),
    "bmg_row_window": (_I, [_PI64, _PI32, _I, _I, _I, _I, _PI32, _PI32]),
    "bmg_tridiag_eigs": (_I, [_I, _PD, _PD, _PD]),
    "bmg_io_read_matrix": (_I, [_P, C.c_char_p, _PP, C.POINTER(_I)]),
    "bmg_io_write_matrix": (_I, [_P, C.c_char_p]),
    "bmg_io_read_vector": (_I, [_P, C.c_char_p, _PP]),
    "bmg_io_write_vector": (_I, [_P, C.c_char_p]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    txt = open(HEADER_PATH).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bmg_[a-z0-9_]+)\s*\(", txt)))


def check(status: int) -> None:
    if status == BMG_OK:
        return
    msg = lib().bmg_last_error().decode()
    if status == BMG_EINVAL:
        raise InvalidArgument(msg)
    if status == BMG_ERANGE:
        raise OutOfRange(msg)
    if status == BMG_ENOTSPD:
        raise NotPositiveDefinite(msg, lib().bmg_last_pivot())
    if status == BMG_ECUDA:
        raise CudaError(msg)
    if status == BMG_ENCCL:
        raise NcclError(msg)
    if status == BMG_EIO:
        raise IoError(msg, lib().bmg_last_pivot())
    raise BmgError(msg)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_PD)


def i32ptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_PI32)


def i64ptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_PI64)
