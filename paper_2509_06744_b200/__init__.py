"""blockmg-b200: B200 (sm_100a) V-cycle application path of arXiv 2509.06744.

The compute is libbmgcuda.so (CUDA, C ABI in include/bmg_cuda.h); this package
is the Python mirror of the reference's hot-path interface over that ABI.
"""
from .native import (CHEB_FIRST, CHEB_FOURTH, RICHARDSON, BmgError, IoError, CudaError, InvalidArgument, NotPositiveDefinite, OutOfRange,  # noqa: F401
                     FSAI_ADAPTIVE, FSAI_DIAGONAL, FSAI_STATIC_LOWER, SetupParams, lib)
from .api import (apply_smoother, spmv_batch, BlockSparseMatrix, Context, LoopbackGroup, Fsai, Hierarchy, HostBsr, Vector, cheb_fourth_apply,  # noqa: F401
                  default_params, dot, galerkin_coarsen, lanczos_lambda_max, residual, spmv, spmv_transpose,
                  triple_product, read_matrix, write_matrix, read_vector, write_vector,
                  tridiag_eigs)
from . import problems  # noqa: F401

__version__ = "0.1.0"
