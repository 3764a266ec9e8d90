"""Python mirror of the reference's hot-path interface over the C ABI.

Names follow /root/reference/proj/include/blockmg: BlockSparseMatrix
(block_matrix.hpp:26-70), spmv / spmv_transpose (kernels.hpp:15,19),
galerkin_coarsen (multilevel.hpp:50), build_fsai / nested_build (fsai.hpp:25,68),
cheb_fourth_apply (chebyshev.hpp:48), lanczos_lambda_max (multilevel.hpp:53),
setup / v_cycle (multilevel.hpp:59,65) and the measure_rates-style solve loop
(experiments.cpp:15-67).  Every object lives on the GPU; host data crosses the
boundary only in the explicit upload/download calls.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native as N
from .native import check, dptr, i32ptr, i64ptr, lib


@dataclass
class HostBsr:
    """Host block-CSR: row-major unpadded blocks in row_ptr/col_idx order."""

    row_sizes: np.ndarray
    col_sizes: np.ndarray
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    symmetric: bool = False

    def __post_init__(self):
        self.row_sizes = np.ascontiguousarray(self.row_sizes, dtype=np.int32)
        self.col_sizes = np.ascontiguousarray(self.col_sizes, dtype=np.int32)
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        self.vals = np.ascontiguousarray(self.vals, dtype=np.float64)

    @property
    def nbr(self):
        return len(self.row_sizes)

    @property
    def nbc(self):
        return len(self.col_sizes)

    @property
    def nnzb(self):
        return int(self.row_ptr[-1])

    @property
    def dim_r(self):
        return int(self.row_sizes.sum())

    @property
    def dim_c(self):
        return int(self.col_sizes.sum())

    def to_dense(self) -> np.ndarray:
        ro = np.concatenate([[0], np.cumsum(self.row_sizes)])
        co = np.concatenate([[0], np.cumsum(self.col_sizes)])
        out = np.zeros((ro[-1], co[-1]))
        v = 0
        for i in range(self.nbr):
            for p in range(self.row_ptr[i], self.row_ptr[i + 1]):
                j = self.col_idx[p]
                mi, mj = self.row_sizes[i], self.col_sizes[j]
                out[ro[i]:ro[i] + mi, co[j]:co[j] + mj] = self.vals[v:v + mi * mj].reshape(mi, mj)
                v += mi * mj
        return out


class LoopbackGroup:
    """bmg_loopback: `world` ranks as threads of this process on one device."""

    def __init__(self, world: int):
        self.h = C.c_void_p()
        self.world = world
        check(lib().bmg_loopback_create(world, C.byref(self.h)))

    def close(self):
        if self.h:
            check(lib().bmg_loopback_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    def __init__(self, device: int = 0, nccl: tuple | None = None, loopback: tuple | None = None):
        """nccl = (rank, world, unique_id_bytes) for a multi-GPU context;
        loopback = (LoopbackGroup, rank) for a rank thread of a loopback group."""
        h = C.c_void_p()
        if nccl is not None:
            rank, world, uid = nccl
            check(lib().bmg_ctx_create_nccl(device, rank, world, bytes(uid), C.byref(h)))
        elif loopback is not None:
            group, rank = loopback
            world = group.world
            check(lib().bmg_ctx_create_loopback(device, group.h, rank, C.byref(h)))
            self._group = group
        else:
            rank, world = 0, 1
            check(lib().bmg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.rank, self.world = rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().bmg_nccl_unique_id(buf))
        return buf.raw

    def transport_selftest(self, count: int = 1 << 16, reps: int = 3) -> int:
        """bmg_ctx_transport_selftest: the halo-exchange pattern with this rank as
        its own peer (captured where the transport allows) + an all-reduce;
        returns the number of mismatching entries."""
        bad = C.c_int64()
        check(lib().bmg_ctx_transport_selftest(self.h, count, reps, C.byref(bad)))
        return int(bad.value)

    def set_stream(self, stream_ptr: int | None):
        check(lib().bmg_ctx_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def sync(self):
        check(lib().bmg_ctx_sync(self.h))

    @property
    def launch_count(self) -> int:
        return int(lib().bmg_ctx_launch_count(self.h))

    def close(self):
        if self.h:
            check(lib().bmg_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BlockSparseMatrix:
    """Device BSR (reference BlockSparseMatrix, block_matrix.hpp:26-70)."""

    def __init__(self, ctx: Context, host: HostBsr | None = None, _handle=None, _owned=True):
        self.ctx = ctx
        self._owned = _owned
        if _handle is not None:
            self.h = _handle
            return
        h = C.c_void_p()
        check(lib().bmg_bsr_create(ctx.h, host.nbr, i32ptr(host.row_sizes), host.nbc, i32ptr(host.col_sizes),
                                   i64ptr(host.row_ptr), i32ptr(host.col_idx), dptr(host.vals),
                                   N.BMG_SYMMETRIC if host.symmetric else 0, C.byref(h)))
        self.h = h

    def info(self) -> dict:
        a, b, d, e = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        nnzb, dev, pb = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().bmg_bsr_info(self.h, C.byref(a), C.byref(b), C.byref(nnzb), C.byref(d), C.byref(e),
                                 C.byref(dev), C.byref(pb)))
        return dict(nbr=a.value, nbc=b.value, nnzb=nnzb.value, dim_r=d.value, dim_c=e.value,
                    device_bytes=dev.value, pass_bytes=pb.value)

    def sym_info(self) -> dict:
        """Symmetric-half streaming of this matrix (bmg_bsr_sym_info)."""
        h, pb = C.c_int(), C.c_int64()
        t1, t0 = C.c_double(), C.c_double()
        check(lib().bmg_bsr_sym_info(self.h, C.byref(h), C.byref(pb), C.byref(t1), C.byref(t0)))
        return dict(half=bool(h.value), pass_bytes=pb.value, half_ms=t1.value, full_ms=t0.value)

    def download(self, row_sizes, col_sizes, symmetric=False) -> HostBsr:
        inf = self.info()
        rp = np.zeros(inf["nbr"] + 1, np.int64)
        ci = np.zeros(max(inf["nnzb"], 1), np.int32)
        rs = np.asarray(row_sizes, np.int64)
        cs = np.asarray(col_sizes, np.int64)
        check(lib().bmg_bsr_download(self.h, i64ptr(rp), i32ptr(ci), None))
        nvals = int(sum(rs[i] * cs[ci[p]] for i in range(inf["nbr"]) for p in range(rp[i], rp[i + 1]))) \
            if not (np.all(rs == rs[0]) and np.all(cs == cs[0])) else int(inf["nnzb"] * rs[0] * cs[0])
        vals = np.zeros(max(nvals, 1))
        check(lib().bmg_bsr_download(self.h, i64ptr(rp), i32ptr(ci), dptr(vals)))
        return HostBsr(row_sizes, col_sizes, rp, ci[:inf["nnzb"]], vals[:nvals], symmetric)

    def transpose(self) -> "BlockSparseMatrix":
        h = C.c_void_p()
        check(lib().bmg_bsr_transpose(self.h, C.byref(h)))
        return BlockSparseMatrix(self.ctx, _handle=h)

    def close(self):
        if self.h and self._owned:
            check(lib().bmg_bsr_destroy(self.h))
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Vector:
    def __init__(self, ctx: Context, n_or_array):
        self.ctx = ctx
        if isinstance(n_or_array, (int, np.integer)):
            n = int(n_or_array)
            data = None
        else:
            data = np.ascontiguousarray(n_or_array, dtype=np.float64)
            n = data.size
        h = C.c_void_p()
        check(lib().bmg_vec_create(ctx.h, n, C.byref(h)))
        self.h = h
        self.n = n
        if data is not None:
            self.upload(data)

    def upload(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        assert a.size == self.n
        check(lib().bmg_vec_upload(self.h, dptr(a)))

    def download(self) -> np.ndarray:
        out = np.empty(self.n)
        check(lib().bmg_vec_download(self.h, dptr(out)))
        return out

    def fill(self, v: float):
        check(lib().bmg_vec_fill(self.h, v))

    @property
    def device_ptr(self) -> int:
        return lib().bmg_vec_device_ptr(self.h)

    def close(self):
        if self.h:
            check(lib().bmg_vec_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spmv(a: BlockSparseMatrix, x: Vector, y: Vector):
    check(lib().bmg_spmv(a.h, x.h, y.h))


def spmv_batch(a: BlockSparseMatrix, nrhs: int, x: Vector, y: Vector):
    """Y = A X, nrhs right-hand sides interleaved per scalar row (bmg_spmv_batch)."""
    check(lib().bmg_spmv_batch(a.h, nrhs, x.h, y.h))


def spmv_transpose(a: BlockSparseMatrix, x: Vector, y: Vector):
    check(lib().bmg_spmv_t(a.h, x.h, y.h))


def residual(a: BlockSparseMatrix, b: Vector, x: Vector, r: Vector):
    check(lib().bmg_residual(a.h, b.h, x.h, r.h))


def dot(a: Vector, b: Vector) -> float:
    out = C.c_double()
    check(lib().bmg_dot(a.h, b.h, C.byref(out)))
    return out.value


def galerkin_coarsen(a: BlockSparseMatrix, p: BlockSparseMatrix) -> BlockSparseMatrix:
    h = C.c_void_p()
    check(lib().bmg_galerkin(a.h, p.h, C.byref(h)))
    return BlockSparseMatrix(a.ctx, _handle=h)


def triple_product(f: BlockSparseMatrix, a: BlockSparseMatrix) -> BlockSparseMatrix:
    h = C.c_void_p()
    check(lib().bmg_triple_product(f.h, a.h, C.byref(h)))
    return BlockSparseMatrix(a.ctx, _handle=h)


class Fsai:
    """Device block-FSAI, M = G^T G (NestedFsai, fsai.hpp:56-66)."""

    def __init__(self, ctx, handle, owned=True):
        self.ctx = ctx
        self.h = handle
        self._owned = owned

    @classmethod
    def from_pattern(cls, a: BlockSparseMatrix, pattern) -> "Fsai":
        """build_fsai(A, LowerPattern p) (fsai.hpp:25); pattern[i] = iterable of j <= i."""
        n = a.info()["nbr"]
        pp = np.zeros(n + 1, np.int64)
        cols = []
        for i in range(n):
            cols.extend(int(j) for j in pattern[i])
            pp[i + 1] = len(cols)
        pc = np.asarray(cols if cols else [0], np.int32)
        h = C.c_void_p()
        check(lib().bmg_fsai_build_pattern(a.h, i64ptr(pp), i32ptr(pc), C.byref(h)))
        return cls(a.ctx, h)

    @classmethod
    def build(cls, a: BlockSparseMatrix, kind=N.FSAI_ADAPTIVE, t_max=1, tau=1.0, nest=0) -> "Fsai":
        h = C.c_void_p()
        check(lib().bmg_fsai_build(a.h, kind, t_max, tau, nest, C.byref(h)))
        return cls(a.ctx, h)

    @classmethod
    def from_factors(cls, ctx: Context, F: BlockSparseMatrix, shat_l_packed: np.ndarray) -> "Fsai":
        h = C.c_void_p()
        s = np.ascontiguousarray(shat_l_packed, np.float64)
        check(lib().bmg_fsai_from_factors(ctx.h, F.h, dptr(s), C.byref(h)))
        return cls(ctx, h)

    def apply(self, r: Vector, z: Vector):
        check(lib().bmg_fsai_apply(self.h, r.h, z.h))

    def apply_transformed(self, a: BlockSparseMatrix, x: Vector, y: Vector):
        check(lib().bmg_fsai_apply_transformed(self.h, a.h, x.h, y.h))

    @property
    def chain_len(self) -> int:
        return int(lib().bmg_fsai_chain_len(self.h))

    def factor(self, k: int) -> BlockSparseMatrix:
        h = C.c_void_p()
        check(lib().bmg_fsai_factor(self.h, k, C.byref(h)))
        return BlockSparseMatrix(self.ctx, _handle=h, _owned=False)

    @property
    def G(self) -> BlockSparseMatrix:
        h = C.c_void_p()
        check(lib().bmg_fsai_G(self.h, C.byref(h)))
        return BlockSparseMatrix(self.ctx, _handle=h, _owned=False)

    def close(self):
        if self.h and self._owned:
            check(lib().bmg_fsai_destroy(self.h))
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cheb_fourth_apply(a: BlockSparseMatrix, m: Fsai, b: Vector, x: Vector, beta: float, k: int):
    """x <- cheb_fourth_apply(A, M, b, x, beta, k) (chebyshev.hpp:48-69), in place."""
    check(lib().bmg_cheb4_apply(a.h, m.h, b.h, x.h, beta, k))


def apply_smoother(a: BlockSparseMatrix, m: Fsai, kind: int, b: Vector, x: Vector, k: int, alpha=0.0, beta=1.0,
                   omega=1.0):
    """x <- apply_smoother(spec, k, A, M, b, x) (chebyshev.hpp:117-129), in place."""
    check(lib().bmg_smoother_apply(a.h, m.h, kind, alpha, beta, omega, k, b.h, x.h))


def lanczos_lambda_max(a: BlockSparseMatrix, m: Fsai, iters=100, safety=1.01, seed=42) -> float:
    out = C.c_double()
    check(lib().bmg_lanczos_lambda_max(a.h, m.h, iters, safety, seed, C.byref(out)))
    return out.value


def default_params(**kw) -> N.SetupParams:
    p = N.SetupParams()
    lib().bmg_setup_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class Hierarchy:
    """Device multigrid hierarchy (Hierarchy, multilevel.hpp:28-33)."""

    def __init__(self, ctx, handle, keep=()):
        self.ctx = ctx
        self.h = handle
        self._keep = list(keep)

    @classmethod
    def setup(cls, a_finest: BlockSparseMatrix, transfers, params: N.SetupParams | None = None) -> "Hierarchy":
        arr = (C.c_void_p * max(len(transfers), 1))(*[t.h.value for t in transfers])
        h = C.c_void_p()
        check(lib().bmg_hier_setup(a_finest.h, len(transfers), arr,
                                   C.byref(params) if params is not None else None, C.byref(h)))
        return cls(a_finest.ctx, h, keep=[a_finest, *transfers])

    @classmethod
    def create(cls, ctx, A, P, M, beta, coarse_dim_cap=1 << 30) -> "Hierarchy":
        L = len(A)
        aa = (C.c_void_p * L)(*[a.h.value for a in A])
        pp = (C.c_void_p * L)(*[(p.h.value if p is not None else None) for p in P])
        mm = (C.c_void_p * L)(*[(m.h.value if m is not None else None) for m in M])
        bb = np.ascontiguousarray(beta, np.float64)
        h = C.c_void_p()
        check(lib().bmg_hier_create(ctx.h, L, aa, pp, mm, dptr(bb), coarse_dim_cap, C.byref(h)))
        return cls(ctx, h, keep=[*A, *P, *M])

    @classmethod
    def setup_dist(cls, ctx, a_ext: BlockSparseMatrix, transfers, granule, radius, agglomerate: int = 1,
                   params: N.SetupParams | None = None) -> "Hierarchy":
        """This rank's share of the distributed setup (bmg_hier_setup_dist):
        a_ext / transfers are the plan's extended strips (problems.dist_inputs)."""
        arr = (C.c_void_p * max(len(transfers), 1))(*[t.h.value for t in transfers])
        g = np.ascontiguousarray(granule, np.int32)
        r = np.ascontiguousarray(radius, np.int32)
        h = C.c_void_p()
        check(lib().bmg_hier_setup_dist(ctx.h, len(transfers) + 1, i32ptr(g), i32ptr(r), agglomerate, a_ext.h, arr,
                                        C.byref(params) if params is not None else None, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def setup_dist_emulated(cls, ctx, a_ext, transfers, granule, radius, agglomerate: int = 1,
                            params: N.SetupParams | None = None) -> "Hierarchy":
        """Every rank of the distributed setup in this process: a_ext[r] and
        transfers[r] (a list per rank)."""
        world = len(a_ext)
        L = len(transfers[0]) + 1
        aa = (C.c_void_p * world)(*[a.h.value for a in a_ext])
        flat = [t.h.value for ts in transfers for t in ts]
        tt = (C.c_void_p * max(len(flat), 1))(*flat)
        g = np.ascontiguousarray(granule, np.int32)
        r = np.ascontiguousarray(radius, np.int32)
        h = C.c_void_p()
        check(lib().bmg_hier_setup_dist_emulated(ctx.h, world, L, i32ptr(g), i32ptr(r), agglomerate, aa, tt,
                                                 C.byref(params) if params is not None else None, C.byref(h)))
        return cls(ctx, h)

    @property
    def levels(self) -> int:
        n = C.c_int()
        check(lib().bmg_hier_info(self.h, C.byref(n), None))
        return n.value

    @property
    def device_bytes(self) -> int:
        b = C.c_int64()
        check(lib().bmg_hier_info(self.h, None, C.byref(b)))
        return b.value

    def beta(self, level: int) -> float:
        out = C.c_double()
        check(lib().bmg_hier_beta(self.h, level, C.byref(out)))
        return out.value

    def set_smoother(self, level: int, kind: int, alpha=0.0, beta=1.0, omega=1.0):
        check(lib().bmg_hier_set_smoother(self.h, level, kind, alpha, beta, omega))

    def level(self, l: int):
        a, p, m = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().bmg_hier_level(self.h, l, C.byref(a), C.byref(p), C.byref(m)))
        A = BlockSparseMatrix(self.ctx, _handle=a, _owned=False)
        P = BlockSparseMatrix(self.ctx, _handle=p, _owned=False) if p.value else None
        M = Fsai(self.ctx, m, owned=False) if m.value else None
        return A, P, M

    def cycle_bytes(self, k_pre, k_post, nrhs: int = 1) -> int:
        out = C.c_int64()
        check(lib().bmg_hier_cycle_bytes_batch(self.h, k_pre, k_post, nrhs, C.byref(out)))
        return out.value

    def cycle_bytes_ref(self, k_pre, k_post) -> int:
        """cycle_bytes with the A passes at full storage (the reference's algorithm)."""
        out = C.c_int64()
        check(lib().bmg_hier_cycle_bytes_ref(self.h, k_pre, k_post, C.byref(out)))
        return out.value

    def partition(self, world: int, granule, agglomerate: int = 1, rank: int = -1):
        """Row-partition the hierarchy (rank = -1: emulate all ranks in-process)."""
        g = np.ascontiguousarray(granule, np.int32)
        check(lib().bmg_hier_partition(self.h, world, rank, i32ptr(g), agglomerate))

    def part_info(self, level: int, rank: int):
        lo, hi, wlo, whi = (C.c_int32() for _ in range(4))
        check(lib().bmg_hier_part_info(self.h, level, rank, C.byref(lo), C.byref(hi), C.byref(wlo), C.byref(whi)))
        return lo.value, hi.value, wlo.value, whi.value

    def use_graph(self, on: bool):
        check(lib().bmg_hier_use_graph(self.h, 1 if on else 0))

    def v_cycle(self, k_pre, k_post, b: Vector, x: Vector):
        check(lib().bmg_vcycle(self.h, k_pre, k_post, b.h, x.h))

    def v_cycle_level(self, k_pre, k_post, level: int, b: Vector, x: Vector):
        """v_cycle(h, spec, level, b, x) (multilevel.hpp:65): start on `level`."""
        check(lib().bmg_vcycle_level(self.h, k_pre, k_post, level, b.h, x.h))

    def v_cycle_batch(self, k_pre, k_post, nrhs: int, b: Vector, x: Vector):
        """K right-hand sides interleaved per scalar row (b[i*K + v]); bmg_vcycle_batch."""
        check(lib().bmg_vcycle_batch(self.h, k_pre, k_post, nrhs, b.h, x.h))

    def v_cycle_batch_host(self, k_pre, k_post, nrhs: int, b: np.ndarray, x: np.ndarray):
        check(lib().bmg_vcycle_batch_host(self.h, k_pre, k_post, nrhs, dptr(b), dptr(x)))

    def v_cycle_batch_host_ptr(self, k_pre, k_post, nrhs: int, b_ptr: int, x_ptr: int):
        check(lib().bmg_vcycle_batch_host(self.h, k_pre, k_post, nrhs, C.cast(b_ptr, N._PD), C.cast(x_ptr, N._PD)))

    def v_cycle_host(self, k_pre, k_post, b: np.ndarray, x: np.ndarray):
        check(lib().bmg_vcycle_host(self.h, k_pre, k_post, dptr(b), dptr(x)))

    def v_cycle_host_ptr(self, k_pre, k_post, b_ptr: int, x_ptr: int):
        check(lib().bmg_vcycle_host(self.h, k_pre, k_post, C.cast(b_ptr, N._PD), C.cast(x_ptr, N._PD)))

    def solve(self, k_pre, k_post, b: Vector, x: Vector, tol=1e-8, max_iter=50):
        hist = np.zeros(max_iter + 1)
        it, st = C.c_int(), C.c_int()
        check(lib().bmg_solve(self.h, k_pre, k_post, b.h, x.h, tol, max_iter, dptr(hist), C.byref(it),
                              C.byref(st)))
        return hist[:it.value + 1], it.value, st.value

    def measure_rates(self, mass: BlockSparseMatrix, b: Vector, u_ref: Vector, k_pre, k_post, seed=0, tol=1e-8,
                      max_iter=50) -> dict:
        """measure_rates (experiments.cpp:15-67): RateReport as a dict."""
        l2, en, rs = np.zeros(max_iter + 1), np.zeros(max_iter + 1), np.zeros(max_iter + 1)
        rates = np.zeros(3)
        it, st, bl = C.c_int(), C.c_int(), C.c_int()
        check(lib().bmg_measure_rates(self.h, mass.h, b.h, u_ref.h, k_pre, k_post, seed, tol, max_iter, dptr(l2),
                                      dptr(en), dptr(rs), C.byref(it), C.byref(st), C.byref(bl), dptr(rates)))
        n = it.value + 1
        return dict(l2_sq=l2[:n], energy_sq=en[:n], residual=rs[:n], iterations=it.value, status=st.value,
                    blowup_iteration=bl.value, rho_l2=rates[0], rho_a=rates[1], rho_r=rates[2])

    def close(self):
        if self.h:
            check(lib().bmg_hier_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dist_plan(nbr, granule, radius, world: int, agglomerate: int = 1, params: N.SetupParams | None = None):
    """bmg_dist_plan: (bounds [L, world+1], ext_lo [L, world], ext_hi [L, world], halo [L])."""
    L = len(nbr)
    n = np.ascontiguousarray(nbr, np.int32)
    g = np.ascontiguousarray(granule, np.int32)
    r = np.ascontiguousarray(radius, np.int32)
    b = np.zeros((L, world + 1), np.int32)
    lo = np.zeros((L, world), np.int32)
    hi = np.zeros((L, world), np.int32)
    ha = np.zeros(L, np.int32)
    check(lib().bmg_dist_plan(L, i32ptr(n), i32ptr(g), i32ptr(r), world, agglomerate,
                              C.byref(params) if params is not None else None, i32ptr(b), i32ptr(lo), i32ptr(hi),
                              i32ptr(ha)))
    return b, lo, hi, ha


def read_matrix(ctx: Context, path: str):
    """read_matrix (matrix_io.hpp:23) straight into a device matrix; returns (A, symmetric)."""
    h = C.c_void_p()
    sym = C.c_int()
    check(lib().bmg_io_read_matrix(ctx.h, path.encode(), C.byref(h), C.byref(sym)))
    return BlockSparseMatrix(ctx, _handle=h), bool(sym.value)


def write_matrix(a: BlockSparseMatrix, path: str):
    check(lib().bmg_io_write_matrix(a.h, path.encode()))


def read_vector(ctx: Context, path: str) -> Vector:
    h = C.c_void_p()
    check(lib().bmg_io_read_vector(ctx.h, path.encode(), C.byref(h)))
    v = Vector.__new__(Vector)
    v.ctx, v.h, v.n = ctx, h, int(lib().bmg_vec_size(h))
    return v


def write_vector(v: Vector, path: str):
    check(lib().bmg_io_write_vector(v.h, path.encode()))


def partition_rows(row_ptr, world: int, granule: int = 1, agglomerate: bool = False) -> np.ndarray:
    rp = np.ascontiguousarray(row_ptr, np.int64)
    out = np.zeros(world + 1, np.int32)
    check(lib().bmg_partition_rows(len(rp) - 1, i64ptr(rp), world, granule, 1 if agglomerate else 0, i32ptr(out)))
    return out


def row_window(row_ptr, col_idx, lo: int, hi: int, clo: int, chi: int):
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx if len(col_idx) else [0], np.int32)
    a, b = C.c_int32(), C.c_int32()
    check(lib().bmg_row_window(i64ptr(rp), i32ptr(ci), lo, hi, clo, chi, C.byref(a), C.byref(b)))
    return a.value, b.value


def tridiag_eigs(d, e) -> np.ndarray:
    d = np.ascontiguousarray(d, np.float64)
    e = np.ascontiguousarray(e, np.float64)
    out = np.zeros(len(d))
    check(lib().bmg_tridiag_eigs(len(d), dptr(d), dptr(e) if len(e) else None, dptr(out)))
    return out
