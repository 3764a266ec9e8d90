"""Synthetic BASELINE problems (BASELINE.json configs).

The generator itself is host C++ in its own library, bmggen/libbmggen.so
(bmggen/generator.cpp, include/bmg_gen.h) -- input data shared by the product
tests, both benchmark arms and the oracle fixtures; this module only sizes the
arrays and names the configs, and it loads neither libbmgcuda.so nor the oracle.  Inputs are data, not the
solver path: the reference's PUM discretiser is out of scope.
The reference's FD test problem (experiments.cpp:104-195) is restated at the end.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

import os
import sys

from .api import HostBsr
from .native import dptr, i32ptr, i64ptr

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)
from bmggen import check, lib  # noqa: E402  (the generator library, not libbmgcuda.so)


@dataclass
class Config:
    name: str
    dim: int
    n: int          # patches per direction on the finest grid
    power: int      # S_p = L_D^p
    m: int          # block size
    levels: int     # hierarchy depth (1 = single level)
    fsai: str       # "static" | "adaptive" | "nested"
    k: int          # Chebyshev degree per smoothing
    nest: int = 0
    seed: int = 0
    reg: float = 0.01
    tol: float = 1e-8
    notes: str = ""
    extra: dict = field(default_factory=dict)

    def scaled(self, n: int, levels: int | None = None) -> "Config":
        return Config(self.name + f"@{n}", self.dim, n, self.power, self.m,
                      self.levels if levels is None else levels, self.fsai, self.k, self.nest,
                      self.seed, self.reg, self.tol, self.notes)

    @property
    def unit(self) -> str:
        return "smoother applications/s" if self.levels == 1 else "V-cycles/s"


CONFIGS = {
    "C1": Config("C1", 2, 64, 2, 10, 1, "static", 3, notes="single-level smoothing, 13-pt"),
    "C2": Config("C2", 2, 256, 2, 10, 4, "adaptive", 3, notes="4-level V(3,3)"),
    "C3": Config("C3", 2, 1024, 3, 21, 5, "nested", 4, nest=1, notes="25-pt triharmonic, V(4,4)"),
    "C4": Config("C4", 3, 64, 2, 20, 4, "adaptive", 3, notes="3-D 25-pt, V(3,3)"),
    "C5": Config("C5", 2, 2048, 2, 15, 6, "adaptive", 3, notes="strong scaling, V(3,3)"),
}


def stencil_matrix(dim: int, n: int, power: int, m: int, seed: int = 0, reg: float = 0.01,
                   rows: tuple | None = None) -> HostBsr:
    """A = S_p (x) C + reg blockdiag(D_i) on an n^dim patch grid; `rows` = (lo, hi)
    restricts to those block rows (global column indices, not symmetric then)."""
    lo, hi = rows if rows is not None else (0, -1)
    nnzb = C.c_int64()
    check(lib().bmg_gen_stencil(dim, n, power, m, seed, reg, lo, hi, C.byref(nnzb), None, None, None))
    nodes = n ** dim
    nr = (hi if hi >= 0 else nodes) - lo
    rp = np.zeros(nr + 1, np.int64)
    ci = np.zeros(nnzb.value, np.int32)
    vals = np.zeros(nnzb.value * m * m)
    check(lib().bmg_gen_stencil(dim, n, power, m, seed, reg, lo, hi, C.byref(nnzb), i64ptr(rp), i32ptr(ci),
                                dptr(vals)))
    return HostBsr(np.full(nr, m, np.int32), np.full(nodes, m, np.int32), rp, ci, vals, symmetric=rows is None)


def prolongation(dim: int, n_fine: int, m: int, seed: int = 0, level: int = 1, rows: tuple | None = None) -> HostBsr:
    lo, hi = rows if rows is not None else (0, -1)
    nnzb = C.c_int64()
    check(lib().bmg_gen_prolongation(dim, n_fine, m, seed, level, lo, hi, C.byref(nnzb), None, None, None))
    nf = n_fine ** dim
    nc = (n_fine // 2) ** dim
    nr = (hi if hi >= 0 else nf) - lo
    rp = np.zeros(nr + 1, np.int64)
    ci = np.zeros(nnzb.value, np.int32)
    vals = np.zeros(nnzb.value * m * m)
    check(lib().bmg_gen_prolongation(dim, n_fine, m, seed, level, lo, hi, C.byref(nnzb), i64ptr(rp), i32ptr(ci),
                                     dptr(vals)))
    return HostBsr(np.full(nr, m, np.int32), np.full(nc, m, np.int32), rp, ci, vals, symmetric=False)


def normal_vector(n: int, seed: int = 0, tag: int = 0) -> np.ndarray:
    out = np.zeros(n)
    check(lib().bmg_gen_normal(seed, tag, n, dptr(out)))
    return out


def make_problem(cfg: Config):
    """Finest A, transfers (transfers[l-1] prolongates level l-1 -> l) and b."""
    A = stencil_matrix(cfg.dim, cfg.n, cfg.power, cfg.m, cfg.seed, cfg.reg)
    transfers = []
    for l in range(1, cfg.levels):
        n_l = cfg.n >> (cfg.levels - 1 - l)
        transfers.append(prolongation(cfg.dim, n_l, cfg.m, cfg.seed, l))
    b = normal_vector(A.dim_r, cfg.seed, 0)
    return A, transfers, b


# ---------------------------------------------------------------------------
# distributed setup inputs (bmg_hier_setup_dist): the plan's extended strips
def level_grid(cfg: Config):
    """Per level (coarsest first): block rows, granule (one grid row in 2-D, one
    plane in 3-D) and coupling radius in granules (S_p: p; Galerkin with the 2:1
    prolongation's support: floor((R + 5) / 2))."""
    L = cfg.levels
    ns = [cfg.n >> (L - 1 - l) for l in range(L)]
    nbr = [n ** cfg.dim for n in ns]
    gran = [n ** (cfg.dim - 1) for n in ns]
    rad = [0] * L
    rad[L - 1] = cfg.power
    for l in range(L - 1, 0, -1):
        rad[l - 1] = (rad[l] + 5) // 2
    return ns, nbr, gran, rad


def dist_inputs(cfg: Config, world: int, rank: int, agglomerate: int = 1, params=None):
    """(A_ext, transfers, b_own, plan) for one rank: rows [ext_lo, ext_hi) of the
    finest A and of P_l (l > agglomerate), whole P_l below; b's own rows."""
    from .api import dist_plan
    ns, nbr, gran, rad = level_grid(cfg)
    L = cfg.levels
    bounds, elo, ehi, halo = dist_plan(nbr, gran, rad, world, agglomerate, params)
    top = L - 1
    A = stencil_matrix(cfg.dim, cfg.n, cfg.power, cfg.m, cfg.seed, cfg.reg,
                       rows=(int(elo[top, rank]), int(ehi[top, rank])))
    agg = max(1, min(agglomerate, L - 1))
    transfers = []
    for l in range(1, L):
        rows = (int(elo[l, rank]), int(ehi[l, rank])) if l > agg else None
        transfers.append(prolongation(cfg.dim, ns[l], cfg.m, cfg.seed, l, rows=rows))
    b = normal_vector(nbr[top] * cfg.m, cfg.seed, 0)
    lo, hi = int(bounds[top, rank]), int(bounds[top, rank + 1])
    return A, transfers, b[lo * cfg.m:hi * cfg.m], (bounds, elo, ehi, halo, gran, rad)


# ---------------------------------------------------------------------------
# variable block layouts (the paper's PUM systems mix block sizes: boundary
# patches carry fewer functions, e.g. 6 vs 10).  Each block of the uniform
# operator is truncated to [:m_i, :m_j], i.e. A is the principal submatrix of the
# uniform S_p (x) C + reg D that keeps the first m_i functions of every patch, so
# it stays symmetric positive definite.
def boundary_sizes(dim: int, n: int, m_int: int, m_bnd: int) -> np.ndarray:
    idx = np.arange(n ** dim)
    on_bnd = np.zeros(idx.size, bool)
    for d in range(dim):
        c = (idx // n ** d) % n
        on_bnd |= (c == 0) | (c == n - 1)
    return np.where(on_bnd, m_bnd, m_int).astype(np.int32)


def truncate_blocks(h: HostBsr, row_sizes, col_sizes, symmetric=None) -> HostBsr:
    rs = np.asarray(row_sizes, np.int32)
    cs = np.asarray(col_sizes, np.int32)
    mr, mc = int(h.row_sizes[0]), int(h.col_sizes[0])
    vals = []
    for i in range(len(rs)):
        for p in range(h.row_ptr[i], h.row_ptr[i + 1]):
            j = h.col_idx[p]
            blk = h.vals[p * mr * mc:(p + 1) * mr * mc].reshape(mr, mc)
            vals.append(blk[:rs[i], :cs[j]].ravel())
    v = np.concatenate(vals) if vals else np.zeros(0)
    return HostBsr(rs, cs, h.row_ptr.copy(), h.col_idx.copy(), v,
                   h.symmetric if symmetric is None else symmetric)


def make_variable_problem(cfg: Config, m_bnd: int):
    """make_problem with boundary patches truncated to m_bnd functions on every level."""
    A, T, _ = make_problem(cfg)
    L = cfg.levels
    sizes = [boundary_sizes(cfg.dim, cfg.n >> (L - 1 - l), cfg.m, m_bnd) for l in range(L)]
    Av = truncate_blocks(A, sizes[-1], sizes[-1])
    Tv = [truncate_blocks(T[l - 1], sizes[l], sizes[l - 1], symmetric=False) for l in range(1, L)]
    b = normal_vector(int(sizes[-1].sum()), cfg.seed, 0)
    return Av, Tv, b


# ---------------------------------------------------------------------------
# the reference's finite-difference test problem (proj/src/experiments.cpp:104-195):
# the problem its own multilevel tests run on (proj/tests/test_multilevel.cpp:20-23)
@dataclass
class FdProblem:
    A: HostBsr                # 13-point biharmonic, scalar blocks
    transfers: list           # transfers[l-1]: bilinear prolongation level l-1 -> l
    b: np.ndarray             # A @ reference
    reference: np.ndarray     # samples of the manufactured field
    mass: HostBsr             # h^2 I
    h: float


def _scalar_csr(nr: int, nc: int, rows, cols, vals, symmetric: bool) -> HostBsr:
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rp = np.zeros(nr + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return HostBsr(np.ones(nr, np.int32), np.ones(nc, np.int32), np.cumsum(rp), cols, vals, symmetric)


def fd_biharmonic_matrix(ng: int) -> HostBsr:
    """13-point bilaplacian on the (ng-1)^2 interior nodes of the unit square,
    h = 1/ng, clamped boundary (experiments.cpp:110-144): Dirichlet values drop,
    the distance-2 ghost reflects onto the first interior line (+s on the
    diagonal per boundary direction).  Node (i, j) is row j*(ng-1) + i."""
    m = ng - 1
    h = 1.0 / ng
    s = 1.0 / (h * h * h * h)
    j, i = np.divmod(np.arange(m * m), m)
    rows, cols, vals = [], [], []

    def put(di, dj, w):
        i1, j1 = i + di, j + dj
        ok = (i1 >= 0) & (i1 < m) & (j1 >= 0) & (j1 < m)
        rows.append((j * m + i)[ok])
        cols.append((j1 * m + i1)[ok])
        vals.append(np.broadcast_to(w, i.shape)[ok])

    put(0, 0, 20.0 * s + s * ((i == 0) | (i == m - 1)) + s * ((j == 0) | (j == m - 1)))
    for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        put(di, dj, -8.0 * s)
        put(2 * di, 2 * dj, 1.0 * s)
    for di, dj in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
        put(di, dj, 2.0 * s)
    return _scalar_csr(m * m, m * m, np.concatenate(rows), np.concatenate(cols).astype(np.int32),
                       np.concatenate(vals).astype(np.float64), True)


def fd_prolongation(ng_fine: int) -> HostBsr:
    """Bilinear interpolation from the (ng/2 - 1)^2 coarse interior nodes to the
    (ng - 1)^2 fine ones (experiments.cpp:146-167): weight
    (1 - |i+1 - 2(ci+1)|/2)(1 - |j+1 - 2(cj+1)|/2) from the surrounding coarse nodes."""
    mf, mc = ng_fine - 1, ng_fine // 2 - 1
    j, i = np.divmod(np.arange(mf * mf), mf)
    rows, cols, vals = [], [], []
    for dcj in (-1, 0, 1):
        for dci in (-1, 0, 1):
            ci, cj = i // 2 + dci, j // 2 + dcj
            wx = 1.0 - 0.5 * np.abs(i + 1 - 2 * (ci + 1))
            wy = 1.0 - 0.5 * np.abs(j + 1 - 2 * (cj + 1))
            ok = (ci >= 0) & (ci < mc) & (cj >= 0) & (cj < mc) & (wx > 0) & (wy > 0)
            rows.append((j * mf + i)[ok])
            cols.append((cj * mc + ci)[ok])
            vals.append((wx * wy)[ok])
    return _scalar_csr(mf * mf, mc * mc, np.concatenate(rows), np.concatenate(cols).astype(np.int32),
                       np.concatenate(vals), False)


def fd_biharmonic(n_grid: int, levels: int) -> FdProblem:
    """experiments.cpp:104-195: finest grid n_grid (a power of two), `levels`
    nested grids n_grid / 2^k, manufactured field cos(2 pi x) sin(2 pi y)."""
    if levels < 1:
        raise ValueError("fd_biharmonic: need at least one level")
    if n_grid & (n_grid - 1):
        raise ValueError("fd_biharmonic: n_grid must be 2^l")
    if (n_grid >> (levels - 1)) < 4:
        raise ValueError("fd_biharmonic: grid too small for the level count")
    A = fd_biharmonic_matrix(n_grid)
    m = n_grid - 1
    h = 1.0 / n_grid
    mass = _scalar_csr(m * m, m * m, np.arange(m * m), np.arange(m * m, dtype=np.int32),
                       np.full(m * m, h * h), True)
    j, i = np.divmod(np.arange(m * m), m)
    ref = np.cos(2.0 * np.pi * (i + 1) * h) * np.sin(2.0 * np.pi * (j + 1) * h)
    b = np.zeros(m * m)
    for r in range(m * m):  # spmv: ascending columns within the row
        lo, hi = A.row_ptr[r], A.row_ptr[r + 1]
        acc = 0.0
        for p in range(lo, hi):
            acc += A.vals[p] * ref[A.col_idx[p]]
        b[r] = acc
    transfers = [fd_prolongation(n_grid >> (levels - 1 - l)) for l in range(1, levels)]
    return FdProblem(A, transfers, b, ref, mass, h)


# ---------------------------------------------------------------------------
# per-rank memory plan of the distributed setup (bmg_dist_plan strips), from the
# structure alone: no matrix is generated.  Upper bounds, printed by bench.py and
# tools/dist_memory_plan.py so a C3 / C5 run is sized before it starts.
def level_offsets(cfg: Config):
    """Per level (coarsest first) the block-column offsets an interior row of A_l
    holds: S_p = L_D^p couples offsets with |o|_1 <= p; Galerkin P^T A P (P row i:
    parents(i) + {-1,0,1}^d) maps a fine offset o of a child with parity x to
    floor((x + o) / 2) + {-2..2}^d on the coarse grid.  Rows near the boundary hold
    the subset that stays on the grid (or fewer): the counts are upper bounds."""
    import itertools
    d = cfg.dim
    rng = range(-cfg.power, cfg.power + 1)
    fine = {o for o in itertools.product(rng, repeat=d) if sum(abs(v) for v in o) <= cfg.power}
    sets = [fine]
    for _ in range(cfg.levels - 1):
        cur = sets[-1]
        base = {tuple((x[k] + o[k]) // 2 for k in range(d)) for o in cur for x in itertools.product((0, 1), repeat=d)}
        nxt = {tuple(b[k] + e[k] for k in range(d)) for b in base for e in itertools.product(range(-2, 3), repeat=d)}
        sets.append(nxt)
    return sets[::-1]


def _count_rows(offsets, n, dim, lo_g, hi_g):
    """sum over grid rows with outermost index in [lo_g, hi_g) of the offsets that
    stay on the n^dim grid"""
    tot = 0
    for o in offsets:
        inner = 1
        for k in range(dim - 1):
            inner *= max(0, n - abs(o[k]))
        oz = o[dim - 1]
        lo, hi = max(lo_g, -oz, 0), min(hi_g, n - oz, n)
        tot += inner * max(0, hi - lo)
    return tot


def memory_plan(cfg: Config, world: int, agglomerate: int = 1, params=None):
    """Per-rank device bytes (upper bounds) of the partitioned hierarchy built by
    bmg_hier_setup_dist: own rows of A_l (padded 16-byte blocks + int32 column),
    the FSAI chain and its transposes (t_max = 1: <= 2 blocks per row per factor),
    P_l / R_l, six work vectors over the extended window, and on rank 0 the
    agglomerated levels plus the packed coarse inverse; `peak` adds the setup's
    transient extended strip of A and the 4 GB Galerkin chunk.  Returns a list of
    dicts (one per rank) in GB."""
    from .api import dist_plan
    ns, nbr, gran, rad = level_grid(cfg)
    L = cfg.levels
    offs = level_offsets(cfg)
    bounds, elo, ehi, _ = dist_plan(nbr, gran, rad, world, agglomerate, params)
    m, d = cfg.m, cfg.dim
    blk = 8 * (m * m + (m * m) % 2) + 4
    nfac = 2 * (cfg.nest + 1)  # forward factors and their transposes
    agg = max(1, min(agglomerate, L - 1))
    out = []
    for r in range(world):
        steady = peak_extra = half_extra = 0
        for l in range(L):
            n = ns[l]
            whole = l < agg
            if whole and r != 0:
                continue
            lo, hi = (0, nbr[l]) if whole else (int(bounds[l, r]), int(bounds[l, r + 1]))
            elo_, ehi_ = (0, nbr[l]) if whole else (int(elo[l, r]), int(ehi[l, r]))
            g = gran[l]
            if l == 0:  # dense coarse level: packed lower 64x64 tiles of the inverse
                n0 = nbr[0] * m
                nt = (n0 + 63) // 64
                steady += nt * (nt + 1) // 2 * 64 * 64 * 8 + nt * nt * 64 * 8
                peak_extra = max(peak_extra, 8 * n0 * n0 - nt * (nt + 1) // 2 * 64 * 64 * 8)
                continue
            a_own = _count_rows(offs[l], n, d, lo // g, -(-hi // g)) * blk
            a_ext = _count_rows(offs[l], n, d, elo_ // g, -(-ehi_ // g)) * blk
            if not whole and m >= 15 and _count_rows(offs[l], n, d, 0, n) * blk >= 3e9:
                # the half form of A beside the full one (hierarchy.cu build_level_psym;
                # built only where it fits, else the level keeps full storage)
                half_extra += a_own // 2 + (hi - lo) * m * 8 * (len(offs[l]) // 2 + 2)
            steady += a_own + nfac * 2 * (hi - lo) * blk
            steady += 2 * (hi - lo) * 3 ** d * blk          # P_l rows and their share of R_l
            steady += 6 * (ehi_ - elo_) * m * 8             # work vectors over the window
            peak_extra = max(peak_extra, a_ext + (4 << 30))
        out.append({"rank": r, "steady_gb": steady / 1e9, "peak_gb": (steady + peak_extra) / 1e9,
                    "half_storage_gb": half_extra / 1e9})
    return out
