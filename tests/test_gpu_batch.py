"""Batched right-hand sides (bmg_vcycle_batch): K interleaved RHS share one
stream of every matrix; each RHS must be bitwise the single-vector cycle (the
reference allows concurrent v_cycle calls on distinct RHS)."""
import threading

import numpy as np
import pytest

from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, LoopbackGroup, Vector, default_params
from paper_2509_06744_b200 import problems as pr

pytestmark = pytest.mark.gpu


def _hier(ctx, cfg, variable=False):
    if variable:
        A, T, b = pr.make_variable_problem(cfg, 6)
    else:
        A, T, b = pr.make_problem(cfg)
    h = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                        default_params(t_max=1, nest=cfg.nest, coarse_dim_cap=1 << 30))
    return h, A, T, b


def _rhs(n, K, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, K)), rng.standard_normal((n, K))


def _single(ctx, h, B, X, cycles):
    out = []
    for v in range(B.shape[1]):
        bv, xv = Vector(ctx, B[:, v].copy()), Vector(ctx, X[:, v].copy())
        for _ in range(cycles):
            h.v_cycle(3, 3, bv, xv)
        out.append(xv.download())
    return np.stack(out, axis=1)


def _batched(ctx, h, B, X, cycles):
    K = B.shape[1]
    bv, xv = Vector(ctx, B.ravel().copy()), Vector(ctx, X.ravel().copy())
    for _ in range(cycles):
        h.v_cycle_batch(3, 3, K, bv, xv)
    return xv.download().reshape(-1, K)


@pytest.mark.parametrize("name,K", [("2d_m10", 2), ("2d_m10", 4), ("2d_m10", 8), ("3d_m20", 4), ("2d_m15", 8),
                                    ("2d_m21_nested", 2), ("var", 4), ("small_m4", 8)])
def test_batched_cycle_equals_single_cycles(ctx, name, K):
    cfg = {"2d_m10": pr.CONFIGS["C2"].scaled(32, 3),
           "3d_m20": pr.CONFIGS["C4"].scaled(8, 3),
           "2d_m15": pr.CONFIGS["C5"].scaled(32, 3),
           "2d_m21_nested": pr.CONFIGS["C3"].scaled(16, 2),
           "var": pr.Config("var", 2, 16, 2, 10, 3, "adaptive", 3),
           "small_m4": pr.Config("m4", 2, 16, 2, 4, 3, "adaptive", 3)}[name]
    h, A, T, b = _hier(ctx, cfg, variable=name == "var")
    B, X = _rhs(b.size, K, 7)
    want = _single(ctx, h, B, X, 2)
    got = _batched(ctx, h, B, X, 2)
    assert np.array_equal(got, want)


def test_batch_size_switching_and_host_api(ctx):
    cfg = pr.CONFIGS["C2"].scaled(32, 3)
    h, A, T, b = _hier(ctx, cfg)
    B8, X8 = _rhs(b.size, 8, 3)
    want8 = _single(ctx, h, B8, X8, 1)
    assert np.array_equal(_batched(ctx, h, B8[:, :4], X8[:, :4], 1), want8[:, :4])
    x1 = Vector(ctx, X8[:, 5].copy())
    h.v_cycle(3, 3, Vector(ctx, B8[:, 5].copy()), x1)  # back to K = 1
    assert np.array_equal(x1.download(), want8[:, 5])
    xb = X8.ravel().copy()
    h.v_cycle_batch_host(3, 3, 8, B8.ravel().copy(), xb)
    assert np.array_equal(xb.reshape(-1, 8), want8)
    # byte model: matrices once, vectors per RHS
    c1, c8 = h.cycle_bytes(3, 3), h.cycle_bytes(3, 3, 8)
    assert c1 < c8 < 8 * c1


@pytest.mark.parametrize("world", [2, 3])
def test_batched_partitioned_emulated(ctx, world):
    cfg = pr.CONFIGS["C2"].scaled(32, 3)
    h1, A, T, b = _hier(ctx, cfg)
    h2, _, _, _ = _hier(ctx, cfg)
    h2.partition(world, pr.level_grid(cfg)[2], agglomerate=1)
    B, X = _rhs(b.size, 4, 11)
    assert np.array_equal(_batched(ctx, h2, B, X, 2), _batched(ctx, h1, B, X, 2))


def test_batched_partitioned_loopback(ctx):
    cfg = pr.CONFIGS["C2"].scaled(32, 3)
    h1, A, T, b = _hier(ctx, cfg)
    K, world = 4, 2
    B, X = _rhs(b.size, K, 5)
    want = _batched(ctx, h1, B, X, 2)
    gran = pr.level_grid(cfg)[2]
    group = LoopbackGroup(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            c = Context(0, loopback=(group, r))
            h = Hierarchy.setup(BlockSparseMatrix(c, A), [BlockSparseMatrix(c, p) for p in T],
                                default_params(t_max=1, coarse_dim_cap=1 << 30))
            h.partition(world, gran, agglomerate=1, rank=r)
            lo, hi = h.part_info(cfg.levels - 1, r)[:2]
            rows = slice(lo * cfg.m, hi * cfg.m)
            out[r] = _batched(c, h, B[rows], X[rows], 2)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    assert np.array_equal(np.concatenate(out), want)


@pytest.mark.parametrize("kpre,kpost", [(0, 4), (5, 0), (1, 2)])
def test_batched_asymmetric_cycles(ctx, kpre, kpost):
    cfg = pr.CONFIGS["C2"].scaled(32, 3)
    h, A, T, b = _hier(ctx, cfg)
    B, X = _rhs(b.size, 4, 9)
    want = []
    for v in range(4):
        xv = Vector(ctx, X[:, v].copy())
        h.v_cycle(kpre, kpost, Vector(ctx, B[:, v].copy()), xv)
        want.append(xv.download())
    bv, xv = Vector(ctx, B.ravel().copy()), Vector(ctx, X.ravel().copy())
    h.v_cycle_batch(kpre, kpost, 4, bv, xv)
    assert np.array_equal(xv.download().reshape(-1, 4), np.stack(want, axis=1))


def test_batch_rejects_bad_sizes(ctx):
    from paper_2509_06744_b200.native import InvalidArgument
    cfg = pr.CONFIGS["C2"].scaled(16, 2)
    h, A, T, b = _hier(ctx, cfg)
    with pytest.raises(InvalidArgument):
        h.v_cycle_batch(3, 3, 3, Vector(ctx, b.size * 3), Vector(ctx, b.size * 3))
    with pytest.raises(InvalidArgument):
        h.v_cycle_batch(3, 3, 4, Vector(ctx, b.size * 2), Vector(ctx, b.size * 2))
    with pytest.raises(InvalidArgument):
        h.v_cycle_batch(0, 0, 2, Vector(ctx, b.size * 2), Vector(ctx, b.size * 2))


def test_host_buffer_cycles_after_batch_sizes_change(ctx):
    # the host-buffer staging grows with K; graphs captured with the old
    # staging buffers must not be replayed.  Sequence: device batch K = 4, host
    # single (pinned, captured graph), host batch K = 2 (grows the staging), host
    # single again -- every result equal to the device-vector cycles.
    import torch

    h, A, T, b = _hier(ctx, pr.CONFIGS["C2"].scaled(32, 3))
    n = b.size
    B4, X4 = _rhs(n, 4, 7)
    got4 = _batched(ctx, h, B4, X4, 1)
    assert np.array_equal(got4, _single(ctx, h, B4, X4, 1))

    hb = torch.from_numpy(b.copy()).pin_memory()  # the same pinned buffers every call:
    hx = torch.zeros(n, dtype=torch.float64).pin_memory()  # the captured graph is reused

    def host_single(x0):
        hx.numpy()[:] = x0
        h.v_cycle_host_ptr(3, 3, hb.data_ptr(), hx.data_ptr())
        return hx.numpy().copy()

    x0 = np.random.default_rng(3).standard_normal(n)
    want = _single(ctx, h, b[:, None], x0[:, None], 1)[:, 0]
    assert np.array_equal(host_single(x0), want)
    B2, X2 = _rhs(n, 2, 9)
    xb = X2.ravel().copy()
    h.v_cycle_batch_host(3, 3, 2, B2.ravel().copy(), xb)
    assert np.array_equal(xb.reshape(n, 2), _single(ctx, h, B2, X2, 1))
    for _ in range(2):
        assert np.array_equal(host_single(x0), want)
