"""The NCCL code path of the partitioned cycle and of the distributed setup,
run with the loopback transport (bmg_ctx_create_loopback): each rank is a host
thread with its own context on the one GPU; sends/receives/all-reduces go through
the same Comm calls NCCL serves on a multi-GPU node.  Results must be bitwise the
single-device ones."""
import threading

import numpy as np
import pytest

from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, LoopbackGroup, Vector, default_params
from paper_2509_06744_b200 import problems as pr

pytestmark = pytest.mark.gpu


def _run_ranks(world, fn):
    group = LoopbackGroup(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            ctx = Context(0, loopback=(group, r))
            out[r] = fn(ctx, r)
        except Exception as e:  # noqa: BLE001 - surfaced below
            errs.append((r, e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "rank thread hung"
    if errs:
        raise errs[0][1]
    return out


def _reference(ctx, cfg, params, cycles=2, iters=5):
    A, T, b = pr.make_problem(cfg)
    h = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T], params)
    h.partition(1, pr.level_grid(cfg)[2])
    bv = Vector(ctx, b)
    x = Vector(ctx, b.size)
    xs = []
    for _ in range(cycles):
        h.v_cycle(3, 3, bv, x)
        xs.append(x.download())
    x2 = Vector(ctx, b.size)
    hist, it, _ = h.solve(3, 3, bv, x2, 1e-8, iters)
    return A, T, b, xs, hist, it, x2.download()


def _rank_cycles(h, ctx, b_own, cycles=2, iters=5):
    bv = Vector(ctx, b_own)
    x = Vector(ctx, b_own.size)
    xs = []
    for _ in range(cycles):
        h.v_cycle(3, 3, bv, x)
        xs.append(x.download())
    x2 = Vector(ctx, b_own.size)
    hist, it, _ = h.solve(3, 3, bv, x2, 1e-8, iters)
    return xs, hist, it, x2.download()


def _check(ref, outs, world, cycles=2):
    _, _, _, xs, hist, it, xsol = ref
    for c in range(cycles):
        assert np.array_equal(np.concatenate([o[0][c] for o in outs]), xs[c]), f"cycle {c}"
    for o in outs:
        assert o[2] == it and np.array_equal(o[1], hist)
    assert np.array_equal(np.concatenate([o[3] for o in outs]), xsol)


@pytest.mark.parametrize("world,agg", [(2, 1), (3, 2), (4, 1)])
def test_partitioned_cycle_through_transport(ctx, world, agg):
    cfg = pr.CONFIGS["C2"].scaled(32, 3)
    params = default_params(t_max=1, coarse_dim_cap=1 << 30)
    ref = _reference(ctx, cfg, params)
    A, T, b = ref[0], ref[1], ref[2]
    gran = pr.level_grid(cfg)[2]

    def rank(c, r):
        h = Hierarchy.setup(BlockSparseMatrix(c, A), [BlockSparseMatrix(c, p) for p in T], params)
        h.partition(world, gran, agglomerate=agg, rank=r)
        lo, hi = h.part_info(cfg.levels - 1, r)[:2]
        return _rank_cycles(h, c, b[lo * cfg.m:hi * cfg.m])

    _check(ref, _run_ranks(world, rank), world)


@pytest.mark.parametrize("name,world,agg", [("c2", 2, 1), ("c2", 3, 2), ("nested", 2, 1), ("3d", 3, 1)])
def test_distributed_setup_through_transport(ctx, name, world, agg):
    dim, n, power, m, levels, nest = {"c2": (2, 32, 2, 4, 4, 0), "nested": (2, 64, 3, 3, 4, 1),
                                      "3d": (3, 16, 2, 3, 3, 0)}[name]
    cfg = pr.Config(name, dim, n, power, m, levels, "adaptive", 3, nest=nest)
    params = default_params(t_max=1, nest=nest, coarse_dim_cap=1 << 30)
    ref = _reference(ctx, cfg, params)
    _, _, gran, rad = pr.level_grid(cfg)

    def rank(c, r):
        A, T, b_own, _ = pr.dist_inputs(cfg, world, r, agg, params)
        h = Hierarchy.setup_dist(c, BlockSparseMatrix(c, A), [BlockSparseMatrix(c, p) for p in T], gran, rad, agg,
                                 params)
        return _rank_cycles(h, c, b_own)

    _check(ref, _run_ranks(world, rank), world)


def test_distributed_setup_failure_on_one_rank_fails_all(ctx):
    # rank 1 passes a strip that does not match the plan: it fails in its own phase,
    # rank 0 must not block in the following row exchange but fail as well
    import time
    cfg = pr.Config("c2", 2, 32, 2, 4, 3, "adaptive", 3)
    params = default_params(t_max=1, coarse_dim_cap=1 << 30)
    _, _, gran, rad = pr.level_grid(cfg)
    world = 2
    group = LoopbackGroup(world)
    errs = [None] * world

    def body(r):
        try:
            c = Context(0, loopback=(group, r))
            A, T, _, _ = pr.dist_inputs(cfg, world, r, 1, params)
            if r == 1:
                A, _, _, _ = pr.dist_inputs(cfg, world, 0, 1, params)  # rank 0's strip: wrong rows
            Hierarchy.setup_dist(c, BlockSparseMatrix(c, A), [BlockSparseMatrix(c, p) for p in T], gran, rad, 1,
                                 params)
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    t0 = time.time()
    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th)
    assert time.time() - t0 < 100  # no transport timeout involved
    assert errs[1] is not None and "dist setup" in str(errs[1])
    assert errs[0] is not None and "another rank failed" in str(errs[0])
