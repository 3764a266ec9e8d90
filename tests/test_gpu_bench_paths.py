"""bench.py's own code paths on one GPU: the CPU legs' byte model against the
device's, and the N > 1 branch (distributed setup + partition-invariance check)
through the loopback transport -- each rank a host thread with its own context,
the same Comm calls NCCL serves on a multi-GPU node."""
import os
import threading

import numpy as np
import pytest

import bench
from oracle import pyoracle as O
from paper_2509_06744_b200 import Context, LoopbackGroup, Vector
from paper_2509_06744_b200 import problems as pr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n,levels", [("C4", 16, 4), ("C3", 64, 4), ("C5", 64, 5)])
def test_cycle_bytes_model_matches_device(ctx, name, n, levels):
    # the CPU legs scale a sample's rate by the algorithmic bytes of bench.cycle_bytes_model
    cfg = pr.CONFIGS[name].scaled(n, levels)
    H, _ = bench.whole_hierarchy(ctx, cfg)
    A, T, _ = pr.make_problem(cfg)
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, nest=cfg.nest, coarse_dim_cap=1 << 30, probe=False)
    n0 = oh.A(0).info()["dim_r"]
    model = bench.cycle_bytes_model(bench.oracle_levels(oh, cfg.m), cfg.k, cfg.k, n0)
    assert model == H.cycle_bytes_ref(cfg.k, cfg.k)


def _loopback(world, fn):
    group = LoopbackGroup(world)
    out, errs = [None] * world, []
    bar = threading.Barrier(world)
    vals = [0] * world

    def all_min(v, r):
        vals[r] = v
        bar.wait()
        res = min(vals)
        bar.wait()
        return res

    def body(r):
        try:
            c = Context(0, loopback=(group, r))
            out[r] = fn(c, r, lambda v: all_min(v, r))
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))
            bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not any(t.is_alive() for t in th), "rank thread hung"
    if errs:
        raise errs[0][1]
    return out


def test_bench_distributed_branch_c5_shape_world4(ctx):
    # the exact N > 1 branch of bench.run_ours at C5's shape (m = 15, 6 levels, the
    # coarsest two agglomerated on rank 0): invariance check, distributed setup from
    # each rank's strips, solve -- residual history and iterate bitwise the 1-GPU ones
    cfg = pr.CONFIGS["C5"].scaled(256)
    world, agg = 4, bench.AGGLOMERATE["C5"]
    assert agg == 2
    H1, b = bench.whole_hierarchy(ctx, cfg)
    H1.partition(1, pr.level_grid(cfg)[2])  # the N-rank residual-norm segmentation
    x1 = Vector(ctx, b.size)
    hist1, it1, _ = H1.solve(cfg.k, cfg.k, Vector(ctx, b), x1, 1e-8, 8)
    xref = x1.download()

    def rank(c, r, all_min):
        assert bench.invariance_check(c, cfg.scaled(128), world, r, agg, all_min)
        H, b_own = bench.partitioned_hierarchy(c, cfg, world, r, agg)
        if os.environ.get("BMG_SYM_HALF") == "1":  # (test_gpu_sym_partitioned.py) the half form is on
            assert H.cycle_bytes(cfg.k, cfg.k) < H.cycle_bytes_ref(cfg.k, cfg.k)
        x = Vector(c, b_own.size)
        hist, it, _ = H.solve(cfg.k, cfg.k, Vector(c, b_own), x, 1e-8, 8)
        lo = H.part_info(cfg.levels - 1, r)[0]
        return lo, x.download(), hist, it

    outs = _loopback(world, rank)
    for lo, x, hist, it in outs:
        assert it == it1 and np.array_equal(hist, hist1)
        assert np.array_equal(x, xref[lo * cfg.m:lo * cfg.m + x.size])
    assert sum(o[1].size for o in outs) == b.size


def test_memory_plan_matches_device_bytes_order(ctx):
    # the plan's steady per-rank bytes bound what the distributed hierarchy holds
    cfg = pr.CONFIGS["C5"].scaled(256)
    world, agg = 2, 2
    plan = pr.memory_plan(cfg, world, agg)

    def rank(c, r, all_min):
        H, _ = bench.partitioned_hierarchy(c, cfg, world, r, agg)
        return H.device_bytes / 1e9

    got = _loopback(world, rank)
    for r in range(world):
        assert got[r] <= plan[r]["steady_gb"], (r, got[r], plan[r])
