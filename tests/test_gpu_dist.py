"""Distributed setup (bmg_hier_setup_dist*): every rank builds
only an extended strip of each partitioned level, yet the resulting hierarchy is
bitwise the single-device one -- same beta per level (distributed Lanczos), same
V-cycle iterates, same residual histories.  Ranks are emulated in-process."""
import numpy as np
import pytest

from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy, Vector, default_params
from paper_2509_06744_b200 import problems as pr
from paper_2509_06744_b200.native import FSAI_ADAPTIVE, FSAI_STATIC_LOWER

pytestmark = pytest.mark.gpu

CASES = {
    # name: (dim, n, power, m, levels, nest, t_max, fsai_kind)
    "c2_like": (2, 32, 2, 4, 4, 0, 1, FSAI_ADAPTIVE),
    "c3_like_nested": (2, 64, 3, 3, 4, 1, 1, FSAI_ADAPTIVE),
    "c4_like_3d": (3, 16, 2, 3, 3, 0, 1, FSAI_ADAPTIVE),
    "tmax2": (2, 32, 2, 3, 3, 0, 2, FSAI_ADAPTIVE),
    "static": (2, 32, 2, 3, 3, 0, 1, FSAI_STATIC_LOWER),
    # streamed block sizes (the BASELINE shapes)
    "c2_m10": (2, 32, 2, 10, 3, 0, 1, FSAI_ADAPTIVE),
    "c5_m15": (2, 32, 2, 15, 3, 0, 1, FSAI_ADAPTIVE),
    "c3_m21_nested": (2, 64, 3, 21, 3, 1, 1, FSAI_ADAPTIVE),
}


def _cfg(name):
    dim, n, power, m, levels, nest, t_max, kind = CASES[name]
    cfg = pr.Config(name, dim, n, power, m, levels, "adaptive", 3, nest=nest)
    params = default_params(t_max=t_max, nest=nest, fsai_kind=kind, coarse_dim_cap=1 << 30)
    return cfg, params


def _whole(ctx, cfg, params):
    A, T, b = pr.make_problem(cfg)
    h = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T], params)
    _, _, gran, _ = pr.level_grid(cfg)
    h.partition(1, gran)  # residual norms segmented per granule, as in the strips
    return h, b


def _dist(ctx, cfg, params, world, agg):
    a_ext, trans = [], []
    for r in range(world):
        A, T, _, plan = pr.dist_inputs(cfg, world, r, agg, params)
        a_ext.append(BlockSparseMatrix(ctx, A))
        trans.append([BlockSparseMatrix(ctx, p) for p in T])
    _, _, gran, rad = pr.level_grid(cfg)
    h = Hierarchy.setup_dist_emulated(ctx, a_ext, trans, gran, rad, agg, params)
    return h, plan


@pytest.mark.parametrize("name,world,agg", [
    ("c2_like", 2, 1), ("c2_like", 3, 2), ("c2_like", 4, 1),
    ("c3_like_nested", 2, 1), ("c4_like_3d", 2, 1), ("c4_like_3d", 3, 2),
    ("tmax2", 2, 1), ("static", 3, 1),
    ("c2_m10", 4, 1), ("c5_m15", 2, 2), ("c3_m21_nested", 2, 1),
])
def test_dist_setup_bitwise_equal_to_single_device(ctx, name, world, agg):
    cfg, params = _cfg(name)
    hw, b = _whole(ctx, cfg, params)
    hd, plan = _dist(ctx, cfg, params, world, agg)
    bounds = plan[0]
    for l in range(cfg.levels):
        for r in range(world):
            assert hd.part_info(l, r)[:2] == (bounds[l, r], bounds[l, r + 1])
    for l in range(1, cfg.levels):
        assert hw.beta(l) == hd.beta(l), f"beta level {l}"
    bv = Vector(ctx, b)
    x1, x2 = Vector(ctx, b.size), Vector(ctx, b.size)
    for _ in range(2):
        hw.v_cycle(3, 3, bv, x1)
        hd.v_cycle(3, 3, bv, x2)
        assert np.array_equal(x1.download(), x2.download())
    x1, x2 = Vector(ctx, b.size), Vector(ctx, b.size)
    h1, i1, _ = hw.solve(3, 3, bv, x1, 1e-8, 5)
    h2, i2, _ = hd.solve(3, 3, bv, x2, 1e-8, 5)
    assert i1 == i2 and np.array_equal(h1, h2)
    assert hw.cycle_bytes_ref(3, 3) == hd.cycle_bytes_ref(3, 3)


def test_dist_setup_world1_plain_context(ctx):
    cfg, params = _cfg("c2_like")
    hw, b = _whole(ctx, cfg, params)
    A, T, b_own, plan = pr.dist_inputs(cfg, 1, 0, 1, params)
    _, _, gran, rad = pr.level_grid(cfg)
    hd = Hierarchy.setup_dist(ctx, BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T], gran, rad, 1,
                              params)
    bv = Vector(ctx, b)
    x1, x2 = Vector(ctx, b.size), Vector(ctx, b.size)
    h1, i1, _ = hw.solve(3, 3, bv, x1, 1e-8, 4)
    h2, i2, _ = hd.solve(3, 3, bv, x2, 1e-8, 4)
    assert i1 == i2 and np.array_equal(h1, h2)
    assert np.array_equal(x1.download(), x2.download())


def test_dist_setup_world1_over_real_nccl():
    """One GPU is enough for a world of one: the context's transport is the real
    NcclComm (ncclGetUniqueId and ncclCommInitRank called from libbmgcuda.so,
    ncclAllReduce in the distributed Lanczos and the residual norms, captured
    V-cycle graphs with a capturable transport).  Bitwise the plain context."""
    from paper_2509_06744_b200 import Context

    cfg, params = _cfg("c5_m15")
    uid = Context.nccl_unique_id()
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128
    nctx = Context(0, nccl=(0, 1, uid))
    pctx = Context(0)
    hw, b = _whole(pctx, cfg, params)
    A, T, b_own, plan = pr.dist_inputs(cfg, 1, 0, 1, params)
    _, _, gran, rad = pr.level_grid(cfg)
    hd = Hierarchy.setup_dist(nctx, BlockSparseMatrix(nctx, A), [BlockSparseMatrix(nctx, p) for p in T], gran, rad, 1,
                              params)
    for l in range(1, cfg.levels):
        assert hw.beta(l) == hd.beta(l)
    x1, x2 = Vector(pctx, b.size), Vector(nctx, b.size)
    h1, i1, _ = hw.solve(3, 3, Vector(pctx, b), x1, 1e-8, 5)
    h2, i2, _ = hd.solve(3, 3, Vector(nctx, b), x2, 1e-8, 5)
    assert i1 == i2 and np.array_equal(h1, h2)
    assert np.array_equal(x1.download(), x2.download())


def test_nccl_point_to_point_pattern_in_a_captured_graph():
    """The exchange pattern of the partitioned cycle (grouped ncclSend / ncclRecv on a
    forked stream, inside a captured graph, replayed) over the real NCCL transport,
    this rank being its own peer -- what one GPU can drive of the multi-GPU path."""
    from paper_2509_06744_b200 import Context

    nctx = Context(0, nccl=(0, 1, Context.nccl_unique_id()))
    for count in (1, 4096, 1 << 20):
        assert nctx.transport_selftest(count, 3) == 0


def test_dist_setup_rejects_underestimated_radius(ctx):
    cfg, params = _cfg("c2_like")
    A, T, _, _ = pr.dist_inputs(cfg, 1, 0, 1, params)
    _, _, gran, rad = pr.level_grid(cfg)
    bad = list(rad)
    bad[-1] = 1  # S_2 couples grid rows 2 apart
    from paper_2509_06744_b200.native import InvalidArgument
    with pytest.raises(InvalidArgument, match="radius"):
        Hierarchy.setup_dist(ctx, BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T], gran, bad, 1,
                             params)


def test_dist_setup_batched_cycles_and_whole_only_apis(ctx):
    # a distributed-setup hierarchy runs batched cycles bitwise like the single-device
    # one; whole-only entry points refuse it cleanly
    from paper_2509_06744_b200.native import InvalidArgument
    cfg, params = _cfg("c2_like")
    hw, b = _whole(ctx, cfg, params)
    hd, _ = _dist(ctx, cfg, params, 3, 1)
    K = 4
    B = np.stack([np.roll(b, 3 * v) for v in range(K)], axis=1).ravel().copy()
    x1, x2 = Vector(ctx, B.size), Vector(ctx, B.size)
    for _ in range(2):
        hw.v_cycle_batch(3, 3, K, Vector(ctx, B), x1)
        hd.v_cycle_batch(3, 3, K, Vector(ctx, B), x2)
    assert np.array_equal(x1.download(), x2.download())
    with pytest.raises(InvalidArgument):
        hd.v_cycle_level(3, 3, 1, Vector(ctx, 16), Vector(ctx, 16))
    with pytest.raises(InvalidArgument):
        hd.measure_rates(BlockSparseMatrix(ctx, pr.stencil_matrix(2, 32, 2, 4)), Vector(ctx, b), Vector(ctx, b), 3, 3)
