"""Size-independent properties at the headline size (BASELINE C2: 256^2 patches,
m = 10, 4 levels, V(3,3)): fixed point, linearity, A-self-adjointness, and the
bitwise identities between execution modes (graph / eager, host / device,
partitioned / whole, batched / single, distributed / single-device setup)."""
import numpy as np
import pytest

from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy, Vector, default_params, spmv
from paper_2509_06744_b200 import problems as pr

pytestmark = pytest.mark.gpu

CFG = pr.CONFIGS["C2"]


@pytest.fixture(scope="module")
def c2(ctx):
    A, T, b = pr.make_problem(CFG)
    params = default_params(t_max=1, coarse_dim_cap=1 << 30)
    dA = BlockSparseMatrix(ctx, A)
    dT = [BlockSparseMatrix(ctx, p) for p in T]
    h = Hierarchy.setup(dA, dT, params)
    h.partition(1, pr.level_grid(CFG)[2])
    return dict(A=A, T=T, b=b, dA=dA, dT=dT, h=h, params=params)


def _cycle(ctx, h, b, x0, n=1):
    x = Vector(ctx, x0.copy())
    bv = Vector(ctx, b)
    for _ in range(n):
        h.v_cycle(3, 3, bv, x)
    return x.download()


def test_fixed_point_and_linearity(ctx, c2, rng):
    h, n = c2["h"], c2["b"].size
    assert np.array_equal(_cycle(ctx, h, np.zeros(n), np.zeros(n)), np.zeros(n))
    b1, b2 = rng.standard_normal(n), rng.standard_normal(n)
    lhs = _cycle(ctx, h, 0.5 * b1 - 2.0 * b2, np.zeros(n))
    rhs = 0.5 * _cycle(ctx, h, b1, np.zeros(n)) - 2.0 * _cycle(ctx, h, b2, np.zeros(n))
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_cycle_is_A_self_adjoint(ctx, c2, rng):
    h, dA, n = c2["h"], c2["dA"], c2["b"].size
    e1, e2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    z = np.zeros(n)
    ce1, ce2 = _cycle(ctx, h, z, e1), _cycle(ctx, h, z, e2)

    def Av(v):
        y = Vector(ctx, n)
        spmv(dA, Vector(ctx, v), y)
        return y.download()

    lhs, rhs = Av(ce1) @ e2, Av(ce2) @ e1
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), 1.0)


def test_execution_modes_are_bitwise_identical(ctx, c2, rng):
    h, b = c2["h"], c2["b"]
    n = b.size
    x0 = rng.standard_normal(n)
    ref = _cycle(ctx, h, b, x0, 2)
    # eager launch (no graph)
    h.use_graph(False)
    eager = _cycle(ctx, h, b, x0, 2)
    h.use_graph(True)
    assert np.array_equal(eager, ref)
    # host buffers through the C ABI
    xh = x0.copy()
    for _ in range(2):
        h.v_cycle_host(3, 3, b.copy(), xh)
    assert np.array_equal(xh, ref)
    # 8 right-hand sides per cycle
    K = 8
    B = np.stack([b] * K, axis=1).ravel().copy()
    X = np.stack([x0] * K, axis=1).ravel().copy()
    xb = Vector(ctx, X)
    for _ in range(2):
        h.v_cycle_batch(3, 3, K, Vector(ctx, B), xb)
    assert all(np.array_equal(col, ref) for col in xb.download().reshape(-1, K).T)


def test_partitioned_and_distributed_equal_single_device(ctx, c2, rng):
    b, params = c2["b"], c2["params"]
    n = b.size
    x0 = rng.standard_normal(n)
    ref = _cycle(ctx, c2["h"], b, x0, 2)
    _, _, gran, rad = pr.level_grid(CFG)
    hp = Hierarchy.setup(c2["dA"], c2["dT"], params)
    hp.partition(4, gran, agglomerate=1)
    assert np.array_equal(_cycle(ctx, hp, b, x0, 2), ref)
    del hp
    a_ext, trans = [], []
    for r in range(2):
        A, T, _, _ = pr.dist_inputs(CFG, 2, r, 1, params)
        a_ext.append(BlockSparseMatrix(ctx, A))
        trans.append([BlockSparseMatrix(ctx, p) for p in T])
    hd = Hierarchy.setup_dist_emulated(ctx, a_ext, trans, gran, rad, 1, params)
    for l in range(1, CFG.levels):
        assert hd.beta(l) == c2["h"].beta(l)
    assert np.array_equal(_cycle(ctx, hd, b, x0, 2), ref)
