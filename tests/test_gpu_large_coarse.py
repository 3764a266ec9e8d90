"""The dense coarse solve beyond 2^31 matrix elements (N0^2 > 2^31: C3's and
C5's coarsest levels are N0 = 86016 / 61440): a single-level hierarchy is a pure
coarse solve, x = A^-1 b; its residual must be at the rounding level."""
import numpy as np
import pytest

from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy, Vector, default_params, residual
from paper_2509_06744_b200 import problems as pr

pytestmark = pytest.mark.gpu


def test_coarse_solve_above_2_31_elements(ctx):
    host = pr.stencil_matrix(2, 71, 2, 10)  # 5041 blocks, N0 = 50410, N0^2 = 2.54e9
    assert host.dim_r ** 2 > 2 ** 31
    A = BlockSparseMatrix(ctx, host)
    h = Hierarchy.setup(A, [], default_params(t_max=1, coarse_dim_cap=1 << 30))
    b = pr.normal_vector(host.dim_r, 0, 0)
    x = Vector(ctx, host.dim_r)
    bv = Vector(ctx, b)
    h.v_cycle(1, 1, bv, x)
    r = Vector(ctx, host.dim_r)
    residual(A, bv, x, r)
    rel = np.linalg.norm(r.download()) / np.linalg.norm(b)
    assert rel < 1e-8, rel


@pytest.mark.parametrize("m", [15, 21])
def test_coarse_solve_at_the_c5_and_c3_coarse_sizes(ctx, m):
    # the coarsest levels of C5 (64^2 patches, m = 15: N0 = 61,440) and C3 (64^2,
    # m = 21: N0 = 86,016) themselves: factor, W = L^-1, packed tiles built in place
    # in the factor's buffer and its tail released (no dense + packed peak)
    host = pr.stencil_matrix(2, 64, 2, m)
    N = host.dim_r
    assert N == 64 * 64 * m
    A = BlockSparseMatrix(ctx, host)
    h = Hierarchy.setup(A, [], default_params(t_max=1, coarse_dim_cap=1 << 30))
    nt = (N + 63) // 64
    packed = nt * (nt + 1) // 2 * 64 * 64 * 8
    assert h.device_bytes < packed + 2 * 2 ** 30, (h.device_bytes, packed)  # not the 8 N^2 dense buffer
    b = pr.normal_vector(N, 0, 0)
    x = Vector(ctx, N)
    bv = Vector(ctx, b)
    h.v_cycle(1, 1, bv, x)
    r = Vector(ctx, N)
    residual(A, bv, x, r)
    rel = np.linalg.norm(r.download()) / np.linalg.norm(b)
    assert rel < 1e-8, rel


def test_triangular_coarse_path_matches_symmetric(ctx):
    # the W^T (W b) path (used when N0^2 >= 2^31), forced on a small hierarchy by a
    # child process with BMG_COARSE_TRIANGULAR=1, against the default symmetric inverse
    import json
    import os
    import subprocess
    import sys
    code = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, Vector, default_params
from paper_2509_06744_b200 import problems as pr
ctx = Context(0)
cfg = pr.CONFIGS["C2"].scaled(16, 3)
A, T, b = pr.make_problem(cfg)
h = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                    default_params(t_max=1, coarse_dim_cap=1 << 30))
x = Vector(ctx, b.size)
bv = Vector(ctx, b)
for _ in range(3):
    h.v_cycle(3, 3, bv, x)
B = np.stack([b, np.roll(b, 5)], axis=1).ravel().copy()
xb = Vector(ctx, B.size)
h.v_cycle_batch(3, 3, 2, Vector(ctx, B), xb)
x1 = Vector(ctx, b.size)
h.v_cycle(3, 3, Vector(ctx, np.roll(b, 5)), x1)
same = bool(np.array_equal(xb.download().reshape(-1, 2)[:, 1], x1.download()))
print(json.dumps({"x": x.download().tolist(), "batch_bitwise": same, "bytes": h.cycle_bytes(3, 3)}))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for tri in ("0", "1"):
        env = dict(os.environ, BMG_COARSE_TRIANGULAR=tri)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    x0, x1 = np.array(outs[0]["x"]), np.array(outs[1]["x"])
    assert np.linalg.norm(x1 - x0) <= 1e-10 * np.linalg.norm(x0)
    assert outs[0]["batch_bitwise"] and outs[1]["batch_bitwise"]
    assert outs[1]["bytes"] > outs[0]["bytes"]
