"""The host-buffer cycle (bmg_vcycle_host, the bench's `e2e` path) on a finest level
in half storage: phase 1 of the first residual runs in row ranges of the lower
triangle as the x slices land, b arrives under it, the merge follows
(vcycle.cu run_vcycle_hostio).  Must be bitwise the device-vector cycle.  The child
process forces half storage on every level (BMG_SYM_HALF=1) so small grids take it."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, %r)
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, Vector, default_params
from paper_2509_06744_b200 import problems as pr
ctx = Context(0)
for name, scaled, nest, cycles in (("C4", (16, 3), 0, ((3, 3), (1, 0))), ("C5", (64, 4), 0, ((3, 3),)),
                                   ("C3", (32, 3), 1, ((4, 4),)), ("C2", (64, 3), 0, ((3, 3), (2, 1)))):
    cfg = pr.CONFIGS[name].scaled(*scaled)
    A, T, b = pr.make_problem(cfg)
    dh = Hierarchy.setup(BlockSparseMatrix(ctx, A), [BlockSparseMatrix(ctx, p) for p in T],
                         default_params(t_max=1, nest=nest, coarse_dim_cap=1 << 30))
    Af, _, _ = dh.level(dh.levels - 1)
    assert Af.sym_info()["half"], name
    for kpre, kpost in cycles:
        x0 = pr.normal_vector(b.size, 0, 9)
        hb = torch.from_numpy(b.copy()).pin_memory()
        hx = torch.from_numpy(x0.copy()).pin_memory()
        xv, bv = Vector(ctx, x0), Vector(ctx, b)
        for _ in range(3):
            dh.v_cycle_host_ptr(kpre, kpost, hb.data_ptr(), hx.data_ptr())
            dh.v_cycle(kpre, kpost, bv, xv)
            assert np.array_equal(hx.numpy(), xv.download()), (name, kpre, kpost)
        assert np.array_equal(hb.numpy(), b)
print("hostio-half ok")
""" % ROOT


def test_host_buffer_cycle_on_half_storage_equals_device_cycle():
    env = dict(os.environ, BMG_SYM_HALF="1")
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "hostio-half ok" in r.stdout
