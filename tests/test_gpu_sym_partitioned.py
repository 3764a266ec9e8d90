"""Half-storage A on partitioned levels (hier.h PSym, vcycle.cu sym_residual_pass):
the partitioned, distributed-setup and bench-branch tests rerun in a child
process with BMG_SYM_HALF=1, which puts every partitioned level (and every whole
one) in half storage -- their cycles, residual histories and iterates must stay
bitwise equal to the single-device runs they compare against (which use the
full- or half-storage pass, bitwise the same)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_partitioned_suites_with_half_storage_forced():
    env = dict(os.environ, BMG_SYM_HALF="1")
    tests = ["tests/test_gpu_loopback.py", "tests/test_gpu_dist.py", "tests/test_gpu_bench_paths.py",
             "tests/test_gpu_solver.py::test_partitioned_vcycle_bitwise_equal_to_single"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "-k", "not memory_plan"] + tests, cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
