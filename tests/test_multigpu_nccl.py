"""Multi-GPU path over real NCCL (skipped with fewer than 2 GPUs): bench.py under
torchrun partitions C2 into row strips (distributed setup, NCCL halos, coarsest
level on rank 0) and itself checks the partitioned cycle bitwise against the
1-GPU cycle before timing; a failure there fails the run (no replica fallback)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("n", [2, 4])
def test_bench_row_strips_over_nccl(n):
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "bench.py"), "--gpus", str(n),
           "--steps", "3", "--warmup", "3", "--config", "C2", "--no-extra", "--no-cpu-baseline", "--no-parity"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-4000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == n
    assert line["run"]["parallelism"].startswith(f"row strips x{n}"), line["run"]["parallelism"]
    assert "verified bitwise" in line["run"]["parallelism"]
    assert len(line["run"]["rank_device_gb"]) == n
    assert line["value"] > 0
