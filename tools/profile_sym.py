"""Three finest-level residual passes r = b - A x of a BASELINE config's device
hierarchy (after setup), inside cudaProfilerStart/Stop so that
  ncu --profile-from-start off --set full -k regex:"bsr_stream|sym_merge" python tools/profile_sym.py C4
captures exactly those launches (BMG_SYM_HALF=1 forces the symmetric-half form,
0 the full one).  Prints the pass's algorithmic bytes."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_06744_b200 import Context, Vector, residual  # noqa: E402
from paper_2509_06744_b200 import problems as pr  # noqa: E402

_arg = sys.argv[1] if len(sys.argv) > 1 else "C4"  # NAME or NAME@N (same shape on an N-per-side grid)
cfg = pr.CONFIGS[_arg.split("@")[0]]
if "@" in _arg:
    cfg = cfg.scaled(int(_arg.split("@")[1]))
ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
H, b = bench.whole_hierarchy(ctx, cfg)
Af, _, _ = H.level(H.levels - 1)
n = b.size
bv, xv, rv = Vector(ctx, b), Vector(ctx, pr.normal_vector(n, 0, 5)), Vector(ctx, n)
residual(Af, bv, xv, rv)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(3):
    residual(Af, bv, xv, rv)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
si = Af.sym_info()
print(json.dumps({"config": cfg.name, "m": cfg.m, "half": si["half"], "algorithmic_bytes": si["pass_bytes"] + 24 * n,
                  "full_storage_bytes": Af.info()["pass_bytes"] + 24 * n, "half_ms": si["half_ms"],
                  "full_ms": si["full_ms"]}), flush=True)
