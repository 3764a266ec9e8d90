"""V-cycles/s of a config's hierarchy whole and row-partitioned in emulation (all
virtual ranks on this GPU, halos as device copies): the partitioned path's
per-pass cost with and without half-storage A (run twice, BMG_SYM_HALF=0 / unset).
Usage: python tools/partitioned_timing.py C4 48 [world]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_06744_b200 import Context, Vector  # noqa: E402
from paper_2509_06744_b200 import problems as pr  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
world = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = pr.CONFIGS[name].scaled(n)
ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
H, b = bench.whole_hierarchy(ctx, cfg)
bv, xv = Vector(ctx, b), Vector(ctx, b.size)
whole_ms = bench.time_cycles(ctx, stream, H, bv, xv, cfg.k, 10)
ref = xv.download()
H.partition(world, pr.level_grid(cfg)[2], agglomerate=1, rank=-1)
x2 = Vector(ctx, b.size)
part_ms = bench.time_cycles(ctx, stream, H, bv, x2, cfg.k, 10)
print(json.dumps({"config": cfg.name, "world": world, "sym_env": os.environ.get("BMG_SYM_HALF", "auto"),
                  "whole_ms": whole_ms, "partitioned_emulated_ms": part_ms,
                  "cycle_bytes": H.cycle_bytes(cfg.k, cfg.k), "cycle_bytes_ref": H.cycle_bytes_ref(cfg.k, cfg.k)}))
