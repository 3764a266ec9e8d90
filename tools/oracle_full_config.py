"""One-off check of the CPU legs' bounded sample: the oracle on the WHOLE config
(setup, then timed V-cycles on all host threads) against the rate bench.py
derives from its smaller sample (CPU_SAMPLE, scaled by algorithmic bytes).
Usage: python tools/oracle_full_config.py C4 [cycles]   (C4 needs ~130 GB host RAM)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_2509_06744_b200 import problems as pr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = pr.CONFIGS[name]
threads = os.cpu_count() or 1
O.set_threads(threads)
t0 = time.perf_counter()
A, T, b = pr.make_problem(cfg)
oA = O.Mat(A)
oT = [O.Mat(p) for p in T]
del A, T
gen_s = time.perf_counter() - t0
t0 = time.perf_counter()
oh = O.Hierarchy(oA, oT, t_max=1, tau=1.0, nest=cfg.nest, coarse_dim_cap=1 << 30, probe=False, consume=True)
setup_s = time.perf_counter() - t0
del oA, oT
n0 = oh.A(0).info()["dim_r"]
full_bytes = bench.cycle_bytes_model(bench.oracle_levels(oh, cfg.m), cfg.k, cfg.k, n0)
x = np.zeros_like(b)
x = oh.v_cycle(cfg.k, cfg.k, b, x)  # warm
t0 = time.perf_counter()
for _ in range(cycles):
    x = oh.v_cycle(cfg.k, cfg.k, b, x)
dt = time.perf_counter() - t0
full_rate = cycles / dt
del oh
s = bench.oracle_sample(cfg, 3, 1, threads)
print(json.dumps({"config": name, "threads": threads, "generate_s": round(gen_s, 1), "setup_s": round(setup_s, 1),
                  "full_cycles": cycles, "full_rate": full_rate, "full_bytes_model": full_bytes,
                  "table_bytes": bench.CYCLE_BYTES.get(name), "sample": s["sample"], "sample_rate": s["rate_sample"],
                  "sample_scaled_rate": s["value"], "scaled_over_full": s["value"] / full_rate}), flush=True)
