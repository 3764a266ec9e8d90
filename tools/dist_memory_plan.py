"""Per-rank device memory of the distributed hierarchy (problems.memory_plan:
structural upper bounds from bmg_dist_plan's strips), for every BASELINE config
at 1/2/4/8 ranks.  Usage: python tools/dist_memory_plan.py [CONFIG ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_06744_b200 import problems as pr  # noqa: E402

AGG = {"C2": 1, "C3": 2, "C4": 1, "C5": 2}
for name in sys.argv[1:] or ["C2", "C4", "C3", "C5"]:
    cfg = pr.CONFIGS[name]
    for world in (1, 2, 4, 8):
        plan = pr.memory_plan(cfg, world, AGG[name])
        worst = max(plan, key=lambda p: p["peak_gb"])
        fits = "fits" if worst["peak_gb"] < 180 else "does not fit"
        half = max(p["steady_gb"] + p["half_storage_gb"] for p in plan)
        print(f"{name} x{world}: steady max {max(p['steady_gb'] for p in plan):6.1f} GB, "
              f"setup peak max {worst['peak_gb']:6.1f} GB (rank {worst['rank']}) -> {fits} in 180 GB; "
              f"with the half-storage A of the large levels: steady max {half:6.1f} GB")
