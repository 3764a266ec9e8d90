"""Writes tests/golden/solve_<case>.json: the CPU oracle (the restatement of the
reference, pinned by tests/test_oracle_pins.py) run on BASELINE-shaped
hierarchies -- setup as the reference's `setup` (multilevel.cpp:36-75) and the
stop-on-tolerance loop of `measure_rates` (experiments.cpp:46-58) to
||r_n|| / ||r_0|| < 1e-8.

Each fixture records, per level, a SHA-256 of the Galerkin operator A_l and of
the FSAI factors (F_0 .. F_{nest-1}, G = L^-1 F_nest) as exported by the oracle
(row_ptr int64, col_idx int32, values f64, concatenated), beta_l (hex), and the
whole residual history (hex), the iteration count and the status.  The GPU tests
(tests/test_gpu_shapes.py, tests/test_gpu_c2_oracle.py) compare the device
setup + solve against these numbers: the reference cannot be built here (Eigen3
absent), so the oracle's outputs are the golden values.

Cases keep each BASELINE config's block size, stencil, nesting, smoother degree
and (where the grid allows) depth, at reduced grid sizes; "C2" is the full
headline configuration (256^2 patches, 4 levels; ~10 min on 8 host threads).

Run:  python tests/golden/make_solve_golden.py [case ...]   (default: all)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))

# case -> (config, n, levels, max_iter)
CASES = {
    "C4@16x4": ("C4", 16, 4, 3000),   # 3-D, m = 20, 25-pt, adaptive, V(3,3); 2^3 coarsest
    "C4@32x4": ("C4", 32, 4, 3000),   # 1/8 of C4's rows, same depth
    "C5@128x6": ("C5", 128, 6, 3000),  # m = 15, 13-pt, 6 levels (4^2 coarsest)
    "C5@256x6": ("C5", 256, 6, 3000),
    "C3@128x5": ("C3", 128, 5, 3000),  # m = 21, 25-pt triharmonic, nest = 1, V(4,4), 5 levels
    "C3@256x5": ("C3", 256, 5, 3000),
    "C2": ("C2", None, None, 4000),    # the full headline configuration
}


def case_config(case):
    from paper_2509_06744_b200 import problems as pr
    name, n, levels, max_iter = CASES[case]
    cfg = pr.CONFIGS[name] if n is None else pr.CONFIGS[name].scaled(n, levels)
    return cfg, max_iter


def bsr_digest(h) -> str:
    d = hashlib.sha256()
    d.update(np.ascontiguousarray(h.row_ptr, np.int64).tobytes())
    d.update(np.ascontiguousarray(h.col_idx, np.int32).tobytes())
    d.update(np.ascontiguousarray(h.vals, np.float64).tobytes())
    return d.hexdigest()


def oracle_case(case, threads=None):
    from oracle import pyoracle as O
    from paper_2509_06744_b200 import problems as pr

    cfg, max_iter = case_config(case)
    O.set_threads(threads or os.cpu_count() or 1)
    A, T, b = pr.make_problem(cfg)
    t0 = time.time()
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, tau=1.0, nest=cfg.nest,
                     fsai_kind=0 if cfg.fsai == "static" else 3, coarse_dim_cap=1 << 30, probe=False)
    setup_s = time.time() - t0
    levels = []
    for l in range(oh.levels()):
        ent = {"A": bsr_digest(oh.A(l).export(symmetric=True))}
        if l >= 1:
            f = oh.fsai(l)
            ent["factors"] = [bsr_digest(f.factor(k).export()) for k in range(f.chain_len() - 1)]
            ent["G"] = bsr_digest(f.G().export())
            ent["beta"] = float(oh.beta(l)).hex()
        levels.append(ent)
    t0 = time.time()
    hist, it, st, x = oh.solve(cfg.k, cfg.k, b, np.zeros_like(b), cfg.tol, max_iter)
    solve_s = time.time() - t0
    return {
        "case": case, "config": cfg.name, "n": cfg.n, "dim": cfg.dim, "m": cfg.m, "levels": cfg.levels,
        "power": cfg.power, "nest": cfg.nest, "k": cfg.k, "fsai": cfg.fsai, "seed": cfg.seed,
        "tol": cfg.tol, "max_iter": max_iter, "t_max": 1, "lanczos": [100, 1.01, 42],
        "level": levels, "iterations": int(it), "status": int(st),
        "history": [float(v).hex() for v in hist],
        "x_norm": float(np.linalg.norm(x)).hex(),
        "oracle_threads": O.get_threads(), "setup_s": round(setup_s, 1), "solve_s": round(solve_s, 1),
        "generator": "tests/golden/make_solve_golden.py (CPU oracle, oracle/bmg_oracle.cpp)",
    }


def path_for(case):
    return os.path.join(HERE, "solve_" + case.replace("@", "_") + ".json")


def load(case):
    with open(path_for(case)) as f:
        d = json.load(f)
    d["history_f"] = np.array([float.fromhex(v) for v in d["history"]])
    return d


def main(argv):
    cases = argv or list(CASES)
    for c in cases:
        d = oracle_case(c)
        with open(path_for(c), "w") as f:
            json.dump(d, f, indent=1)
        print(f"{c}: {d['iterations']} iterations (status {d['status']}), rho_end "
              f"{float.fromhex(d['history'][-1]) / float.fromhex(d['history'][0]):.3e}, "
              f"setup {d['setup_s']} s, solve {d['solve_s']} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
