"""Runs THE REFERENCE ITSELF (oracle/_ref/libblockmg_ref.so: the reference's own
sources built against oracle/eigen_shim, see oracle/ref_driver.cpp) on the solve
fixtures of tests/golden/ and checks every recorded quantity bitwise: the SHA-256
of each level's Galerkin operator and FSAI factors, beta_l, the whole residual
history to 1e-8, the iteration count and the status.  The fixtures were written by
the oracle (the restatement); this closes the loop oracle == reference on the
BASELINE shapes.  Single-threaded (the reference is), so minutes per case.

Run here (the GPU box has no /root/reference; the library travels prebuilt):
  python tools/reference_vs_fixtures.py C4@16x4 C5@128x6 C3@128x5
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def run(case):
    import make_solve_golden as G
    from oracle import pyref as R
    from paper_2509_06744_b200 import problems as pr

    want = G.load(case)
    cfg, max_iter = G.case_config(case)
    A, T, b = pr.make_problem(cfg)
    t0 = time.time()
    rh = R.Hierarchy(R.Mat(A), [R.Mat(p) for p in T], t_max=1, tau=1.0, nest=cfg.nest, fsai_kind=3,
                     coarse_dim_cap=1 << 30)
    setup_s = time.time() - t0
    bad = []
    for l in range(rh.levels()):
        ent = want["level"][l]
        if G.bsr_digest(rh.A(l).export(symmetric=True)) != ent["A"]:
            bad.append(f"A[{l}]")
        if l >= 1:
            f = rh.fsai(l)
            got = [G.bsr_digest(f.factor(k).export()) for k in range(f.chain_len() - 1)]
            if got != ent["factors"]:
                bad.append(f"factors[{l}]")
            if G.bsr_digest(f.G().export()) != ent["G"]:
                bad.append(f"G[{l}]")
            if float(rh.beta(l)).hex() != ent["beta"]:
                bad.append(f"beta[{l}]")
    t0 = time.time()
    hist, it, st, x = rh.solve(cfg.k, cfg.k, b, np.zeros_like(b), cfg.tol, max_iter)
    solve_s = time.time() - t0
    if int(it) != want["iterations"] or int(st) != want["status"]:
        bad.append(f"iterations {it} vs {want['iterations']}")
    if [float(v).hex() for v in hist] != want["history"]:
        bad.append("history")
    if float(np.linalg.norm(x)).hex() != want["x_norm"]:
        bad.append("x_norm")
    return {"case": case, "reference_equals_fixture_bitwise": not bad, "differences": bad, "levels": rh.levels(),
            "iterations": int(it), "status": int(st), "history_entries_compared": len(hist),
            "reference_setup_s": round(setup_s, 1), "reference_solve_s": round(solve_s, 1),
            "reference_cycles_per_s_1_thread": round(it / solve_s, 3) if solve_s > 0 else None,
            "fixture": os.path.relpath(G.path_for(case), ROOT)}


if __name__ == "__main__":
    for c in sys.argv[1:]:
        print(json.dumps(run(c)), flush=True)
