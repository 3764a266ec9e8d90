"""Writes tests/golden/*.json.

Two kinds of fixtures:
  * known_answers.json -- the hand-derived expected values the reference's own
    tests assert (proj/tests/test_blockcore.cpp, test_fsai.cpp, test_chebyshev.cpp,
    test_multilevel.cpp), with the line they come from.  The reference ships no
    data files and cannot be built here (Eigen3 absent), so these are its only
    golden values.
  * oracle_*.json -- outputs of the CPU oracle (itself pinned to the known
    answers by tests/test_oracle_pins.py) on small seeded BASELINE-shaped inputs;
    the GPU tests compare against these committed numbers, and the CPU tests
    check the oracle still reproduces them bitwise.

Run:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))


def known_answers():
    return {
        "source": "/root/reference/proj/tests (values asserted there)",
        "cholesky_4_2_5": {"b": [[4, 2], [2, 5]], "l": [[2, 0], [1, 2]], "ref": "test_blockcore.cpp:129-134"},
        "cholesky_indefinite_pivot": {"b": [[1, 2], [2, 1]], "pivot": 1, "ref": "test_blockcore.cpp:139-146"},
        "fsai_scalar22": {"a": [[4, 1], [1, 3]], "F21": -0.25, "S": [4.0, 2.75], "ref": "test_fsai.cpp:71-77"},
        "triple_product_hand": {"a": [[4, 1], [1, 3]], "F21": -0.25, "diag": [4.0, 2.75], "offdiag_dropped": True,
                                "ref": "test_blockcore.cpp:94-101"},
        "cheb4_degree1_factor": {"value": -1.0 / 3.0, "ref": "test_chebyshev.cpp:83-89"},
        "fourth_kind_W_at_one": {"k": list(range(7)), "value": [2 * k + 1 for k in range(7)],
                                 "ref": "test_chebyshev.cpp:22-27"},
        "lanczos_diag_1_50": {"lo": 49.5, "hi": 50.0, "ref": "test_multilevel.cpp:60-69"},
        "lanczos_scaled_identity": {"c": 7.5, "n": 20, "ref": "test_multilevel.cpp:71-73"},
        "galerkin_aggregation": {"value": 2.0, "ref": "test_multilevel.cpp:35-41"},
    }


def oracle_fixtures():
    from oracle import pyoracle as O
    from paper_2509_06744_b200 import problems as pr

    out = {}
    # C1-shaped smoother application on a 16^2 grid
    A = pr.stencil_matrix(2, 16, 2, 10)
    om = O.Mat(A)
    of = O.Fsai(om, O.Fsai.STATIC)
    beta = O.lanczos_lambda_max(om, of, 100, 1.01, 42)
    b = pr.normal_vector(A.dim_r, 0, 0)
    x0 = pr.normal_vector(A.dim_r, 0, 3)
    x = O.smoother_apply(om, of, O.CHEB_FOURTH, b, x0, 3, beta=beta)
    y = om.spmv(x0)
    out["c1_16"] = {"grid": 16, "m": 10, "beta": beta, "spmv_x0_head": y[:64].tolist(),
                    "spmv_x0_norm": float(np.linalg.norm(y)), "cheb4_k3_head": x[:64].tolist(),
                    "cheb4_k3_norm": float(np.linalg.norm(x))}
    # C2-shaped hierarchy, residual history
    cfg = pr.CONFIGS["C2"].scaled(32, 3)
    A, T, b = pr.make_problem(cfg)
    h = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, coarse_dim_cap=1 << 30, probe=False)
    hist, it, st, _ = h.solve(3, 3, b, np.zeros_like(b), 1e-8, 20)
    out["c2_32_3lev"] = {"grid": 32, "levels": 3, "m": 10, "betas": [h.beta(l) for l in range(1, h.levels())],
                         "rho": (hist / hist[0]).tolist(), "r0": float(hist[0])}
    return out


if __name__ == "__main__":
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(known_answers(), f, indent=1)
    with open(os.path.join(HERE, "oracle_small.json"), "w") as f:
        json.dump(oracle_fixtures(), f, indent=1)
    print("wrote", os.listdir(HERE))
