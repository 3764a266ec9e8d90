"""The committed solve fixtures (tests/golden/solve_*.json) are the oracle's own
output: the oracle still reproduces them bitwise (setup digests, beta, the first
residual-history entries) -- CPU only, so a change to the restatement that would
move the golden values fails here before any GPU comparison."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import problems as pr
from tests.golden.make_solve_golden import bsr_digest, case_config, load


@pytest.mark.parametrize("case", ["C4@16x4"])
def test_oracle_reproduces_solve_fixture(case):
    fx = load(case)
    cfg, _ = case_config(case)
    A, T, b = pr.make_problem(cfg)
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, tau=1.0, nest=cfg.nest, coarse_dim_cap=1 << 30,
                     probe=False)
    for l in range(oh.levels()):
        assert bsr_digest(oh.A(l).export(symmetric=True)) == fx["level"][l]["A"]
        if l >= 1:
            assert bsr_digest(oh.fsai(l).G().export()) == fx["level"][l]["G"]
            assert float(oh.beta(l)).hex() == fx["level"][l]["beta"]
    hist, it, st, _ = oh.solve(cfg.k, cfg.k, b, np.zeros_like(b), cfg.tol, 20)
    assert np.array_equal(hist, fx["history_f"][:21])
