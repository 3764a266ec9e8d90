"""Host planning of the distributed setup (bmg_dist_plan; no device needed)."""
import numpy as np
import pytest

from paper_2509_06744_b200 import default_params
from paper_2509_06744_b200 import problems as pr
from paper_2509_06744_b200.api import dist_plan


def _keep(R, t, nest):
    keep, Rq = (t + 1) * R, R
    for _ in range(nest):
        Rq = (2 * t + 1) * Rq
        keep += (t + 2) * Rq
    return keep


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_invariants(name, world):
    cfg = pr.CONFIGS[name]
    if cfg.levels < 2:
        cfg = cfg.scaled(cfg.n, 3)
    ns, nbr, gran, rad = pr.level_grid(cfg)
    params = default_params(t_max=1, nest=cfg.nest)
    for agg in (1, cfg.levels - 1):
        B, lo, hi, halo = dist_plan(nbr, gran, rad, world, agg, params)
        for l in range(cfg.levels):
            b = B[l]
            assert b[0] == 0 and b[-1] == nbr[l] and np.all(np.diff(b) >= 0)
            if l < agg:
                assert np.all(b[1:] == nbr[l]) and lo[l, 0] == 0 and hi[l, 0] == nbr[l]
                continue
            assert np.all(b[:-1] % gran[l] == 0)
            assert halo[l] >= max(_keep(rad[l], 1, cfg.nest), rad[l] + 3)
            for r in range(world):
                if b[r + 1] > b[r]:
                    assert lo[l, r] == max(0, b[r] - halo[l] * gran[l])
                    assert hi[l, r] == min(nbr[l], b[r + 1] + halo[l] * gran[l])


def test_level_grid_radii():
    ns, nbr, gran, rad = pr.level_grid(pr.CONFIGS["C3"])
    assert rad[-1] == 3 and rad[:-1] == [4, 4, 4, 4]
    assert gran == ns and nbr == [n * n for n in ns]
    ns, nbr, gran, rad = pr.level_grid(pr.CONFIGS["C4"])
    assert gran == [n * n for n in ns]


def test_plan_rejects_bad_input():
    from paper_2509_06744_b200.native import InvalidArgument
    with pytest.raises(InvalidArgument):
        dist_plan([4], [2], [1], 2)
    with pytest.raises(InvalidArgument):
        dist_plan([4, 16], [2, 4], [1, 1], 0)


@pytest.mark.parametrize("name,n,levels", [("C5", 32, 3), ("C4", 8, 3), ("C3", 16, 3)])
def test_structural_offsets_bound_the_galerkin_levels(name, n, levels):
    # problems.level_offsets (the memory plan's structure) against the oracle's
    # Galerkin operators: every row holds at most the offsets on the grid, and
    # interior-dominated levels match exactly
    from oracle import pyoracle as O
    cfg = pr.CONFIGS[name].scaled(n, levels)
    A, T, _ = pr.make_problem(cfg)
    Ac = O.Mat(A)
    ns, nbr, gran, _ = pr.level_grid(cfg)
    offs = pr.level_offsets(cfg)
    mats = [None] * levels
    mats[-1] = Ac
    for l in range(levels - 1, 0, -1):
        mats[l - 1] = O.galerkin(mats[l], O.Mat(T[l - 1]))
    for l in range(levels):
        actual = mats[l].info()["nnzb"]
        bound = pr._count_rows(offs[l], ns[l], cfg.dim, 0, ns[l])
        assert actual <= bound, (l, actual, bound)
        if l == levels - 1:
            assert actual == bound  # the fine stencil itself


def test_memory_plan_fits_c3_c5_from_four_gpus():
    # BASELINE C3 / C5 do not fit one B200; from 4 ranks (coarsest two levels on
    # rank 0) every rank's setup peak stays under the 180 GB of HBM
    for name in ("C3", "C5"):
        cfg = pr.CONFIGS[name]
        assert max(p["peak_gb"] for p in pr.memory_plan(cfg, 1, 2)) > 180
        for world in (4, 8):
            plan = pr.memory_plan(cfg, world, 2)
            assert len(plan) == world
            assert max(p["peak_gb"] for p in plan) < 180, (name, world, plan)
