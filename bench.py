#!/usr/bin/env python
"""Benchmark: V-cycle application of the multilevel Chebyshev(4th kind) + block-FSAI
solver (arXiv 2509.06744 hot path, the reference's `v_cycle`, multilevel.cpp:77-103,
driven as in `measure_rates`, experiments.cpp:15-67) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A step is one V(k,k) cycle on the finest level of the config's hierarchy, with the
hierarchy, b and x resident in HBM.  Default workload: C4 (BASELINE.json
configs[3]: 64^3 patches, m = 20, 3-D 25-point, 4 levels, adaptive block-FSAI,
V(3,3)) -- the largest BASELINE config that fits one B200 (C3 and C5 need >= 4,
problems.memory_plan).  Every cycle streams ~434 GB (>> 126 MB L2), so no flush
is needed between cycles.

N > 1 (torchrun, one rank per GPU, NCCL): the hierarchy is built by the
distributed setup (bmg_hier_setup_dist) from each rank's strips only -- no rank
ever holds a whole partitioned level -- with the config's coarsest levels
agglomerated on rank 0 (C5: 2, per BASELINE), NCCL halo exchanges inside the
captured cycle, strong scaling.  Partition invariance is checked bitwise on a
scaled copy before timing; a failing distributed path fails the run.
`--replicas` runs independent copies instead (weak scaling).

`--impl reference` times the CPU oracle (oracle/: the plain-C++ restatement of
the reference, which itself needs Eigen3, absent) on the host cores.  It maps
only oracle/liboracle.so and the input generator bmggen/libbmggen.so -- never the
product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0
# coarsest levels held whole on rank 0 in N > 1 runs (BASELINE configs[4]: C5 "coarsest
# two levels agglomerated on one GPU"; the dense level alone for the single-GPU configs)
AGGLOMERATE = {"C2": 1, "C3": 2, "C4": 1, "C5": 2}
# the CPU legs (cpu_baseline, --impl reference) time oracle V-cycles on a bounded
# sample: the config's own shape (block size, stencil, FSAI, depth, smoother) on a
# smaller grid, its rate scaled to the full config by the ratio of algorithmic bytes
# per cycle.  C2 runs whole.
CPU_SAMPLE = {"C2": None, "C4": ("C4", 32, 4), "C3": ("C3", 256, 5), "C5": ("C5", 512, 6)}
# algorithmic bytes per V(k,k) cycle of each full config with A stored whole, as the
# reference (and the oracle) store it -- the scale of the CPU samples; the GPU arm
# re-derives it (bmg_hier_cycle_bytes_ref) and reports a mismatch
CYCLE_BYTES = {"C2": 13_813_927_776, "C4": 433_649_594_288}
# residual-history fixtures of the oracle (tests/golden/make_solve_golden.py) the
# GPU arm reproduces in every run: the headline shape and the full C2
PARITY_CASE = {"C4": "C4@16x4", "C2": "C2", "C5": "C5@128x6", "C3": "C3@128x5"}
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r02_traffic.json")


def hbm_peak():
    try:
        with open(MEASURED_PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def read_peak_gbs():
    """Read-only HBM bandwidth of this GPU, measured here (torch.sum over 4 GB of
    fp64, best of 5): the streaming passes are ~97 % reads, while MEASURED_PEAKS'
    figure is a copy (read + write), which a read-dominated kernel can exceed."""
    import torch

    n = 1 << 29
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    x.sum()
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x.sum()
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 8 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del x
    torch.cuda.empty_cache()
    return best


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower().startswith("active")})
        under_load = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(under_load) if under_load else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons, "samples": len(self.rows),
                "power_w": statistics.median(pw) if pw else None}


def cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return model


def config_dict(cfg):
    """The workload description, identical in both arms."""
    return {"workload": f"{cfg.name}: {cfg.n}^{cfg.dim} patches, m={cfg.m}, {cfg.levels} levels, "
                        f"{'3-D' if cfg.dim == 3 else '2-D'} {cfg_points(cfg)}-point block stencil, "
                        f"V({cfg.k},{cfg.k}), {cfg.fsai} block-FSAI t_max=1" + (f", nest={cfg.nest}" if cfg.nest else ""),
            "config": cfg.name, "patches": cfg.n ** cfg.dim, "m": cfg.m, "levels": cfg.levels,
            "cycle": f"V({cfg.k},{cfg.k})", "seed": cfg.seed,
            "l2": "inputs larger than L2 (>= 14 GB streamed per cycle vs 126 MB of L2): no flush needed"}


def cfg_points(cfg):
    from paper_2509_06744_b200 import problems as pr
    return len(pr.level_offsets(cfg.scaled(cfg.n, 1))[0])


# ------------------------------------------------------------------ byte model (both arms)
def cycle_bytes_model(levels, kpre, kpost, n0):
    """Algorithmic bytes of one V(kpre, kpost) cycle from per-level structure
    (coarsest first): dict(n, a_pass, m_pass, r_pass, p_pass) -- the same model as
    the device's bmg_hier_cycle_bytes (hierarchy.cu), so the CPU legs scale with it."""
    tot = 0
    top = len(levels) - 1
    for l in range(1, top + 1):
        s = levels[l]
        n, nc = s["n"], levels[l - 1]["n"]
        apass = s["a_pass"] + 24 * n
        gvec = 16 * n + 40 * n
        lvl = (kpre + kpost) * (apass + s["m_pass"] + gvec)
        if l < top and kpre > 0:
            lvl -= apass + 8 * n
        lvl += apass
        lvl += s["r_pass"] + 8 * n + 8 * nc
        lvl += s["p_pass"] + 8 * nc + 16 * n
        tot += lvl
    nt = (n0 + 63) // 64
    one = nt * (nt + 1) // 2 * 64 * 64 * 8 + 16 * n0 + 2 * nt * nt * 64 * 8
    tot += 2 * one if n0 * n0 >= (1 << 31) - 1 else one
    return tot


def oracle_levels(oh, m):
    """Per-level structure of an oracle hierarchy for cycle_bytes_model."""
    def pass_bytes(mat, mr, mc):
        return mat.info()["nnzb"] * (8 * mr * mc + 4)
    out = []
    for l in range(oh.levels()):
        A = oh.A(l)
        s = {"n": A.info()["dim_r"], "a_pass": pass_bytes(A, m, m)}
        if l >= 1:
            f = oh.fsai(l)
            mp = sum(pass_bytes(f.factor(k), m, m) for k in range(f.chain_len() - 1)) + pass_bytes(f.G(), m, m)
            s["m_pass"] = 2 * mp
            s["r_pass"] = s["p_pass"] = pass_bytes(oh.P(l), m, m)
        out.append(s)
    return out


# ------------------------------------------------------------------ CPU oracle legs
def oracle_sample(cfg, steps, warmup, threads, single_core=False):
    """Oracle V-cycles on CPU_SAMPLE[cfg]: setup untimed, `warmup` + `steps` cycles
    timed by wall clock on `threads` threads; the rate is scaled to the full config
    by the ratio of algorithmic bytes per cycle."""
    from oracle import pyoracle as O
    from paper_2509_06744_b200 import problems as pr

    spec = CPU_SAMPLE.get(cfg.name)
    scfg = cfg if spec is None else pr.CONFIGS[spec[0]].scaled(spec[1], spec[2])
    O.set_threads(threads)
    A, T, b = pr.make_problem(scfg)
    t0 = time.perf_counter()
    oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, tau=1.0, nest=scfg.nest,
                     fsai_kind=0 if scfg.fsai == "static" else 3, coarse_dim_cap=1 << 30, probe=False, consume=True)
    setup_s = time.perf_counter() - t0
    del A, T
    n0 = oh.A(0).info()["dim_r"]
    sample_bytes = cycle_bytes_model(oracle_levels(oh, scfg.m), scfg.k, scfg.k, n0)
    x = np.zeros_like(b)
    for _ in range(warmup):
        x = oh.v_cycle(scfg.k, scfg.k, b, x)
    t0 = time.perf_counter()
    for _ in range(steps):
        x = oh.v_cycle(scfg.k, scfg.k, b, x)
    dt = time.perf_counter() - t0
    rate = steps / dt
    full_bytes = CYCLE_BYTES.get(cfg.name) if spec is not None else sample_bytes
    scale = sample_bytes / full_bytes if full_bytes else None
    out = {"rate_sample": rate, "sample": scfg.name, "sample_bytes": sample_bytes, "setup_s": setup_s, "dt": dt,
           "steps": steps, "scale": scale, "value": rate * scale if scale else None}
    if single_core:  # the reference itself is single-threaded
        O.set_threads(1)
        t1 = time.perf_counter()
        x = oh.v_cycle(scfg.k, scfg.k, b, x)
        r1 = 1.0 / (time.perf_counter() - t1)
        out["single_core"] = {"rate_sample": r1, "value": r1 * scale if scale else None}
        O.set_threads(threads)
    return out


# the reference's own sources (oracle/_ref, built against oracle/eigen_shim): a small
# same-shape sample, since they are single-threaded and the stand-in's dense
# primitives are not vectorised
REF_BUILD_SAMPLE = {"C4": ("C4", 8, 3), "C2": ("C2", 32, 3), "C3": ("C3", 32, 3), "C5": ("C5", 32, 4)}


def reference_build_sample(cfg, steps=2):
    """V-cycles of THE REFERENCE ITSELF (oracle/_ref/libblockmg_ref.so) on a small
    hierarchy of cfg's shape, one thread, scaled to cfg by algorithmic bytes."""
    from oracle import pyref as R
    from paper_2509_06744_b200 import problems as pr

    if not R.available() or cfg.name not in REF_BUILD_SAMPLE:
        return None
    name, n, levels = REF_BUILD_SAMPLE[cfg.name]
    scfg = pr.CONFIGS[name].scaled(n, levels)
    A, T, b = pr.make_problem(scfg)
    t0 = time.perf_counter()
    rh = R.Hierarchy(R.Mat(A), [R.Mat(p) for p in T], t_max=1, tau=1.0, nest=scfg.nest, coarse_dim_cap=1 << 30)
    setup_s = time.perf_counter() - t0
    sample_bytes = cycle_bytes_model(oracle_levels(rh, scfg.m), scfg.k, scfg.k, rh.A(0).info()["dim_r"])
    x = rh.v_cycle(scfg.k, scfg.k, b, np.zeros_like(b))
    t0 = time.perf_counter()
    for _ in range(steps):
        x = rh.v_cycle(scfg.k, scfg.k, b, x)
    rate = steps / (time.perf_counter() - t0)
    full = CYCLE_BYTES.get(cfg.name)
    return {"value": rate * sample_bytes / full if full else None, "unit": "V-cycles/s", "cores": 1,
            "kind": "reference",
            "sample": f"{steps} V-cycles of the reference's own sources (oracle/_ref: proj/src/*.cpp compiled in "
                      f"place against oracle/eigen_shim, Eigen3 being absent; single-threaded as the reference is, "
                      f"dense primitives not vectorised) on {scfg.name} after {setup_s:.1f} s setup; measured "
                      f"{rate:.4g} cycles/s, {sample_bytes / 1e9:.3f} GB per cycle, scaled to {cfg.name} by bytes"}


def sample_text(s, threads, cfg):
    if s["sample"] == cfg.name:
        return (f"{s['steps']} V-cycles of the C++ oracle (reference restatement; the reference needs Eigen3, "
                f"absent) on {cfg.name} itself after {s['setup_s']:.0f} s untimed setup, {threads} OpenMP threads, "
                f"CPU {cpu_info()}")
    return (f"{s['steps']} V-cycles of the C++ oracle (reference restatement) on {s['sample']} -- {cfg.name}'s shape "
            f"(m={cfg.m}, same stencil, FSAI, depth, V({cfg.k},{cfg.k})) on a smaller grid -- after "
            f"{s['setup_s']:.0f} s untimed setup, {threads} OpenMP threads, CPU {cpu_info()}; measured "
            f"{s['rate_sample']:.4g} cycles/s on the sample, scaled to {cfg.name} by the algorithmic bytes per cycle "
            f"({s['sample_bytes'] / 1e9:.2f} GB sample vs {CYCLE_BYTES.get(cfg.name, 0) / 1e9:.1f} GB full)")


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    s = oracle_sample(cfg, max(1, args.steps), args.warmup, threads)
    unit = "V-cycles/s"
    line = {
        "impl": "reference",
        "metric": f"V-cycles/s ({cfg.name}, V({cfg.k},{cfg.k}))",
        "value": s["value"], "unit": unit, "n_gpus": args.gpus, "steps": max(1, args.steps), "warmup": args.warmup,
        "ms_per_step": 1e3 / s["value"] if s["value"] else None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.md §3 generator bmggen/, seed 0)",
        "config": config_dict(cfg),
        "cpu_baseline": {"value": s["value"], "unit": unit, "cores": threads, "kind": "port",
                         "sample": sample_text(s, threads, cfg)},
        "e2e": {"value": s["value"], "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:  # the reference's own sources on one thread, reported beside the (faster) 16-thread port
        rb = reference_build_sample(cfg)
        if rb is not None:
            line["cpu_baseline"]["reference_build"] = rb
    except Exception as e:
        line["cpu_baseline"]["reference_build"] = {"error": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm helpers
def setup_params(cfg):
    from paper_2509_06744_b200 import default_params
    return default_params(t_max=1, tau=1.0, nest=cfg.nest, coarse_dim_cap=1 << 30,
                          fsai_kind=0 if cfg.fsai == "static" else 3)


def whole_hierarchy(ctx, cfg):
    """Single-device setup (bmg_hier_setup) of the whole config; host inputs freed."""
    from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy
    from paper_2509_06744_b200 import problems as pr
    A, T, b = pr.make_problem(cfg)
    dA = BlockSparseMatrix(ctx, A)
    dT = [BlockSparseMatrix(ctx, p) for p in T]
    del A, T
    H = Hierarchy.setup(dA, dT, setup_params(cfg))
    return H, b


def partitioned_hierarchy(ctx, cfg, world, rank, agglomerate):
    """This rank's share of the distributed setup (bmg_hier_setup_dist): the
    generator produces only the plan's extended strips for this rank."""
    from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy
    from paper_2509_06744_b200 import problems as pr
    params = setup_params(cfg)
    _, _, gran, rad = pr.level_grid(cfg)
    A_ext, T_ext, b_own, _ = pr.dist_inputs(cfg, world, rank, agglomerate, params)
    H = Hierarchy.setup_dist(ctx, BlockSparseMatrix(ctx, A_ext), [BlockSparseMatrix(ctx, p) for p in T_ext], gran,
                             rad, agglomerate, params)
    return H, b_own


def invariance_check(ctx, cfg, world, rank, agglomerate, all_min, cycles=2):
    """The partitioned cycle (distributed setup, halo exchanges through the
    context's transport) must reproduce the single-device cycle bitwise on every
    rank's rows; raises otherwise.  Run on a scaled copy of the config."""
    from paper_2509_06744_b200 import Vector
    H1, b = whole_hierarchy(ctx, cfg)
    x1 = Vector(ctx, b.size)
    bv = Vector(ctx, b)
    for _ in range(cycles):
        H1.v_cycle(cfg.k, cfg.k, bv, x1)
    ref = x1.download()
    del H1, x1, bv
    Hp, b_own = partitioned_hierarchy(ctx, cfg, world, rank, agglomerate)
    lo = Hp.part_info(cfg.levels - 1, rank)[0]
    xp = Vector(ctx, b_own.size)
    bp = Vector(ctx, b_own)
    for _ in range(cycles):
        Hp.v_cycle(cfg.k, cfg.k, bp, xp)
    ok = bool(np.array_equal(xp.download(), ref[lo * cfg.m:lo * cfg.m + b_own.size]))
    if all_min(1 if ok else 0) != 1:
        raise RuntimeError(f"partitioned V-cycle of {cfg.name} differs from the single-GPU cycle")
    return True


def parity_check(ctx, case):
    """Device setup + solve to 1e-8 on an oracle fixture case (the residual-history
    criterion of BASELINE.md §2): iteration counts and the largest |rho_gpu - rho_cpu|."""
    from paper_2509_06744_b200 import Vector
    from tests.golden.make_solve_golden import case_config, load, path_for
    if not os.path.exists(path_for(case)):
        return {"case": case, "skipped": "fixture not generated"}
    fx = load(case)
    cfg, _ = case_config(case)
    H, b = whole_hierarchy(ctx, cfg)
    bv, xv = Vector(ctx, b), Vector(ctx, b.size)
    t0 = time.perf_counter()
    hist, it, st = H.solve(cfg.k, cfg.k, bv, xv, cfg.tol, fx["max_iter"])
    dt = time.perf_counter() - t0
    ho = fx["history_f"]
    n = min(hist.size, ho.size)
    d = np.abs(hist[:n] / hist[0] - ho[:n] / ho[0])
    betas = [abs(H.beta(l) - float.fromhex(fx["level"][l]["beta"])) / float.fromhex(fx["level"][l]["beta"])
             for l in range(1, H.levels)]
    return {"case": case, "iters_gpu": int(it), "iters_cpu": fx["iterations"], "status_gpu": int(st),
            "status_cpu": fx["status"], "max_abs_drho": float(d.max()), "max_rel_dbeta": float(max(betas)),
            "tol": cfg.tol, "solve_s": round(dt, 2),
            "oracle": "tests/golden/" + os.path.basename(path_for(case))}


def time_cycles(ctx, stream, H, bv, xv, k, steps, ws=1):
    import torch
    import torch.distributed as dist
    for _ in range(3):
        H.v_cycle(k, k, bv, xv)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        H.v_cycle(k, k, bv, xv)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def measure_batch(ctx, stream, H, b, k, K, steps, name):
    """K independent right-hand sides per cycle, interleaved per scalar row: one
    stream of every matrix serves all K (each RHS bitwise the single cycle)."""
    import torch

    from paper_2509_06744_b200 import Vector
    B = np.stack([np.roll(b, 7 * v) for v in range(K)], axis=1).ravel().copy()
    bv, xv = Vector(ctx, B), Vector(ctx, B.size)
    for _ in range(3):
        H.v_cycle_batch(k, k, K, bv, xv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        H.v_cycle_batch(k, k, K, bv, xv)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    by = H.cycle_bytes(k, k, K)
    return {"workload": f"{name} hierarchy, {K} right-hand sides per V({k},{k}) cycle (bmg_vcycle_batch)",
            "value": K * 1e3 / ms, "unit": "right-hand-side V-cycles/s", "ms_per_batch": ms,
            "batch_bytes": by, "effective_gbs": by / ms / 1e6}


def measure_c1(ctx, stream, steps, with_cpu=False):
    """BASELINE configs[0] (C1): one fourth-kind smoother application, k = 3, static
    block-FSAI lower(P(A)) on the 64^2 m = 10 operator.  Working set ~0.09 GB, so
    the number is L2-resident by construction (labelled so)."""
    import torch

    from paper_2509_06744_b200 import (FSAI_STATIC_LOWER, BlockSparseMatrix, Fsai, Vector, cheb_fourth_apply,
                                       lanczos_lambda_max)
    from paper_2509_06744_b200 import problems as pr

    c1 = pr.CONFIGS["C1"]
    A = pr.stencil_matrix(c1.dim, c1.n, c1.power, c1.m, c1.seed, c1.reg)
    dA = BlockSparseMatrix(ctx, A)
    M = Fsai.build(dA, FSAI_STATIC_LOWER)
    beta = lanczos_lambda_max(dA, M, 100, 1.01, 42)
    b = Vector(ctx, pr.normal_vector(A.dim_r, c1.seed, 0))
    x = Vector(ctx, pr.normal_vector(A.dim_r, c1.seed, 3))
    for _ in range(5):
        cheb_fourth_apply(dA, M, b, x, beta, c1.k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(steps, 50)
    e0.record(stream)
    for _ in range(reps):
        cheb_fourth_apply(dA, M, b, x, beta, c1.k)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    n = A.dim_r
    g, gt = M.G, M.G.transpose()
    per = c1.k * (dA.info()["pass_bytes"] + 24 * n + g.info()["pass_bytes"] + gt.info()["pass_bytes"] + 56 * n)
    out = {"workload": "C1: 64^2 patches, m=10, static block-FSAI lower(P(A)), one cheb4 application k=3",
           "value": 1e3 / ms, "unit": "smoother applications/s", "ms": ms, "bytes_per_application": per,
           "gbs": per / ms / 1e6, "l2": "L2-resident (0.09 GB working set < 126 MB L2)"}
    if with_cpu:  # the same application on the CPU oracle (the reference's own CPU-runnable case)
        from oracle import pyoracle as O
        om = O.Mat(A)
        of = O.Fsai(om, O.Fsai.STATIC)
        bh, xh = b.download(), x.download()
        for threads in (os.cpu_count() or 1, 1):
            O.set_threads(threads)
            O.smoother_apply(om, of, O.CHEB_FOURTH, bh, xh, c1.k, beta=beta)
            t0 = time.perf_counter()
            reps_c = 0
            while time.perf_counter() - t0 < 1.0:
                O.smoother_apply(om, of, O.CHEB_FOURTH, bh, xh, c1.k, beta=beta)
                reps_c += 1
            rate = reps_c / (time.perf_counter() - t0)
            out["cpu_oracle_threads" if threads > 1 else "cpu_oracle_1_thread"] = {
                "value": rate, "unit": "smoother applications/s", "cores": threads}
        O.set_threads(os.cpu_count() or 1)
    return out


def measure_extra(ctx, stream, cfg, steps, batch=0, with_cpu=False, parity=None):
    """Extra line: V(k,k) cycles/s of another config's whole device hierarchy."""
    import torch
    from paper_2509_06744_b200 import Vector

    t0 = time.perf_counter()
    H, b = whole_hierarchy(ctx, cfg)
    ctx.sync()
    setup_s = time.perf_counter() - t0
    bv, xv = Vector(ctx, b), Vector(ctx, b.size)
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    time.sleep(0.3)
    ms = time_cycles(ctx, stream, H, bv, xv, cfg.k, steps)
    clocks = sampler.stop()
    cb = H.cycle_bytes(cfg.k, cfg.k)
    peak, _ = hbm_peak()
    out = {"workload": config_dict(cfg)["workload"], "value": 1e3 / ms, "unit": "V-cycles/s", "ms_per_step": ms,
           "cycle_bytes": cb, "effective_gbs": cb / ms / 1e6, "frac_of_roofline": cb / ms / 1e6 / peak,
           "device_gb": H.device_bytes / 1e9, "setup_s": round(setup_s, 1), "clocks": clocks}
    if batch > 1:
        out[f"x{batch}"] = measure_batch(ctx, stream, H, b, cfg.k, batch, max(steps // 2, 3), cfg.name)
    del H, bv, xv
    ctx.sync()
    if parity:
        out["parity"] = parity_check(ctx, parity)
    if with_cpu:
        threads = os.cpu_count() or 1
        s = oracle_sample(cfg, 2, 0, threads)
        out["cpu_baseline"] = {"value": s["value"], "unit": "V-cycles/s", "cores": threads, "kind": "port",
                               "sample": sample_text(s, threads, cfg)}
    return out


def residual_roofline(ctx, stream, H, bv, xv, n_own, m):
    """The dominant kernel -- the finest-level residual pass r = b - A x
    (bsr_stream_kernel<m,m,1,EpiResidual>, 2k+1 launches per cycle) -- timed alone
    with CUDA events on the launching stream."""
    import torch
    from paper_2509_06744_b200 import Vector, residual
    Af, _, _ = H.level(H.levels - 1)
    rv = Vector(ctx, n_own)
    reps = 20
    residual(Af, bv, xv, rv)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for _ in range(reps):
        residual(Af, bv, xv, rv)
    k1.record(stream)
    torch.cuda.synchronize()
    kern_ms = k0.elapsed_time(k1) / reps
    sym = Af.sym_info()
    kern_bytes = sym["pass_bytes"] + 24 * n_own
    achieved = kern_bytes / (kern_ms / 1e3) / 1e9
    try:
        rpeak = read_peak_gbs()
    except Exception:
        rpeak = None
    peak, peak_kind = hbm_peak()
    traffic, tsrc = None, None
    try:
        with open(TRAFFIC_FILE) as f:
            t = json.load(f)
        ent = t.get(f"residual_m{m}" + ("_sym" if sym["half"] else ""))
        if ent and ent.get("algorithmic_bytes") == kern_bytes:
            traffic, tsrc = ent["dram_bytes_per_launch"], ent["source"]
    except Exception:
        pass
    kname = (f"bsr_stream_kernel<{m},{m},1,EpiStore,0,1> + sym_merge_kernel<{m},EpiResidual> (finest A, r = b - A x "
             f"with the lower triangle streamed; both launches timed as one pass)" if sym["half"] else
             f"bsr_stream_kernel<{m},{m},1,EpiResidual> (finest A, r = b - A x)")
    return {"bound": "hbm", "kernel": kname,
            "full_storage_pass_ms": sym["full_ms"] or None, "half_storage_pass_ms": sym["half_ms"] or None,
            "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": tsrc, "traffic_over_algorithmic": (traffic / kern_bytes)
            if traffic else None, "frac_of_nominal_8000": achieved / 8000.0, "read_peak_gbs": rpeak,
            "frac_of_read_peak": (achieved / rpeak) if rpeak else None, "bytes_per_launch": kern_bytes,
            "ms_per_launch": kern_ms}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2509_06744_b200 import Context, Vector
    from paper_2509_06744_b200 import problems as pr

    if ws > 1:
        uid = [Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = Context(local, nccl=(rank, ws, uid[0]))
    else:
        ctx = Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    def all_min(v):
        if ws == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return int(t.item())

    agglomerate = AGGLOMERATE.get(cfg.name, 1)
    run_info = {}
    t0 = time.perf_counter()
    if ws > 1 and not args.replicas:
        # partition invariance through the real transport on a scaled copy first
        small = cfg.scaled(max(cfg.n // 4, 2 ** (cfg.levels + 1)))
        invariance_check(ctx, small, ws, rank, agglomerate, all_min)
        H, b_own = partitioned_hierarchy(ctx, cfg, ws, rank, agglomerate)
        scaling = "strong"
        run_info["parallelism"] = (f"row strips x{ws} (distributed setup, NCCL halo exchanges in the captured cycle, "
                                   f"coarsest {agglomerate} level(s) on rank 0; verified bitwise against the 1-GPU "
                                   f"cycle on {small.name})")
        plan = pr.memory_plan(cfg, ws, agglomerate, setup_params(cfg))
        run_info["memory_plan_gb"] = [round(p["peak_gb"], 1) for p in plan]
    else:
        H, b_own = whole_hierarchy(ctx, cfg)
        if ws == 1:
            H.partition(1, pr.level_grid(cfg)[2])  # residual-norm segmentation as in the N-GPU runs
        scaling = "weak" if ws > 1 else "strong"
        run_info["parallelism"] = f"replicas x{ws}" if ws > 1 else "single GPU"
    ctx.sync()
    setup_s = time.perf_counter() - t0
    dev = torch.tensor([H.device_bytes / 1e9], device="cuda")
    if ws > 1:
        gathered = [torch.zeros_like(dev) for _ in range(ws)]
        dist.all_gather(gathered, dev)
        run_info["rank_device_gb"] = [round(float(g.item()), 1) for g in gathered]
    else:
        run_info["rank_device_gb"] = [round(float(dev.item()), 1)]
    run_info["setup_s"] = round(setup_s, 2)
    levels_sym = []
    for l in range(1, H.levels):
        try:
            Al, _, _ = H.level(l)
            si = Al.sym_info()
        except Exception:  # a level this rank does not hold
            continue
        levels_sym.append({"level": l, "half_storage": si["half"], "half_ms": round(si["half_ms"], 4),
                           "full_ms": round(si["full_ms"], 4)})
    run_info["symmetric_half_A"] = levels_sym

    m, k = cfg.m, cfg.k
    n_own = b_own.size
    bv, xv = Vector(ctx, b_own), Vector(ctx, n_own)
    for _ in range(max(args.warmup, 3)):
        H.v_cycle(k, k, bv, xv)
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.profiler.start()  # `ncu --profile-from-start off` captures exactly the timed steps
    e0.record(stream)
    for _ in range(args.steps):
        H.v_cycle(k, k, bv, xv)
    e1.record(stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = ctx.launch_count - launches0
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per = ms / args.steps
    mult = ws if scaling == "weak" else 1
    rate = mult * args.steps / (ms / 1e3)
    cycle_bytes = H.cycle_bytes(k, k)
    if ws > 1 and scaling == "strong":  # every rank's share of the cycle's bytes
        cb = torch.tensor([float(cycle_bytes)], device="cuda", dtype=torch.float64)
        dist.all_reduce(cb)
        cycle_bytes = int(cb.item())
    peak, peak_kind = hbm_peak()
    eff_gbs = mult * cycle_bytes / (ms_per / 1e3) / 1e9
    if ws == 1:
        ref_bytes = H.cycle_bytes_ref(k, k)
        run_info["cycle_bytes_reference_storage"] = ref_bytes
        if cfg.name in CYCLE_BYTES and CYCLE_BYTES[cfg.name] != ref_bytes:
            run_info["cycle_bytes_table_mismatch"] = {"table": CYCLE_BYTES[cfg.name], "device": ref_bytes}

    roof = residual_roofline(ctx, stream, H, bv, xv, n_own, m)

    # ---- e2e through the public C ABI (bmg_vcycle_host) with pinned host buffers
    hb = torch.from_numpy(b_own).pin_memory()
    hx = torch.zeros(n_own, dtype=torch.float64).pin_memory()
    for _ in range(2):
        H.v_cycle_host_ptr(k, k, hb.data_ptr(), hx.data_ptr())
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q0.record(stream)
    for _ in range(args.steps):
        H.v_cycle_host_ptr(k, k, hb.data_ptr(), hx.data_ptr())
    q1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = q0.elapsed_time(q1)
    if ws > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_rate = mult * args.steps / (e2e_ms / 1e3)
    del hb, hx

    extra = None
    parity = None
    cpu = None
    if rank == 0 and ws == 1:
        extra = {}
        if not args.no_batch:
            try:  # the same hierarchy on 4 right-hand sides per cycle (bmg_vcycle_batch)
                extra[f"{cfg.name}x4"] = measure_batch(ctx, stream, H, b_own, k, 4, max(args.steps // 2, 3), cfg.name)
            except Exception as e:
                extra[f"{cfg.name}x4"] = {"error": f"{type(e).__name__}: {e}"}
        del H, bv, xv
        ctx.sync()
        torch.cuda.empty_cache()
        if not args.no_parity and cfg.name in PARITY_CASE:
            parity = parity_check(ctx, PARITY_CASE[cfg.name])
        if not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            s = oracle_sample(cfg, 2, 1, threads, single_core=not args.no_single_core)
            cpu = {"value": s["value"], "unit": "V-cycles/s", "cores": threads, "kind": "port",
                   "sample": sample_text(s, threads, cfg)}
            if "single_core" in s:
                cpu["single_core"] = {"value": s["single_core"]["value"], "unit": "V-cycles/s", "cores": 1,
                                      "sample": "1 V-cycle of the same sample on one thread, scaled the same way "
                                                "(the reference is single-threaded, SURVEY.md §0.1)"}
            try:
                rb = reference_build_sample(cfg)
                if rb is not None:
                    cpu["reference_build"] = rb
            except Exception as e:
                cpu["reference_build"] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_extra:
            try:
                extra["C1"] = measure_c1(ctx, stream, args.steps, with_cpu=not args.no_cpu_baseline)
            except Exception as e:  # secondary lines never fail the headline run
                extra["C1"] = {"error": f"{type(e).__name__}: {e}"}
            others = [("C2", pr.CONFIGS["C2"], 8, True, "C2")]
            others += [("C3@512", pr.CONFIGS["C3"].scaled(512), 0, False, None),
                       ("C5@1024", pr.CONFIGS["C5"].scaled(1024), 0, False, None)]
            if cfg.name != "C4":
                others.append(("C4", pr.CONFIGS["C4"], 4, False, None))
            for key, c, batch, with_cpu, par in others:
                if c.name == cfg.name:
                    continue
                try:
                    extra[key] = measure_extra(ctx, stream, c, min(args.steps, 10), batch,
                                               with_cpu=with_cpu and not args.no_cpu_baseline, parity=par)
                    if "@" in key:
                        extra[key]["note"] = "reduced size: a quarter of the named config's fine rows, same shape"
                except Exception as e:
                    extra[key] = {"error": f"{type(e).__name__}: {e}"}
                torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": f"V-cycles/s ({cfg.name}, V({k},{k}))",
            "value": rate,
            "unit": "V-cycles/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": max(args.warmup, 3),
            "ms_per_step": ms_per,
            "higher_is_better": True,
            "scaling": scaling,
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE.md §3 generator bmggen/, seed 0; hierarchy built on the device)",
            "config": config_dict(cfg),
            "run": run_info,
            "effective_gbs": eff_gbs,
            "cycle_bytes": cycle_bytes,
            "frac_of_roofline_cycle": eff_gbs / peak,
            "roofline": roof,
            "clocks": clocks,
            "e2e": {"value": e2e_rate, "unit": "V-cycles/s", "h2d_bytes_per_step": 2 * 8 * n_own,
                    "d2h_bytes_per_step": 8 * n_own, "path": "bmg_vcycle_host (C ABI), pinned host b and x"},
            "gpu_launches": launches,
        }
        if parity is not None:
            line["parity"] = parity
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if extra is not None:
            line["extra_configs"] = extra
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of row strips")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra config lines (C1, C2, C3/C5 shapes)")
    ap.add_argument("--no-batch", action="store_true", help="skip the 4-right-hand-side line")
    ap.add_argument("--no-parity", action="store_true", help="skip the solve-to-1e-8 parity check")
    ap.add_argument("--no-single-core", action="store_true", help="skip the 1-thread oracle cycle")
    args = ap.parse_args()
    from paper_2509_06744_b200 import problems as pr

    cfg = pr.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
