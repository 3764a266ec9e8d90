#!/usr/bin/env python
"""Benchmark: V-cycle application of the multilevel Chebyshev(4th kind) + block-FSAI
solver (arXiv 2509.06744 hot path) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one V(k,k) cycle on the finest level of the config's hierarchy with the
inputs (hierarchy, b, x) resident in HBM.  Workload: config C2 (BASELINE.json
configs[1]: 256^2 patches, m = 10, 4 levels, V(3,3), adaptive block-FSAI), the
configs[1] case that fits one GPU; its per-cycle traffic (14+ GB) exceeds L2, so
no explicit flush is needed between cycles.  For N > 1 the hierarchy is split
into row strips per rank with NCCL halo exchanges inside the captured cycle and
the coarsest two levels on rank 0 (strong scaling); `--replicas`
runs independent copies instead (weak scaling).

One JSON line is printed by rank 0.  `--impl reference` times the CPU oracle
(the restatement of the reference, which cannot be built here) on the host cores.
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


# ------------------------------------------------------------------ CPU oracle arm
def oracle_vcycles(cfg, steps, warmup, threads, single_core=None):
    """Time V-cycles of the CPU oracle (restatement of the reference) on `threads`
    host threads: setup untimed, then warmup + `steps` cycles timed by wall clock."""
    from oracle import pyoracle as O
    from paper_2509_06744_b200 import problems as pr

    O.set_threads(threads)
    A, T, b = pr.make_problem(cfg)
    t0 = time.perf_counter()
    H = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], t_max=1, tau=1.0, nest=cfg.nest,
                    fsai_kind=0 if cfg.fsai == "static" else 3, coarse_dim_cap=1 << 30, probe=False)
    setup_s = time.perf_counter() - t0
    x = np.zeros_like(b)
    for _ in range(warmup):
        x = H.v_cycle(cfg.k, cfg.k, b, x)
    t0 = time.perf_counter()
    for _ in range(steps):
        x = H.v_cycle(cfg.k, cfg.k, b, x)
    dt = time.perf_counter() - t0
    if single_core is not None:
        # the reference itself is single-threaded: one cycle on one
        # thread is its faithful per-cycle cost
        O.set_threads(1)
        t1 = time.perf_counter()
        x = H.v_cycle(cfg.k, cfg.k, b, x)
        single_core.append(1.0 / (time.perf_counter() - t1))
        O.set_threads(threads)
    return steps / dt, setup_s, dt


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    steps = max(1, args.steps)
    warm = max(0, min(args.warmup, 3))
    rate, setup_s, dt = oracle_vcycles(cfg, steps, warm, threads)
    unit = "V-cycles/s"
    line = {
        "impl": "reference",
        "metric": f"V-cycles/s ({cfg.name}, V({cfg.k},{cfg.k}))",
        "value": rate, "unit": unit, "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * dt / steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.md §3 generator, seed 0)",
        "config": {"workload": f"{cfg.name}: {cfg.n}^{cfg.dim} patches, m={cfg.m}, {cfg.levels} levels, "
                               f"V({cfg.k},{cfg.k}), {cfg.fsai} block-FSAI t_max=1"},
        "cpu_baseline": {"value": rate, "unit": unit, "cores": threads, "kind": "port",
                         "sample": f"{steps} V-cycles of the C++ oracle (reference restatement; the reference "
                                   f"itself needs Eigen3, absent) after {setup_s:.0f}s untimed setup; "
                                   f"CPU {cpu_info()}"},
        "e2e": {"value": rate, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
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


def measure_hierarchy(ctx, stream, cfg, steps, batch=0):
    """Extra line: V(k,k) cycles/s of another config's full device hierarchy (and,
    with batch=K, the same hierarchy on K right-hand sides per cycle)."""
    import torch

    from paper_2509_06744_b200 import BlockSparseMatrix, Hierarchy, Vector, default_params
    from paper_2509_06744_b200 import problems as pr

    t0 = time.perf_counter()
    A, T, b = pr.make_problem(cfg)
    dA = BlockSparseMatrix(ctx, A)
    dT = [BlockSparseMatrix(ctx, p) for p in T]
    del A, T
    H = Hierarchy.setup(dA, dT, default_params(t_max=1, coarse_dim_cap=1 << 30, nest=cfg.nest))
    ctx.sync()
    setup_s = time.perf_counter() - t0
    bv, xv = Vector(ctx, b), Vector(ctx, b.size)
    for _ in range(3):
        H.v_cycle(cfg.k, cfg.k, bv, xv)
    torch.cuda.synchronize()
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        H.v_cycle(cfg.k, cfg.k, bv, xv)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / steps
    cb = H.cycle_bytes(cfg.k, cfg.k)
    peak, _ = hbm_peak()
    out = {"workload": f"{cfg.name}: {cfg.n}^{cfg.dim} patches, m={cfg.m}, {cfg.levels} levels, V({cfg.k},{cfg.k})",
           "value": 1e3 / ms, "unit": "V-cycles/s", "ms_per_step": ms, "cycle_bytes": cb,
           "effective_gbs": cb / ms / 1e6, "frac_of_roofline": cb / ms / 1e6 / peak,
           "device_gb": H.device_bytes / 1e9, "setup_s": round(setup_s, 1), "clocks": clocks}
    if batch > 1:
        try:
            out[f"x{batch}"] = measure_batch(ctx, stream, H, b, cfg.k, batch, max(steps // 2, 3), cfg.name)
        except Exception as e:
            out[f"x{batch}"] = {"error": f"{type(e).__name__}: {e}"}
    del H, dA, dT, bv, xv
    ctx.sync()
    return out


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, Vector, default_params, residual
    from paper_2509_06744_b200 import problems as pr

    mode = "single GPU"
    if ws > 1:
        uid = [Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = Context(local, nccl=(rank, ws, uid[0]))
    else:
        ctx = Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    A, T, b = pr.make_problem(cfg)
    dA = BlockSparseMatrix(ctx, A)
    dT = [BlockSparseMatrix(ctx, p) for p in T]
    t0 = time.perf_counter()
    params = default_params(t_max=1, tau=1.0, nest=cfg.nest, coarse_dim_cap=1 << 30,
                            fsai_kind=0 if cfg.fsai == "static" else 3)
    H = Hierarchy.setup(dA, dT, params)
    granule = [(cfg.n >> (cfg.levels - 1 - l)) ** (cfg.dim - 1) for l in range(cfg.levels)]
    agglomerate = 1  # the dense coarsest level on rank 0; every other level stays split
    cycle_bytes = H.cycle_bytes(cfg.k, cfg.k)
    n = A.dim_r
    lo_row, hi_row = 0, A.nbr
    scaling = "weak" if (ws > 1 and args.replicas) else "strong"
    if ws > 1 and not args.replicas:
        try:
            # reference result of two unpartitioned cycles (every rank has the whole hierarchy)
            H.partition(1, granule)
            x_ref = Vector(ctx, n)
            b_all = Vector(ctx, b)
            for _ in range(2):
                H.v_cycle(cfg.k, cfg.k, b_all, x_ref)
            x_ref_h = x_ref.download()
            del x_ref, b_all
            del H
            try:
                # the scalable route: every rank builds only its extended strips
                # (bmg_hier_setup_dist); no rank holds a whole partitioned level
                _, _, gran_l, rad_l = pr.level_grid(cfg)
                A_ext, T_ext, _, _ = pr.dist_inputs(cfg, ws, rank, agglomerate, params)
                H = Hierarchy.setup_dist(ctx, BlockSparseMatrix(ctx, A_ext),
                                         [BlockSparseMatrix(ctx, p) for p in T_ext], gran_l, rad_l, agglomerate,
                                         params)
                del A_ext, T_ext
                setup_kind = "distributed setup"
            except Exception as e:  # every rank builds the whole hierarchy and keeps its strip
                H = Hierarchy.setup(dA, dT, params)
                H.partition(ws, granule, agglomerate=agglomerate, rank=rank)
                setup_kind = f"replicated setup ({type(e).__name__} in the distributed one)"
            lo_row, hi_row, _, _ = H.part_info(cfg.levels - 1, rank)
            # the partitioned cycle must reproduce it bitwise on every rank's strip
            m_ = cfg.m
            bp = Vector(ctx, np.ascontiguousarray(b[lo_row * m_:hi_row * m_]))
            xp = Vector(ctx, (hi_row - lo_row) * m_)
            for _ in range(2):
                H.v_cycle(cfg.k, cfg.k, bp, xp)
            ok = bool(np.array_equal(xp.download(), x_ref_h[lo_row * m_:hi_row * m_]))
            flags = torch.tensor([1 if ok else 0], device="cuda")
            dist.all_reduce(flags, op=dist.ReduceOp.MIN)
            if flags.item() != 1:
                raise RuntimeError("partitioned V-cycle differs from the 1-GPU cycle")
            del bp, xp
            mode = (f"row strips x{ws} ({setup_kind}, NCCL halos, coarsest {agglomerate} level(s) on rank 0; "
                    f"verified bitwise against the 1-GPU cycle)")
            scaling = "strong"
        except Exception as e:  # keep the run alive: independent replicas instead
            H = Hierarchy.setup(dA, dT, params)
            lo_row, hi_row = 0, A.nbr
            mode = f"replicas x{ws} (partitioned path failed: {type(e).__name__}: {e})"
            scaling = "weak"
    elif ws > 1:
        mode = f"replicas x{ws}"
    else:
        H.partition(1, granule)  # residual-norm segmentation identical to the N-GPU runs
    ctx.sync()
    setup_s = time.perf_counter() - t0
    m = cfg.m
    b_own = np.ascontiguousarray(b[lo_row * m:hi_row * m])
    n_own = b_own.size
    bv = Vector(ctx, b_own)
    xv = Vector(ctx, n_own)
    k = cfg.k

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
    rate = (1 if scaling == "strong" else ws) * args.steps / (ms / 1e3)
    cycle_bytes = H.cycle_bytes(k, k)
    peak, peak_kind = hbm_peak()
    eff_gbs = (1 if scaling == "strong" else ws) * cycle_bytes / (ms_per / 1e3) / 1e9

    # ---- dominant kernel: finest-level residual pass r = b - A x (2k+1 per cycle)
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
    inf = Af.info()
    kern_bytes = inf["pass_bytes"] + 24 * n_own
    achieved = kern_bytes / (kern_ms / 1e3) / 1e9
    try:
        rpeak = read_peak_gbs()
    except Exception:
        rpeak = None
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as f:
                traffic = json.load(f).get("residual_dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e through the public C ABI with pinned host buffers
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
    e2e_rate = (1 if scaling == "strong" else ws) * args.steps / (e2e_ms / 1e3)

    extra = None
    if rank == 0 and ws == 1:
        extra = {}
        try:
            extra["C1"] = measure_c1(ctx, stream, args.steps, with_cpu=not args.no_cpu_baseline)
        except Exception as e:  # secondary lines never fail the headline run
            extra["C1"] = {"error": f"{type(e).__name__}: {e}"}
        try:  # the same hierarchy on 8 right-hand sides per cycle (bmg_vcycle_batch)
            extra["C2x8"] = measure_batch(ctx, stream, H, b_own, k, 8, args.steps)
        except Exception as e:
            extra["C2x8"] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_c4 or not args.no_quarter:
            # the large lines: free the headline hierarchy first
            del H, dA, dT, bv, xv, rv
            ctx.sync()
        if not args.no_quarter:
            # C3 and C5 do not fit one GPU; their shapes (C3: nested FSAI, m = 21, 25-pt,
            # V(4,4), 5 levels; C5: m = 15, 6 levels) at a quarter of the rows do
            for key, c in (("C3@512", pr.CONFIGS["C3"].scaled(512)), ("C5@1024", pr.CONFIGS["C5"].scaled(1024))):
                try:
                    extra[key] = measure_hierarchy(ctx, stream, c, min(args.steps, 10))
                    extra[key]["note"] = "reduced size: a quarter of the named config's fine rows, same shape"
                except Exception as e:
                    extra[key] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_c4:
            try:
                free = torch.cuda.mem_get_info()[0]
                if free < 125e9:
                    extra["C4"] = {"skipped": f"needs ~115 GB free, {free / 1e9:.0f} GB available"}
                else:
                    extra["C4"] = measure_hierarchy(ctx, stream, pr.CONFIGS["C4"], min(args.steps, 10), batch=4)
            except Exception as e:
                extra["C4"] = {"error": f"{type(e).__name__}: {e}"}

    # ---- CPU baseline (rank 0, N = 1 only): bounded oracle sample
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        one = [] if not args.no_single_core else None
        crate, csetup, cdt = oracle_vcycles(cfg, 2, 0, threads, one)
        cpu = {"value": crate, "unit": "V-cycles/s", "cores": threads, "kind": "port",
               "sample": f"2 V-cycles of the C++ oracle (reference restatement) on {cfg.name} after "
                         f"{csetup:.0f}s untimed setup, {threads} OpenMP threads, CPU {cpu_info()}"}
        if one:
            cpu["single_core"] = {"value": one[0], "unit": "V-cycles/s", "cores": 1,
                                  "sample": f"1 V-cycle of the oracle on one thread ({cfg.name}, same hierarchy)"}

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
            "data": "synthetic (BASELINE.md §3 generator, seed 0; random-init hierarchy built on the device)",
            "config": {"workload": f"{cfg.name}: {cfg.n}^{cfg.dim} patches, m={cfg.m}, {cfg.levels} levels, "
                                   f"V({k},{k}), {cfg.fsai} block-FSAI t_max=1",
                       "parallelism": mode,
                       "l2": "inputs larger than L2 (>= 14 GB streamed per cycle)",
                       "setup_s": round(setup_s, 2)},
            "effective_gbs": eff_gbs,
            "cycle_bytes": cycle_bytes,
            "frac_of_roofline_cycle": eff_gbs / peak,
            "roofline": {"bound": "hbm", "kernel": "bsr_stream_kernel<10,10,1,EpiResidual> (finest A, r = b - A x)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "frac_of_nominal_8000": achieved / 8000.0,
                         "read_peak_gbs": rpeak, "frac_of_read_peak": (achieved / rpeak) if rpeak else None,
                         "bytes_per_launch": kern_bytes, "ms_per_launch": kern_ms},
            "clocks": clocks,
            "e2e": {"value": e2e_rate, "unit": "V-cycles/s", "h2d_bytes_per_step": 2 * 8 * n_own,
                    "d2h_bytes_per_step": 8 * n_own},
            "gpu_launches": launches,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if extra is not None:
            line["extra_configs"] = extra
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def measure_batch(ctx, stream, H, b, k, K, steps, name="C2"):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of row strips")
    ap.add_argument("--no-c4", action="store_true", help="skip the extra C4 (largest single-GPU config) line")
    ap.add_argument("--no-single-core", action="store_true", help="skip the 1-thread oracle cycle")
    ap.add_argument("--no-quarter", action="store_true", help="skip the quarter-size C3 / C5 shape lines")
    args = ap.parse_args()
    from paper_2509_06744_b200 import problems as pr

    cfg = pr.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
