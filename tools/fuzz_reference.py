"""Randomized campaign (CPU): the oracle against THE REFERENCE ITSELF
(oracle/_ref/libblockmg_ref.so, the reference's own sources -- oracle/ref_driver.cpp)
on random 2-D / 3-D hierarchies: block size, depth, nesting, t_max, smoother kind,
variable layouts, asymmetric cycles.  Every comparison is bitwise: each level's
Galerkin operator, FSAI chain factors, S-hat, beta_l, and the iterate after a
V(k_pre, k_post) cycle from a random start.
Usage: python tools/fuzz_reference.py SEED SECONDS"""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import pyoracle as O
from oracle import pyref as R
from paper_2509_06744_b200 import problems as pr


def digest(m):
    e = m.export()
    d = hashlib.sha256()
    for a in (e.row_ptr, e.col_idx, e.vals):
        d.update(np.ascontiguousarray(a).tobytes())
    return d.hexdigest()


rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
budget = float(sys.argv[2] if len(sys.argv) > 2 else 120)
O.set_threads(2)
t0 = time.time()
cases = fails = 0
by_m = {}
while time.time() - t0 < budget:
    dim = int(rng.choice([2, 2, 3]))
    levels = int(rng.integers(2, 4))
    n = int(rng.choice([8, 16])) if dim == 2 else 8
    m = int(rng.choice([3, 4, 6, 10, 15, 20, 21]))
    if dim == 3 and m > 10:
        n = 4 if levels == 2 else 8
    power = int(rng.choice([1, 2])) if dim == 3 else int(rng.choice([2, 3]))
    nest = int(rng.choice([0, 0, 1, 2]))
    t_max = int(rng.choice([1, 2, 3]))
    kind = int(rng.choice([0, 1, 2]))
    var = bool(rng.integers(0, 2)) and m == 10 and dim == 2
    cfg = pr.Config("f", dim, n, power, m, levels, "adaptive", 3, nest=nest, seed=int(rng.integers(100)))
    try:
        A, T, b = pr.make_variable_problem(cfg, 6) if var else pr.make_problem(cfg)
    except Exception:
        continue
    kpre, kpost = int(rng.integers(0, 4)), int(rng.integers(0, 4))
    if kpre + kpost == 0:
        kpost = 1
    kw = dict(t_max=t_max, nest=nest, coarse_dim_cap=1 << 30, smoother_kind=kind)
    try:
        oh = O.Hierarchy(O.Mat(A), [O.Mat(p) for p in T], probe=False, **kw)
    except O.OracleError as e:
        try:
            R.Hierarchy(R.Mat(A), [R.Mat(p) for p in T], **kw)
            print("FAIL only-the-oracle-raised", e.status, flush=True)
            fails += 1
        except R.OracleError as e2:
            if e2.status != e.status:
                print("FAIL statuses differ", e.status, e2.status, flush=True)
                fails += 1
        cases += 1
        continue
    rh = R.Hierarchy(R.Mat(A), [R.Mat(p) for p in T], **kw)
    bad = []
    for l in range(oh.levels()):
        if digest(oh.A(l)) != digest(rh.A(l)):
            bad.append(f"A{l}")
        if l >= 1:
            fo, fr = oh.fsai(l), rh.fsai(l)
            if fo.chain_len() != fr.chain_len() or any(
                    digest(fo.factor(q)) != digest(fr.factor(q)) for q in range(fo.chain_len())):
                bad.append(f"F{l}")
            if not np.array_equal(fo.shat(), fr.shat()):
                bad.append(f"S{l}")
            if oh.beta(l) != rh.beta(l):
                bad.append(f"beta{l}")
    x0 = rng.standard_normal(b.size)
    if not np.array_equal(oh.v_cycle(kpre, kpost, b, x0), rh.v_cycle(kpre, kpost, b, x0)):
        bad.append("cycle")
    cases += 1
    by_m[m] = by_m.get(m, 0) + 1
    if bad:
        fails += 1
        print("FAIL", bad, "dim", dim, "p", power, "n", n, "m", m, "L", levels, "nest", nest, "t", t_max, "kind", kind,
              "var", var, "k", kpre, kpost, flush=True)
print("cases", cases, "bitwise failures", fails, "by block size", dict(sorted(by_m.items())))
