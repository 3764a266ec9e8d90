"""Multi-rank (world_size 2, gloo, CPU) check of the partitioned V-cycle's host
logic: the row partition (bmg_partition_rows), the per-level vector windows
(bmg_row_window) and the contiguous-slice halo protocol that hierarchy.cu's
exchange() implements with NCCL.  Each rank keeps only its strip, exchanges halos
with torch.distributed send/recv, applies A, R = P^T and P to its rows with the
oracle, and the gathered result must equal the unpartitioned product bitwise.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice(h, lo, hi, col_lo, ncols):
    from paper_2509_06744_b200.api import HostBsr

    m_r, m_c = int(h.row_sizes[0]), int(h.col_sizes[0])
    p0, p1 = int(h.row_ptr[lo]), int(h.row_ptr[hi])
    rp = h.row_ptr[lo:hi + 1] - p0
    ci = h.col_idx[p0:p1] - col_lo
    assert ci.size == 0 or (ci.min() >= 0 and ci.max() < ncols)
    vals = h.vals[p0 * m_r * m_c:p1 * m_r * m_c]
    return HostBsr(np.full(hi - lo, m_r, np.int32), np.full(ncols, m_c, np.int32), rp, ci, vals)


def _exchange(buf, m, bounds, wlo, whi, rank, world):
    """hierarchy.cu exchange(): send own rows inside each peer's window, receive
    each peer's own rows inside mine (contiguous slices)."""
    import torch

    reqs = []
    for s in range(world):
        if s == rank:
            continue
        a0, a1 = max(bounds[rank], wlo[s]), min(bounds[rank + 1], whi[s])
        if a1 > a0:
            t = torch.from_numpy(np.ascontiguousarray(buf[(a0 - wlo[rank]) * m:(a1 - wlo[rank]) * m]))
            reqs.append(dist.isend(t, s))
    for s in range(world):
        if s == rank:
            continue
        b0, b1 = max(bounds[s], wlo[rank]), min(bounds[s + 1], whi[rank])
        if b1 > b0:
            t = torch.zeros((b1 - b0) * m, dtype=torch.float64)
            dist.recv(t, s)
            buf[(b0 - wlo[rank]) * m:(b1 - wlo[rank]) * m] = t.numpy()
    for r in reqs:
        r.wait()


def _worker(rank, world, port, agglomerate, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from oracle import pyoracle as O
    from paper_2509_06744_b200 import problems as pr
    from paper_2509_06744_b200.api import partition_rows, row_window

    cfg = pr.CONFIGS["C2"].scaled(16, 2)
    m = cfg.m
    A1, (P1,), b = pr.make_problem(cfg)           # fine level 16^2, prolongation from 8^2
    A0 = O.galerkin(O.Mat(A1), O.Mat(P1)).export(symmetric=True)
    R1 = O.Mat(P1)                                 # R = P^T applied with spmv_t below
    levels = [A0, A1]
    gran = [8, 16]
    bounds = [partition_rows(A.row_ptr, world, gran[l], agglomerate=(l == 0 and agglomerate)) for l, A in
              enumerate(levels)]
    # R as an explicit matrix (rows: coarse, cols: fine) for the row-wise protocol
    Rh = O.Mat(P1)
    rp = np.zeros(A0.nbr + 1, np.int64)
    cols = [[] for _ in range(A0.nbr)]
    vals = [[] for _ in range(A0.nbr)]
    for i in range(P1.nbr):
        for p in range(P1.row_ptr[i], P1.row_ptr[i + 1]):
            j = P1.col_idx[p]
            cols[j].append(i)
            vals[j].append(P1.vals[p * m * m:(p + 1) * m * m].reshape(m, m).T.ravel())
    from paper_2509_06744_b200.api import HostBsr

    for j in range(A0.nbr):
        rp[j + 1] = rp[j] + len(cols[j])
    R = HostBsr(np.full(A0.nbr, m, np.int32), np.full(A1.nbr, m, np.int32), rp,
                np.array([c for cc in cols for c in cc], np.int32), np.concatenate([v for vv in vals for v in vv]))
    # windows: level 1 is read by A1 (own rows) and R (coarse own rows); level 0 by A0 and P1
    W = {}
    for l in (0, 1):
        W[l] = ([0] * world, [0] * world)
        for r in range(world):
            lo, hi = bounds[l][r], bounds[l][r + 1]
            hull = []
            if l == 1:
                hull.append(row_window(A1.row_ptr, A1.col_idx, lo, hi, lo, hi))
                hull.append(row_window(R.row_ptr, R.col_idx, bounds[0][r], bounds[0][r + 1], lo, hi))
            else:
                hull.append(row_window(A0.row_ptr, A0.col_idx, lo, hi, lo, hi))
                hull.append(row_window(P1.row_ptr, P1.col_idx, bounds[1][r], bounds[1][r + 1], lo, hi))
            hull = [h for h in hull if h[1] > h[0]]
            W[l][0][r] = min(h[0] for h in hull) if hull else 0
            W[l][1][r] = max(h[1] for h in hull) if hull else 0
    # global vectors (every rank can generate them; each keeps its own rows only)
    x1 = pr.normal_vector(A1.dim_r, 0, 11)
    x0 = pr.normal_vector(A0.dim_r, 0, 12)
    res = {}
    for l, A, x in ((1, A1, x1), (0, A0, x0)):
        lo, hi = bounds[l][rank], bounds[l][rank + 1]
        wl, wh = W[l][0][rank], W[l][1][rank]
        buf = np.zeros((wh - wl) * m)
        buf[(lo - wl) * m:(hi - wl) * m] = x[lo * m:hi * m]
        _exchange(buf, m, bounds[l], W[l][0], W[l][1], rank, world)
        y = O.Mat(_slice(A, lo, hi, wl, wh - wl)).spmv(buf) if hi > lo else np.zeros(0)
        res[f"A{l}"] = (lo, y)
        if l == 1:  # restriction rc = R r for the coarse own rows
            c0, c1 = bounds[0][rank], bounds[0][rank + 1]
            res["R"] = (c0, O.Mat(_slice(R, c0, c1, wl, wh - wl)).spmv(buf) if c1 > c0 else np.zeros(0))
        else:  # prolongation P x0 for the fine own rows
            f0, f1 = bounds[1][rank], bounds[1][rank + 1]
            res["P"] = (f0, O.Mat(_slice(P1, f0, f1, wl, wh - wl)).spmv(buf) if f1 > f0 else np.zeros(0))
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    if rank == 0:
        full = {}
        for key, n in (("A1", A1.dim_r), ("A0", A0.dim_r), ("R", A0.dim_r), ("P", A1.dim_r)):
            v = np.full(n, np.nan)
            for g in gathered:
                lo, y = g[key]
                v[lo * m:lo * m + y.size] = y
            full[key] = v
        want = {"A1": O.Mat(A1).spmv(x1), "A0": O.Mat(A0).spmv(x0), "R": R1.spmv_t(x1), "P": O.Mat(P1).spmv(x0)}
        out.put({k: bool(np.array_equal(full[k], want[k])) for k in want})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("agglomerate", [False, True])
def test_partitioned_halo_protocol_world2(agglomerate):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, agglomerate, q)) for r in range(2)]
    for p in procs:
        p.start()
    result = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(result.values()), result


def test_partition_rows_properties():
    from paper_2509_06744_b200 import problems as pr
    from paper_2509_06744_b200.api import partition_rows, row_window

    A = pr.stencil_matrix(2, 32, 2, 2)
    for world in (1, 2, 3, 4, 8):
        b = partition_rows(A.row_ptr, world, 32)
        assert b[0] == 0 and b[-1] == A.nbr and np.all(np.diff(b) >= 0)
        assert np.all(b % 32 == 0)  # strips of whole grid rows
        if world <= 4:
            sizes = np.diff(b)
            assert sizes.max() - sizes.min() <= 32
    agg = partition_rows(A.row_ptr, 4, 32, agglomerate=True)
    assert list(agg) == [0] + [A.nbr] * 4
    # 13-point stencil: the window of a strip reaches exactly 2 grid rows each side
    lo, hi = 10 * 32, 20 * 32
    assert row_window(A.row_ptr, A.col_idx, lo, hi, lo, hi) == (8 * 32, 22 * 32)
