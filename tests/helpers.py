"""Test fixtures: random block-sparse matrices (in the spirit of the reference's
testsup::random_layout / random_spd, proj/tests/test_support.hpp:10-44) and
conversions between the product's host BSR and the oracle."""
from __future__ import annotations

import numpy as np

from paper_2509_06744_b200.api import HostBsr


def random_layout(rng, max_blocks, max_size):
    n = 1 + int(rng.integers(max_blocks))
    return (1 + rng.integers(max_size, size=n)).astype(np.int32)


def random_bsr(rng, row_sizes, col_sizes, density, min_per_row=0, symmetric=False):
    """Random block-sparse matrix; blocks in (-1, 1)."""
    nbr, nbc = len(row_sizes), len(col_sizes)
    rows = []
    for i in range(nbr):
        cols = [j for j in range(nbc) if rng.uniform() < density]
        if len(cols) < min_per_row:
            extra = rng.choice(nbc, size=min(min_per_row, nbc), replace=False)
            cols = sorted(set(cols) | set(int(e) for e in extra))
        rows.append(sorted(cols))
    rp = np.zeros(nbr + 1, np.int64)
    for i in range(nbr):
        rp[i + 1] = rp[i] + len(rows[i])
    ci = np.array([j for r in rows for j in r], np.int32)
    vals = np.concatenate([rng.uniform(-1, 1, int(row_sizes[i]) * int(col_sizes[j]))
                           for i in range(nbr) for j in rows[i]]) if len(ci) else np.zeros(0)
    return HostBsr(row_sizes, col_sizes, rp, ci, vals, symmetric)


def from_dense_blocks(row_sizes, col_sizes, blocks: dict, symmetric=False):
    """blocks: {(i, j): ndarray}."""
    nbr = len(row_sizes)
    rows = [[] for _ in range(nbr)]
    for (i, j) in blocks:
        rows[i].append(j)
    rp = np.zeros(nbr + 1, np.int64)
    for i in range(nbr):
        rows[i].sort()
        rp[i + 1] = rp[i] + len(rows[i])
    ci = np.array([j for r in rows for j in r], np.int32)
    vals = np.concatenate([np.asarray(blocks[(i, j)], np.float64).ravel() for i in range(nbr) for j in rows[i]]) \
        if len(ci) else np.zeros(0)
    return HostBsr(row_sizes, col_sizes, rp, ci, vals, symmetric)


def random_spd(rng, sizes, density):
    """Symmetric, block diagonally dominant (s.p.d. by Gershgorin), both halves stored
    (test_support.hpp:25-44)."""
    n = len(sizes)
    blocks = {}
    for i in range(n):
        for j in range(i):
            if rng.uniform() < density:
                b = rng.uniform(-1, 1, (sizes[i], sizes[j]))
                blocks[(i, j)] = b
                blocks[(j, i)] = b.T.copy()
    for i in range(n):
        m = int(sizes[i])
        r = rng.uniform(-1, 1, (m, m))
        d = r + r.T
        off = 0.0
        for (a, b), blk in blocks.items():
            if a == i and b != i:
                off = max(off, np.abs(blk).sum(axis=1).max())
        d += (off * 1.0 + 2.0 * m + 3.0) * np.eye(m)
        # row sums over all off-diagonal blocks (Gershgorin across blocks)
        tot = sum(np.abs(blk).sum(axis=1).max() for (a, b), blk in blocks.items() if a == i and b != i)
        d += tot * np.eye(m)
        blocks[(i, i)] = d
    return from_dense_blocks(np.asarray(sizes, np.int32), np.asarray(sizes, np.int32), blocks, symmetric=True)
