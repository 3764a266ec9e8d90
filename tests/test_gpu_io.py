"""The reference's text exchange format (matrix_io.hpp:15-27, matrix_io.cpp:39-149)
read into / written from device objects: bitwise round trips, the symmetry-flag
restore, and IoError{line} on malformed input (test_blockcore.cpp:161-208)."""
import os

import numpy as np
import pytest

from paper_2509_06744_b200 import IoError, Vector, read_matrix, read_vector, write_matrix, write_vector
from paper_2509_06744_b200 import problems as pr
from tests.helpers import random_bsr, random_layout, random_spd

pytestmark = pytest.mark.gpu


def _write_reference_format(h, path):
    """write_matrix (matrix_io.cpp:39-58), restated for the test fixture."""
    ro = np.concatenate([[0], np.cumsum(h.row_sizes)])
    co = np.concatenate([[0], np.cumsum(h.col_sizes)])
    lines = []
    v = 0
    for i in range(h.nbr):
        for p in range(h.row_ptr[i], h.row_ptr[i + 1]):
            j = h.col_idx[p]
            mi, mj = int(h.row_sizes[i]), int(h.col_sizes[j])
            for r in range(mi):
                for c in range(mj):
                    lines.append(f"{ro[i] + r + 1} {co[j] + c + 1} {float(h.vals[v + r * mj + c]):.17g}")
            v += mi * mj
    with open(path, "w") as f:
        f.write(f"%%block-matrix {ro[-1]} {co[-1]} {len(lines)}\n")
        f.write("\n".join(lines) + ("\n" if lines else ""))
    with open(path + ".blocks", "w") as f:
        f.write("".join(f"{m}\n" for m in h.row_sizes))


def test_matrix_round_trip_bitwise(ctx, rng, tmp_path):
    for rep in range(4):
        sizes = random_layout(rng, 8, 4)
        h = random_spd(rng, sizes, 0.5) if rep % 2 else random_bsr(rng, sizes, sizes, 0.5)
        p = str(tmp_path / f"a{rep}.mtx")
        _write_reference_format(h, p)
        A, sym = read_matrix(ctx, p)
        assert sym == bool(rep % 2)
        got = A.download(sizes, sizes)
        assert np.array_equal(got.row_ptr, h.row_ptr) and np.array_equal(got.col_idx, h.col_idx)
        assert np.array_equal(got.vals, h.vals)
        q = str(tmp_path / f"b{rep}.mtx")
        write_matrix(A, q)
        assert open(q).read() == open(p).read()
        assert open(q + ".blocks").read() == open(p + ".blocks").read()


def test_stencil_operator_round_trip(ctx, tmp_path):
    h = pr.stencil_matrix(2, 6, 2, 10)
    p = str(tmp_path / "c1.mtx")
    _write_reference_format(h, p)
    A, sym = read_matrix(ctx, p)
    assert sym
    assert np.array_equal(A.download(h.row_sizes, h.col_sizes).vals, h.vals)


def test_vector_round_trip(ctx, rng, tmp_path):
    x = rng.standard_normal(37) * 10.0 ** rng.integers(-30, 30, 37)
    p = str(tmp_path / "x.vec")
    with open(p, "w") as f:
        f.write("".join(f"{v:.17g}\n" for v in x))
    v = read_vector(ctx, p)
    assert np.array_equal(v.download(), x)
    q = str(tmp_path / "y.vec")
    write_vector(v, q)
    assert open(q).read() == open(p).read()


def test_io_errors_carry_line(ctx, tmp_path):
    p = str(tmp_path / "bad.mtx")
    with open(p + ".blocks", "w") as f:
        f.write("2\n1\n")
    with open(p, "w") as f:
        f.write("%%block-matrix 3 3 2\n1 1 1.0\n")
    with pytest.raises(IoError) as e:
        read_matrix(ctx, p)  # header count does not match
    assert "count" in str(e.value)
    with open(p, "w") as f:
        f.write("%%block-matrix 3 3 1\n1 x 1.0\n")
    with pytest.raises(IoError) as e:
        read_matrix(ctx, p)
    assert e.value.line == 2
    with open(p, "w") as f:
        f.write("%%blockmatrix 3 3 1\n")
    with pytest.raises(IoError) as e:
        read_matrix(ctx, p)
    assert e.value.line == 1
    with open(p + ".blocks", "w") as f:
        f.write("2\n0\n")
    with pytest.raises(IoError) as e:
        read_matrix(ctx, p)
    assert e.value.line == 2
    with pytest.raises(IoError):
        read_matrix(ctx, str(tmp_path / "missing.mtx"))
