"""CPU-side checks of the product library: it loads, exports every symbol the
public header declares, refuses to compute without a GPU (no CPU fallback), and
its host-only pieces (synthetic generator, tridiagonal eigensolver) behave."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2509_06744_b200 import native as N
from paper_2509_06744_b200 import problems as pr
from paper_2509_06744_b200.api import tridiag_eigs


def test_library_exports_every_header_symbol():
    lib = N.lib()
    syms = N.header_symbols()
    assert len(syms) >= 45
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes table covers the whole header (the Python mirror binds everything)
    assert set(syms) <= set(N._SIGS), set(syms) - set(N._SIGS)


def test_generator_is_a_separate_library():
    # the synthetic inputs come from bmggen/libbmggen.so (include/bmg_gen.h), so the
    # reference arm of bench.py maps neither the product nor its kernels
    import re

    import bmggen

    hdr = open(os.path.join(os.path.dirname(N.HEADER_PATH), "bmg_gen.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    gen_syms = sorted(set(re.findall(r"\b(bmg_gen_[a-z_]+)\s*\(", hdr)))
    assert len(gen_syms) == 4
    g = bmggen.lib()
    assert all(hasattr(g, s) for s in gen_syms)
    assert set(gen_syms) == set(bmggen._SIGS)
    nm = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "bmg_gen_" not in nm, "libbmgcuda.so must not carry the generator"


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    archs = {line.split(".")[-2] for line in out.splitlines() if ".sm_" in line}
    assert archs and all(a.startswith("sm_100a") for a in archs), out


def test_no_cpu_fallback_without_gpu():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    from paper_2509_06744_b200 import Context, CudaError

    with pytest.raises(CudaError):
        Context(0)


def test_status_codes_map_to_reference_exceptions():
    assert issubclass(N.InvalidArgument, ValueError)
    assert issubclass(N.OutOfRange, IndexError)
    e = N.NotPositiveDefinite("x", 3)
    assert e.pivot == 3


def test_generator_stencil_counts_and_values():
    # 13-point 2-D biharmonic, 25-point 3-D biharmonic and 2-D triharmonic
    for dim, n, p, want in [(2, 8, 2, 13), (3, 6, 2, 25), (2, 9, 3, 25)]:
        A = pr.stencil_matrix(dim, n, p, 2)
        assert np.diff(A.row_ptr).max() == want
    # unscaled L_D^2 centre: 20 interior, 19 edge, 18 corner (reg = 0 isolates S (x) C)
    A = pr.stencil_matrix(2, 8, 2, 1, reg=0.0)
    d = A.to_dense()
    c = d[0, 0] / 18.0
    assert d[9, 9] / c == pytest.approx(20.0) and d[1, 1] / c == pytest.approx(19.0)


def test_generator_symmetric_spd_and_deterministic():
    A = pr.stencil_matrix(2, 6, 2, 4)
    D = A.to_dense()
    assert np.array_equal(D, D.T)
    assert np.linalg.eigvalsh(D).min() > 0
    B = pr.stencil_matrix(2, 6, 2, 4)
    assert np.array_equal(A.vals, B.vals)
    assert not np.array_equal(pr.stencil_matrix(2, 6, 2, 4, seed=1).vals, A.vals)


def test_generator_prolongation_structure():
    for dim, nf, per in [(2, 8, 9), (3, 8, 27)]:
        P = pr.prolongation(dim, nf, 3)
        cnt = np.diff(P.row_ptr)
        assert cnt.max() == per and cnt.min() >= 2 ** dim
        m = 3
        for i in range(P.nbr):
            blk = P.vals[P.row_ptr[i] * m * m:P.row_ptr[i + 1] * m * m]
            assert np.linalg.norm(blk) == pytest.approx(np.sqrt(m), rel=1e-12)
        # parent of fine (x, y) is (x >> 1, y >> 1)
        nc = nf // 2
        i = 5 + nf * 3 if dim == 2 else 1 + nf * (2 + nf * 3)
        x, y, z = i % nf, (i // nf) % nf, i // (nf * nf)
        parent = (x >> 1) + nc * ((y >> 1) + (nc * (z >> 1) if dim == 3 else 0))
        assert parent in P.col_idx[P.row_ptr[i]:P.row_ptr[i + 1]]


def test_normal_vector_moments():
    v = pr.normal_vector(200000, 0, 0)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1) < 0.01


def test_product_tridiagonal_eigensolver_vs_oracle(rng):
    for n in (1, 2, 3, 17, 100):
        d, e = rng.standard_normal(n), rng.standard_normal(max(n - 1, 0))
        got = tridiag_eigs(d, e)
        want = O.tridiag_eigs(d, e)
        assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_configs_match_baseline_json():
    import json

    with open(os.path.join(os.path.dirname(os.path.dirname(N.LIB_PATH)), "BASELINE.json")) as f:
        js = json.load(f)
    assert len(js["configs"]) == 5
    c = pr.CONFIGS
    assert (c["C1"].n, c["C1"].m, c["C1"].levels) == (64, 10, 1)
    assert (c["C2"].n, c["C2"].m, c["C2"].levels, c["C2"].k) == (256, 10, 4, 3)
    assert (c["C3"].n, c["C3"].m, c["C3"].power, c["C3"].levels, c["C3"].k) == (1024, 21, 3, 5, 4)
    assert (c["C4"].dim, c["C4"].n, c["C4"].m, c["C4"].levels) == (3, 64, 20, 4)
    assert (c["C5"].n, c["C5"].m, c["C5"].levels) == (2048, 15, 6)
