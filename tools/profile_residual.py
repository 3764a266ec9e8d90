"""One fine-level residual pass r = b - A x per BASELINE block size, for ncu:
  ncu --set full -k regex:bsr_stream_kernel --launch-skip 2 --launch-count 1 \\
      python tools/profile_residual.py --m 20
runs 3 identical launches (2 warm, the third is captured).  The operators are
the BASELINE fine levels (full C4 and C2; C5 and C3 shapes at a quarter of their
rows, which already exceed L2 by 190x).  Prints the algorithmic bytes of one
launch (nnzb * (8 m^2 + 4) + 24 N), the number bench.py's roofline uses."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Vector, residual  # noqa: E402
from paper_2509_06744_b200 import problems as pr  # noqa: E402

CASES = {10: ("C2 fine (256^2, 13-pt)", 2, 256, 2), 15: ("C5 fine shape (1024^2, 13-pt)", 2, 1024, 2),
         20: ("C4 fine (64^3, 3-D 25-pt)", 3, 64, 2), 21: ("C3 fine shape (512^2, 25-pt)", 2, 512, 3)}

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=20)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
name, dim, n, p = CASES[a.m]
ctx = Context(0)
A = pr.stencil_matrix(dim, n, p, a.m)
dA = BlockSparseMatrix(ctx, A)
x = Vector(ctx, pr.normal_vector(A.dim_r, 0, 1))
b = Vector(ctx, pr.normal_vector(A.dim_r, 0, 2))
r = Vector(ctx, A.dim_r)
for _ in range(a.reps):
    residual(dA, b, x, r)
ctx.sync()
print(json.dumps({"case": name, "m": a.m, "nnzb": int(A.nnzb), "N": int(A.dim_r),
                  "algorithmic_bytes": int(dA.info()["pass_bytes"] + 24 * A.dim_r)}), flush=True)
