import sys, time, torch
sys.path.insert(0, '.')
from paper_2509_06744_b200 import BlockSparseMatrix, Context, Hierarchy, Vector, default_params
from paper_2509_06744_b200 import problems as pr
ctx = Context(0)
for m in (21,):
    host = pr.stencil_matrix(2, 64, 2, m)
    A = BlockSparseMatrix(ctx, host)
    print('free before', torch.cuda.mem_get_info(), flush=True)
    t0 = time.time()
    try:
        h = Hierarchy.setup(A, [], default_params(t_max=1, coarse_dim_cap=1 << 30))
        print('ok', time.time() - t0, h.device_bytes, torch.cuda.mem_get_info(), flush=True)
    except Exception as e:
        print('ERR', e, torch.cuda.mem_get_info(), flush=True)
