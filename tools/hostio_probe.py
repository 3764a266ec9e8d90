"""Launch counts and timing of the host-buffer cycle (bmg_vcycle_host) against the
device-resident one on a BASELINE config: python tools/hostio_probe.py C4"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2509_06744_b200 import Context, Vector
from paper_2509_06744_b200 import problems as pr
cfg = pr.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ctx = Context(0)
stream = torch.cuda.current_stream(); ctx.set_stream(stream.cuda_stream)
H, b = bench.whole_hierarchy(ctx, cfg)
k = cfg.k
hb = torch.from_numpy(b).pin_memory(); hx = torch.zeros(b.size, dtype=torch.float64).pin_memory()
bv, xv = Vector(ctx, b), Vector(ctx, b.size)
def timed(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_count
    e0.record(stream)
    for _ in range(n): fn()
    e1.record(stream); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, (ctx.launch_count - l0) / n
print("device V(%d,%d): %.3f ms, %.0f launches" % ((k, k) + timed(lambda: H.v_cycle(k, k, bv, xv))))
print("host   V(%d,%d): %.3f ms, %.0f launches" % ((k, k) + timed(lambda: H.v_cycle_host_ptr(k, k, hb.data_ptr(), hx.data_ptr()))))
print("device V(%d,0): %.3f ms, %.0f launches" % ((2 * k,) + timed(lambda: H.v_cycle(2 * k, 0, bv, xv))))
print("host   V(%d,0): %.3f ms, %.0f launches" % ((2 * k,) + timed(lambda: H.v_cycle_host_ptr(2 * k, 0, hb.data_ptr(), hx.data_ptr()))))
