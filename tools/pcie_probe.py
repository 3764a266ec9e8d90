import torch, time
n=42*1024*1024//8
h=torch.empty(n,dtype=torch.float64).pin_memory(); d=torch.empty(n,dtype=torch.float64,device='cuda')
for name,fn in (("h2d",lambda: d.copy_(h,non_blocking=True)),("d2h",lambda: h.copy_(d,non_blocking=True))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/10
    print(name, "42 MB in %.3f ms = %.1f GB/s"%(ms, n*8/ms/1e6))
