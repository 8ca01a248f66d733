import torch, time
dev=torch.device('cuda')
for mb in (4, 37.3, 112):
    n=int(mb*1e6)
    h=torch.empty(n,dtype=torch.uint8).pin_memory(); d=torch.empty(n,dtype=torch.uint8,device=dev)
    for _ in range(3): d.copy_(h,non_blocking=True)
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): d.copy_(h,non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms=s.elapsed_time(e)/20
    print(f"H2D {mb} MB: {n/ms/1e6:.1f} GB/s")
    s.record()
    for _ in range(20): h.copy_(d,non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms=s.elapsed_time(e)/20
    print(f"D2H {mb} MB: {n/ms/1e6:.1f} GB/s")
# concurrent H2D + D2H
n=int(37.3e6); h=torch.empty(n,dtype=torch.uint8).pin_memory(); d=torch.empty(n,dtype=torch.uint8,device=dev)
h2=torch.empty(n//6,dtype=torch.uint8).pin_memory(); d2=torch.empty(n//6,dtype=torch.uint8,device=dev)
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(20):
    with torch.cuda.stream(s1): d.copy_(h,non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2,non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/20
print(f"concurrent 37.3MB H2D + 6.2MB D2H: {dt*1e3:.3f} ms/iter -> H2D {n/dt/1e9:.1f} GB/s")
