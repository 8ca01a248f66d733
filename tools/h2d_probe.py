"""PCIe probe: H2D / D2H bandwidth of pinned copies by size, and one c1
frame (3 cameras x RGB + mm + validity, 37.3 MB) as 9 copies vs one packed
copy. Used to size the e2e path (bench.py e2e, engine.FrameUploader)."""
import torch

dev = torch.device("cuda")


def rate(fn, nbytes, reps=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return nbytes / (s.elapsed_time(e) / reps) / 1e6


for mb in (2, 4, 8, 37.3, 112):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    print(f"H2D {mb:6} MB: {rate(lambda: d.copy_(h, non_blocking=True), n):6.1f} GB/s   "
          f"D2H: {rate(lambda: h.copy_(d, non_blocking=True), n):6.1f} GB/s")
N = 1920 * 1080
sizes = [3 * N, 2 * N, N] * 3
hs = [torch.empty(s, dtype=torch.uint8).pin_memory() for s in sizes]
ds = [torch.empty(s, dtype=torch.uint8, device=dev) for s in sizes]
tot = sum(sizes)


def nine():
    for d, h in zip(ds, hs):
        d.copy_(h, non_blocking=True)


hp = torch.empty(tot, dtype=torch.uint8).pin_memory()
dp = torch.empty(tot, dtype=torch.uint8, device=dev)
print(f"c1 frame as 9 copies: {rate(nine, tot):6.1f} GB/s; "
      f"packed: {rate(lambda: dp.copy_(hp, non_blocking=True), tot):6.1f} GB/s")
