"""Raw pinned host<->device copy bandwidth for the bench step's byte counts (the e2e copy floor)."""
import torch, time
n = 2_973_791_232 // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
o = torch.empty(1_001_244_672 // 4, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(o.numel(), dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    torch.cuda.synchronize(); t = time.perf_counter()
    o.copy_(d2, non_blocking=True); torch.cuda.synchronize()
    dt2 = time.perf_counter() - t
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): o.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt3 = time.perf_counter() - t
    print(f"H2D {h.nbytes/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)  D2H {o.nbytes/dt2/1e9:.1f} GB/s ({dt2*1e3:.1f} ms)  both concurrently {dt3*1e3:.1f} ms")
