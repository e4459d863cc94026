"""Pinned host->device copy bandwidth with 1, 2 and 4 concurrent streams (does a second copy engine help?)."""
import torch
n = 2_973_791_232 // 4
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4, 1):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[k * part:(k + 1) * part].copy_(h[k * part:(k + 1) * part], non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if False else torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{ns} stream(s): H2D {4 * part * ns / best / 1e6:.1f} GB/s ({best:.1f} ms)")
