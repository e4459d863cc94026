"""HBM ceilings on this GPU for read-only, write-only and copy streams (torch kernels, CUDA events)."""
import json, torch
dev = torch.device("cuda", 0)
n = 1 << 30  # floats (4 GiB)
a = torch.ones(n, device=dev)
b = torch.empty(n, device=dev)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
r = {}
r["read_GBps"] = 4 * n / t(lambda: a.sum()) / 1e6
r["write_GBps"] = 4 * n / t(lambda: b.fill_(2.0)) / 1e6
r["copy_GBps"] = 8 * n / t(lambda: b.copy_(a)) / 1e6
print(json.dumps({k: round(v, 1) for k, v in r.items()}))
