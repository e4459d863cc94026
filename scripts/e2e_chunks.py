"""e2e (host numpy, pinned) time of the config-3 batch through run_fastfca_batch for several pipeline chunk counts."""
import os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200.fastfca import run_fastfca_batch
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cfg = CONFIGS[3]
dev = torch.device("cuda", 0)
y, P0, l0, v0 = make_torch(cfg, 7, 256, dev)
pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t).numpy()
Y, P, L, V = pin(y), pin(P0), pin(l0), pin(v0)
outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).numpy() for t in (P0, l0, v0)]
for ch in sys.argv[1:]:
    os.environ["FFCA_PIPELINE_CHUNKS"] = ch
    run_fastfca_batch(Y, P, L, V, iterations=20, out=outs)
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        run_fastfca_batch(Y, P, L, V, iterations=20, out=outs)
        ts.append(time.perf_counter() - t)
    print("chunks", ch, "ms", round(1e3 * min(ts), 2), flush=True)
