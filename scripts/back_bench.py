"""Back-transform x_j = P^-H mu_tilde_j (wiener.mmse_images_fastfca's device pass, fastfca.py:258-273 /
wiener.py:38-43) from device-resident statistics, images layout: ms and algorithmic GB/s."""
import json, os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cfg = CONFIGS[int(os.environ.get("CFG", "3"))]
U = int(os.environ.get("MIX", 256 if cfg.mixtures > 1 else 1))
I, J, N, F = cfg.I, cfg.J, cfg.N, cfg.F
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
y, P, lam, v = make_torch(cfg, 5, U, dev)
mu = torch.randn((U, J, N, F, I), dtype=torch.complex64, device=dev)
img = torch.empty((U, J, I, N, F), dtype=torch.complex64, device=dev)


def back():
    _lib.check(lib.ffca_back_transform(0, None, _lib.MEM_DEVICE, _lib.C64, U, I, J, N, F, P.data_ptr(), mu.data_ptr(),
                                       img.data_ptr(), 1, None), "back")


back()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    back()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
nbytes = U * N * F * J * I * 8 * 2
print(json.dumps({"what": f"back-transform {U} x (I={I}, J={J}, F={F}, N={N}) c64", "ms": round(ms, 3),
                  "GBps": round(nbytes / ms / 1e6, 1)}))
