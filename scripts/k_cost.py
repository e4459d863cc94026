"""Cost of one extra fixed-point solve round per iteration: config-3 kernel time at K=1,2,3."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cfg = CONFIGS[3]
U = 256
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
y, P0, l0, v0 = make_torch(cfg, 7, U, dev)
P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
lib.ffca_set_kernel_timing(1)
for K in (1, 2, 3):
    ms = []
    for _ in range(3):
        _lib.check(lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, _lib.C64, U, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(),
                                        P0.data_ptr(), l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None,
                                        cfg.iterations, K, 0, P.data_ptr(), l.data_ptr(), v.data_ptr(), None, None, None))
        ms.append(lib.ffca_last_kernel_ms())
    print("K", K, "kernel ms", round(min(ms[1:]), 3))
