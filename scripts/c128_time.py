"""Kernel time of the complex128 loop at the config-3 shape (MIX mixtures) and at config 0."""
import os, sys, json
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch
cfg = CONFIGS[3]
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
lib.ffca_set_kernel_timing(1)
for U in (1, int(os.environ.get("MIX", "256"))):
    y, P0, l0, v0 = make_torch(cfg, 7, U, dev)
    y, P0, l0, v0 = y.to(torch.complex128), P0.to(torch.complex128), l0.double(), v0.double()
    P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
    ms = []
    for _ in range(4):
        _lib.check(lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, _lib.C128, U, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(),
                                        P0.data_ptr(), l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None,
                                        cfg.iterations, 1, 0, P.data_ptr(), l.data_ptr(), v.data_ptr(), None, None, None))
        ms.append(lib.ffca_last_kernel_ms())
    print(json.dumps({"mixtures": U, "kernel_ms": round(min(ms[1:]), 4)}))
    del y, P0, l0, v0, P, l, v
