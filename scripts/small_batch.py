"""Kernel time for U mixtures of a config's shape (plan-heuristic checks on small problems)."""
import json, os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import dataclasses
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cid, U = int(sys.argv[1]), int(sys.argv[2])
cfg = CONFIGS[cid]
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
lib.ffca_set_kernel_timing(1)
y, P0, l0, v0 = make_torch(cfg, 7, U, dev)
code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
best = 1e9
for _ in range(5):
    _lib.check(lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, code, U, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(),
                                    P0.data_ptr(), l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None,
                                    cfg.iterations, 1, 0, P.data_ptr(), l.data_ptr(), v.data_ptr(), None, None, None))
    best = min(best, lib.ffca_last_kernel_ms())
print(json.dumps({"config": cid, "mixtures": U, "plan": os.environ.get("FFCA_FORCE_PLAN", "default"), "ms": round(best, 4)}))
