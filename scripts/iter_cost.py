"""Loop-kernel time vs iteration count for one config (fixed cost = gather + write-back)."""
import dataclasses, json, os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
if os.environ.get("FFCA_LIB"):  # an experiment build (e.g. build/libffca_exp1.so)
    _lib.LIB_PATH = os.environ["FFCA_LIB"]
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = CONFIGS[cid]
U = cfg.mixtures
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
lib.ffca_set_kernel_timing(1)
y, P0, l0, v0 = make_torch(cfg, 7, U, dev)
code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
for it in [0, 1, 2, 5, cfg.iterations]:
    best = 1e9
    for rep in range(3):
        _lib.check(lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, code, U, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(),
                                        P0.data_ptr(), l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None,
                                        it, 1, 0, P.data_ptr(), l.data_ptr(), v.data_ptr(), None, None, None))
        best = min(best, lib.ffca_last_kernel_ms())
    print(json.dumps({"config": cid, "iterations": it, "kernel_ms": round(best, 3)}))
