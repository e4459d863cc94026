"""Time the loop kernel for several forced launch plans (device-resident inputs)."""
import os, sys, json
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mix = int(sys.argv[2]) if len(sys.argv) > 2 else 64
plans = sys.argv[3].split(";") if len(sys.argv) > 3 else [""]
cfg = CONFIGS[cfg_id]
mix = min(mix, cfg.mixtures)
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
y, P0, l0, v0 = make_torch(cfg, 1, mix, dev)
P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
lib.ffca_set_kernel_timing(1)
units = mix * cfg.N * cfg.F * cfg.iterations
for plan in plans:
    if plan:
        os.environ["FFCA_FORCE_PLAN"] = plan
    else:
        os.environ.pop("FFCA_FORCE_PLAN", None)
    ms = []
    for rep in range(4):
        rc = lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, code, mix, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(),
                                  P0.data_ptr(), l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None,
                                  cfg.iterations, 1, 0, P.data_ptr(), l.data_ptr(), v.data_ptr(), None, None, None)
        _lib.check(rc)
        ms.append(lib.ffca_last_kernel_ms())
    out = (ctypes_arr := None)
    import numpy as np
    o6 = np.zeros(6, np.int32)
    lib.ffca_plan_loop(0, code, mix, cfg.I, cfg.J, cfg.N, cfg.F, _lib.VF_AUTO, o6.ctypes.data_as(_lib._ip))
    best = min(ms[1:])
    print(json.dumps({"config": cfg_id, "mix": mix, "plan": plan or "auto", "auto_plan": o6.tolist(),
                      "kernel_ms": round(best, 3), "Gunits_per_s": round(units / best / 1e6, 2)}), flush=True)
