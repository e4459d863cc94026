"""Kernel time for forced plans on a (possibly F-reduced) config: plan_sweep_cfg.py CFG F 'G,C,res,thr;...'"""
import dataclasses, json, os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cid, F = int(sys.argv[1]), int(sys.argv[2])
plans = sys.argv[3].split(";")
cfg = dataclasses.replace(CONFIGS[cid], F=F) if F else CONFIGS[cid]
U = int(os.environ.get("MIX", str(cfg.mixtures if cid != 3 else 32)))
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
y, P0, l0, v0 = make_torch(cfg, 7, U, dev)
code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
lib.ffca_set_kernel_timing(1)
units = U * cfg.N * cfg.F * cfg.iterations
for plan in plans:
    if plan:
        os.environ["FFCA_FORCE_PLAN"] = plan
    else:
        os.environ.pop("FFCA_FORCE_PLAN", None)
    ms = []
    for _ in range(3):
        _lib.check(lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, code, U, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(),
                                        P0.data_ptr(), l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None,
                                        cfg.iterations, 1, 0, P.data_ptr(), l.data_ptr(), v.data_ptr(), None, None, None))
        ms.append(lib.ffca_last_kernel_ms())
    o6 = np.zeros(6, np.int32)
    lib.ffca_plan_loop(0, code, U, cfg.I, cfg.J, cfg.N, cfg.F, _lib.VF_AUTO, o6.ctypes.data_as(_lib._ip))
    print(json.dumps({"cfg": cid, "F": cfg.F, "plan": plan or "auto", "resolved": o6.tolist(), "ms": round(min(ms[1:]), 3),
                      "Gunits_per_s": round(units / min(ms[1:]) / 1e6, 3)}), flush=True)
