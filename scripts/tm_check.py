"""Tensor-memory plan vs the shared-memory plan on the config-3 shape: results and kernel time."""
import os, sys, json
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cfg = CONFIGS[int(os.environ.get('CFG', '3'))]
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
lib.ffca_set_kernel_timing(1)
code = _lib.C64


def run(y, P0, l0, v0, mix, env, iters=cfg.iterations, N=cfg.N, F=cfg.F):
    for k in ("FFCA_NO_TMEM", "FFCA_FORCE_PLAN"):
        os.environ.pop(k, None)
    os.environ.update(env)
    P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
    ms = []
    for rep in range(3):
        _lib.check(lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, code, mix, cfg.I, cfg.J, N, F, y.data_ptr(),
                                        P0.data_ptr(), l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None,
                                        iters, 1, 0, P.data_ptr(), l.data_ptr(), v.data_ptr(), None, None, None))
        ms.append(lib.ffca_last_kernel_ms())
    torch.cuda.synchronize()
    return P, l, v, min(ms)


def rel(a, b):
    return float((a - b).abs().max() / b.abs().max())


mix = int(sys.argv[1]) if len(sys.argv) > 1 else 8
y, P0, l0, v0 = make_torch(cfg, 1, mix, dev)
ref = run(y, P0, l0, v0, mix, {"FFCA_NO_TMEM": "1"})
tm = run(y, P0, l0, v0, mix, {})
g4 = run(y, P0, l0, v0, mix, {"FFCA_FORCE_PLAN": "4,1,1,128"}) if cfg.I == 3 else ref
print(json.dumps({"mix": mix, "ms_default": ref[3], "ms_tm": tm[3], "ms_g4_128": g4[3],
                  "tm_vs_default": [rel(tm[i], ref[i]) for i in range(3)],
                  "tm_vs_g4": [rel(tm[i], g4[i]) for i in range(3)],
                  "finite": bool(torch.isfinite(tm[2]).all())}))
