"""Config-1 FCA kernel time vs threads per CTA (FFCA_FCA_THREADS tuning hook)."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cfg = CONFIGS[1]
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
y, P0, l0, v0 = make_torch(cfg, 3, 1, dev)
I, J, N, F = cfg.I, cfg.J, cfg.N, cfg.F
S0 = torch.eye(I, dtype=y.dtype, device=dev).expand(1, J, F, I, I).contiguous()
S, v = torch.empty_like(S0), torch.empty_like(v0)
for thr in sys.argv[1:]:
    if thr == "auto":
        os.environ.pop("FFCA_FCA_THREADS", None)
    else:
        os.environ["FFCA_FCA_THREADS"] = thr
    ms = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.ffca_fca_run(0, None, _lib.MEM_DEVICE, _lib.C128, 1, I, J, N, F, y.data_ptr(), S0.data_ptr(),
                                    v0.data_ptr(), _lib.VF_AUTO, 0.0, None, cfg.iterations, 0, S.data_ptr(),
                                    v.data_ptr(), None, None, None, None))
        e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1))
    print("threads", thr, "ms", round(min(ms[1:]), 3), flush=True)
