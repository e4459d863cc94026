"""Per-phase cycle breakdown of the config-3 loop kernel (development probe build:
make EXTRA=-DFFCA_PHASE_PROBE BUILD=../../build/probe OUT=../../build/libffca_probe.so)."""
import ctypes, os, sys
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1805_09498_b200 import _lib
_lib.LIB_PATH = os.environ.get("FFCA_PROBE_LIB", os.path.join(ROOT, "build", "libffca_probe.so"))
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
U = 256 if cfg.mixtures > 1 else 1
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
lib.ffca_debug_phase.argtypes = [ctypes.c_void_p]
y, P0, l0, v0 = make_torch(cfg, 7, U, dev)
P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
out = np.zeros(16, np.uint64)
for rep in range(2):
    lib.ffca_debug_phase(out.ctypes.data)
    rc = (lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, code, U, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(),
                                    P0.data_ptr(), l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None,
                                    cfg.iterations, 1, 0, P.data_ptr(), l.data_ptr(), v.data_ptr(), None, None, None))
    if rc != 0:  # timing experiments (e.g. -DFFCA_SKIP_BLOOP) may produce singular results
        print("note: call returned", rc, _lib.last_error())
    torch.cuda.synchronize()
lib.ffca_debug_phase(out.ctypes.data)
names = ["A points", "A reduce", "lambda'+bar", "B points", "B reduce+bar", "B_i factor", "adj(P), det (I<=4)", "solve+bar"]
for t in range(2):
    tot = out[8 * t: 8 * t + 8].astype(float)
    print(f"thread {t}: total {tot.sum() / cfg.iterations:.0f} cycles/iteration")
    for k, nm in enumerate(names):
        print(f"   {nm:20s} {tot[k] / cfg.iterations:8.0f}  {100 * tot[k] / max(tot.sum(), 1):5.1f}%")
