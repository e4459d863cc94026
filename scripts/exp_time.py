"""Config kernel time with whatever library FFCA_LIB points at; ignores status errors (timing experiments)."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = CONFIGS[cid]
if os.environ.get("DTYPE"):  # e.g. DTYPE=c128: the same shape in the other precision
    import dataclasses
    cfg = dataclasses.replace(cfg, dtype=os.environ["DTYPE"])
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
U = cfg.mixtures
y, P0, l0, v0 = make_torch(cfg, 7, U, dev)
code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
def call():
    return lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, code, U, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(), P0.data_ptr(),
                                l0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None, cfg.iterations, 1, 0, P.data_ptr(),
                                l.data_ptr(), v.data_ptr(), None, None, None)
for _ in range(2):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    rc = call()
e1.record()
torch.cuda.synchronize()
print(f"{os.path.basename(os.environ.get('FFCA_LIB', 'default'))} config{cid}: {e0.elapsed_time(e1) / 5:.3f} ms rc={rc}")
