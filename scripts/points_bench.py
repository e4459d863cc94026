"""Output-side streaming kernels at config-3 scale (256 mixtures, I=J=3, F=513, N=626), device-resident:
Wiener images (wiener.mmse_images_fastfca, fused refresh + back-solve) and the statistics refresh
(fastfca._stats_refresh).  Reports ms and algorithmic GB/s vs the measured HBM peak."""
import json, os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

code_name = sys.argv[1] if len(sys.argv) > 1 else "c64"
cfg = CONFIGS[int(os.environ.get("CFG", "3"))]  # CFG=4: the I = 8, J = 6 shape (untiled point_kernel path)
U = (256 if code_name == "c64" else 64) if cfg.mixtures > 1 else 1
U, I, J, N, F = int(os.environ.get("MIX", U)), cfg.I, cfg.J, cfg.N, cfg.F
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
y, P, lam, v = make_torch(cfg, 5, U, dev)
code = _lib.C64
if code_name == "c128":
    y, P, lam, v = y.to(torch.complex128), P.to(torch.complex128), lam.double(), v.double()
    code = _lib.C128
cs, rs = y.element_size(), v.element_size()
img = torch.empty((U, J, I, N, F), dtype=y.dtype, device=dev)
mu = torch.empty((U, J, N, F, I), dtype=y.dtype, device=dev)
phi = torch.empty((U, J, N, F, I), dtype=v.dtype, device=dev)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def images():
    _lib.check(lib.ffca_fastfca_images(0, None, _lib.MEM_DEVICE, code, U, I, J, N, F, y.data_ptr(), P.data_ptr(),
                                       lam.data_ptr(), v.data_ptr(), img.data_ptr(), None), "images")


def stats():
    _lib.check(lib.ffca_fastfca_stats(0, None, _lib.MEM_DEVICE, code, U, I, J, N, F, y.data_ptr(), P.data_ptr(),
                                      lam.data_ptr(), v.data_ptr(), mu.data_ptr(), phi.data_ptr()), "stats")


pts = U * N * F
b_img = pts * (I * cs + J * rs + J * I * cs)
b_st = pts * (I * cs + J * rs + J * I * (cs + rs))
ti, ts = timeit(images), timeit(stats)
print(json.dumps({"what": f"{U} mixtures x (I={I}, J={J}, F={F}, N={N}) {code_name}, device-resident",
                  "images_ms": round(ti, 3), "images_GBps": round(b_img / ti / 1e6, 1),
                  "stats_ms": round(ts, 3), "stats_GBps": round(b_st / ts / 1e6, 1), "hbm_peak_GBps": 6549.1}))
