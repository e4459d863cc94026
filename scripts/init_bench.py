"""Throughput of the device initialisers (oracle / diffuse covariances) at config-3 scale
(256 mixtures, I=J=3, F=513, N=626, c64), device-resident, vs the numpy oracle."""
import json, os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch
from paper_1805_09498_b200 import _lib
from oracle import scene_ref

lib = _lib.require_gpu()
U, I, J, N, F = 256, 3, 3, 626, 513
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
refs = torch.randn((U, J, I, N, F), dtype=torch.complex64, device=dev, generator=g)
y = refs.sum(dim=1).contiguous()
fl = torch.empty((U, F), dtype=torch.float64, device=dev)
W = torch.from_numpy(scene_ref.perturbations(I, J, 7).astype(np.complex64)).to(dev)
S = torch.empty((U, J, F, I, I), dtype=torch.complex64, device=dev)
v = torch.empty((U, J, N, F), dtype=torch.float32, device=dev)


def floor():
    _lib.check(lib.ffca_power_floor(0, None, _lib.MEM_DEVICE, _lib.C64, U, I, N, F, y.data_ptr(), fl.data_ptr()))


def run(mode):
    x = refs if mode == 0 else y
    _lib.check(lib.ffca_init_covariances(0, None, _lib.MEM_DEVICE, _lib.C64, mode, U, I, J, N, F, x.data_ptr(),
                                         fl.data_ptr(), W.data_ptr(), S.data_ptr(), v.data_ptr()))


floor()
res = {}
for mode, name in ((0, "oracle"), (1, "diffuse")):
    for _ in range(3):
        run(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run(mode)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    xb = (U * J if mode == 0 else U) * I * N * F * 8
    vb = U * J * N * F * 4
    res[name] = {"ms": round(ms, 3), "GBps": round((xb + vb) / ms / 1e6, 1),
                 "mixtures_per_s": round(U / ms * 1e3, 1)}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    floor()
e1.record()
torch.cuda.synchronize()
res["power_floor_ms"] = round(e0.elapsed_time(e1) / 10, 3)
# numpy oracle on 4 mixtures (c128), extrapolated to U
r4 = refs[:4].cpu().numpy().astype(np.complex128)
t = time.perf_counter()
for u in range(4):
    scene_ref.oracle_covariances(r4[u], r4[u].sum(axis=0))
res["numpy_oracle_ms_extrapolated"] = round((time.perf_counter() - t) / 4 * U * 1e3, 1)
t = time.perf_counter()
for u in range(4):
    scene_ref.diffuse_covariances(r4[u].sum(axis=0), J, 7)
res["numpy_diffuse_ms_extrapolated"] = round((time.perf_counter() - t) / 4 * U * 1e3, 1)
res["what"] = "initialisers, 256 mixtures x (I=J=3, F=513, N=626) c64, device-resident; GBps = input + v_hat bytes"
res["hbm_peak_GBps"] = 6549.1
print(json.dumps(res))
