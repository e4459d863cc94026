"""Kernel time of every BASELINE.json config on device-resident synthetic inputs (1 GPU)."""
import json, os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_1805_09498_b200 import _lib
from paper_1805_09498_b200.workloads import CONFIGS, make_torch

ids = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "0,1,2,3,4".split(","))]
dev = torch.device("cuda", 0)
lib = _lib.require_gpu()
lib.ffca_set_kernel_timing(1)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
for cid in ids:
    cfg = CONFIGS[cid]
    U = cfg.mixtures
    y, P0, l0, v0 = make_torch(cfg, 7, U, dev)
    code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
    c = 8 if cfg.dtype == "c64" else 16
    r = c // 2
    units = U * cfg.N * cfg.F * cfg.iterations
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if cfg.algorithm == "fca":
        S0 = torch.eye(cfg.I, dtype=y.dtype, device=dev).expand(U, cfg.J, cfg.F, cfg.I, cfg.I).contiguous()
        S, v = torch.empty_like(S0), torch.empty_like(v0)
        def step():
            _lib.check(lib.ffca_fca_run(0, None, _lib.MEM_DEVICE, code, U, cfg.I, cfg.J, cfg.N, cfg.F, y.data_ptr(),
                                        S0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None, cfg.iterations, 0,
                                        S.data_ptr(), v.data_ptr(), None, None, None, None))
        algo = cfg.I * c + 2 * cfg.J * r
    else:
        P, l, v = torch.empty_like(P0), torch.empty_like(l0), torch.empty_like(v0)
        def step():
            _lib.check(lib.ffca_fastfca_run(0, None, _lib.MEM_DEVICE, code, U, cfg.I, cfg.J, cfg.N, cfg.F,
                                            y.data_ptr(), P0.data_ptr(), l0.data_ptr(), v0.data_ptr(),
                                            _lib.VF_AUTO, 0.0, None, cfg.iterations, 1, 0, P.data_ptr(),
                                            l.data_ptr(), v.data_ptr(), None, None, None))
        algo = 2 * cfg.I * c + 3 * cfg.J * r
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    ev0.record()
    reps = 3
    for _ in range(reps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    o6 = __import__("numpy").zeros(6, "int32")
    lib.ffca_plan_loop(0, code, U, cfg.I, cfg.J, cfg.N, cfg.F, _lib.VF_AUTO, o6.ctypes.data_as(_lib._ip))
    print(json.dumps({"config": cid, "name": cfg.name, "ms": round(ms, 3), "units_per_s": units / ms * 1e3,
                      "streaming_model_GBps": round(algo * units / ms / 1e6, 1),
                      "frac_of_measured_hbm": round(algo * units / ms / 1e6 / peak, 3),
                      "plan(G,C,NL,threads,res,smem)": o6.tolist() if cfg.algorithm != "fca" else None}), flush=True)
    del y, P0, l0, v0
    torch.cuda.empty_cache()
