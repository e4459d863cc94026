"""Throughput of the device STFT vs the numpy oracle (samples/s), 8 s x 3 channels x 64 signals."""
import json, os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch
from paper_1805_09498_b200 import _lib
from oracle import stft_ref

lib = _lib.require_gpu()
rng = np.random.default_rng(0)
I, S, L, sh = 3 * 64, 8 * 16000, 1024, 512
audio = rng.standard_normal((I, S))
N = (S - L) // sh + 1
dev = torch.device("cuda", 0)
a_d = torch.from_numpy(audio).to(dev)
o_d = torch.empty((I, N, L // 2), dtype=torch.complex128, device=dev)
r_d = torch.empty((I, (N - 1) * sh + L), dtype=torch.float64, device=dev)
for _ in range(3):
    _lib.check(lib.ffca_stft_analyze(0, None, _lib.MEM_DEVICE, _lib.C128, I, S, L, sh, a_d.data_ptr(), o_d.data_ptr()))
    _lib.check(lib.ffca_stft_synthesize(0, None, _lib.MEM_DEVICE, _lib.C128, I, N, L, sh, o_d.data_ptr(), r_d.data_ptr()))
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record()
for _ in range(10):
    _lib.check(lib.ffca_stft_analyze(0, None, _lib.MEM_DEVICE, _lib.C128, I, S, L, sh, a_d.data_ptr(), o_d.data_ptr()))
e1.record()
for _ in range(10):
    _lib.check(lib.ffca_stft_synthesize(0, None, _lib.MEM_DEVICE, _lib.C128, I, N, L, sh, o_d.data_ptr(), r_d.data_ptr()))
e2.record()
torch.cuda.synchronize()
ta, ts = e0.elapsed_time(e1) / 10, e1.elapsed_time(e2) / 10
t = time.perf_counter(); obs = stft_ref.analyze(audio[:24]); ca = (time.perf_counter() - t) * I / 24 * 1e3
t = time.perf_counter(); stft_ref.synthesize(obs); cs = (time.perf_counter() - t) * I / 24 * 1e3
bytes_a = I * S * 8 + I * N * (L // 2) * 16
print(json.dumps({"what": "STFT analyze/synthesize, 192 channels x 8 s @16 kHz, c128, device-resident",
                  "analyze_ms": round(ta, 3), "synthesize_ms": round(ts, 3),
                  "analyze_Msamples_per_s": round(I * S / ta / 1e3, 1),
                  "analyze_io_GBps": round(bytes_a / ta / 1e6, 1),
                  "numpy_oracle_analyze_ms_extrapolated": round(ca, 1),
                  "numpy_oracle_synthesize_ms_extrapolated": round(cs, 1)}))
