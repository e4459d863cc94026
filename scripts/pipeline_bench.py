"""End-to-end separation (cli.separate_once scope, plus analysis/init/images/resynthesis) on an
8 s, 3-channel, 3-source mixture: device pipeline vs the oracle chain on the host (c128).

Reports per (algorithm, dtype): host-to-host wall time of the whole pipeline, the device time
of the estimator alone and the real-time factors (estimator / duration, the reference's RTF
definition), and the oracle-chain wall time on one host core for the same scene."""
import json, os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
import torch
from paper_1805_09498_b200 import pipeline
from oracle import pipeline_ref

rng = np.random.default_rng(0)
J, I, S = 3, 3, 8 * 16000
refs = rng.standard_normal((J, I, S))
mix = refs.sum(axis=0)
out = {"what": "separate_once, 8 s x 3 ch x 3 src, oracle init, 20 iterations, L=1024/512"}
for algo in ("fastfca", "fca"):
    for c64 in (False, True):
        cfg = pipeline.PipelineConfig(algorithm=algo, init="oracle", sources=J, complex64=c64)
        for _ in range(2):
            pipeline.separate_once(cfg, mix, refs)
        walls, ests = [], []
        for _ in range(5):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = pipeline.separate_once(cfg, mix, refs)
            walls.append(time.perf_counter() - t)
            ests.append(r.estimator_seconds)
        key = f"{algo}_{'c64' if c64 else 'c128'}"
        out[key] = {"pipeline_wall_ms": round(1e3 * float(np.median(walls)), 3),
                    "estimator_ms": round(1e3 * float(np.median(ests)), 4),
                    "rtf_estimator": float(np.median(ests)) / 8.0,
                    "rtf_pipeline": float(np.median(walls)) / 8.0,
                    "sdr_mean": float(np.mean(r.sdr_per_source))}
for algo in ("fastfca", "fca"):
    t = time.perf_counter()
    _, sdrs, _ = pipeline_ref.separate_once(mix, refs, algo, "oracle", sources=J, iterations=20)
    out[f"oracle_chain_{algo}_c128_wall_s_1core"] = round(time.perf_counter() - t, 3)
    out[f"oracle_chain_{algo}_sdr_mean"] = float(np.mean(sdrs))
print(json.dumps(out))
