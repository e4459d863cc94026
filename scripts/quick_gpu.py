"""Quick GPU sanity: fused loop vs oracle on golden cases + config-0 timing."""
import sys, os, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
from paper_1805_09498_b200 import fastfca as F, ObservationTensor
from paper_1805_09498_b200 import workloads as W
from oracle import fastfca_ref as ffr

def rel(a, b):
    return float(np.abs(np.asarray(a) - b).max() / max(np.abs(b).max(), 1e-300))

g = dict(np.load("tests/golden/golden.npz"))
for key in ["g33", "g44", "g86", "g22", "g12", "g23"]:
    y, P0, l0, v0, it = g[key+"/y"], g[key+"/P0"], g[key+"/lam0"], g[key+"/v0"], int(g[key+"/iters"])
    for c64 in (False, True):
        yy = y.astype(np.complex64) if c64 else y
        PP = P0.astype(np.complex64) if c64 else P0
        run = F.run_fastfca(ObservationTensor(yy), F.FastFcaParams(PP, l0, v0), iterations=it, record_likelihood=True)
        ll = np.array([run.loglik_init] + run.loglik_after_em + run.loglik_after_p)
        print(key, "c64" if c64 else "c128", "P %.2e lam %.2e v %.2e ll %.2e" % (
            rel(run.params.P, g[key+"/P"]), rel(run.params.Lam, g[key+"/lam"]), rel(run.params.v, g[key+"/v"]),
            np.abs(ll - g[key+"/ll"]).max() / np.abs(g[key+"/ll"]).max()))

for cfg_id in (0,):
    cfg = W.CONFIGS[cfg_id]
    y, P, l, v = W.make(cfg)
    obs = ObservationTensor(y[0])
    init = F.FastFcaParams(P[0], l[0], v[0])
    for rep in range(3):
        t = time.perf_counter()
        run = F.run_fastfca(obs, init, iterations=cfg.iterations)
        dt = time.perf_counter() - t
        print("config", cfg_id, "e2e %.4f s  -> %.3e TFpt-it/s" % (dt, cfg.point_iterations / dt))
    t = time.perf_counter()
    ref = ffr.run_fastfca(y[0], P[0], l[0], v[0], iterations=cfg.iterations, stats=False)
    print("oracle cpu %.3f s" % (time.perf_counter() - t))
    print("config0 P %.2e lam %.2e v %.2e" % (rel(run.params.P, ref.P), rel(run.params.Lam, ref.lam), rel(run.params.v, ref.v)))

cfg = W.CONFIGS[3]
y, P, l, v = W.make(cfg, mixtures=16)
from paper_1805_09498_b200.fastfca import run_fastfca_batch
for rep in range(3):
    t = time.perf_counter()
    out = run_fastfca_batch(y, P, l, v, iterations=20)
    dt = time.perf_counter() - t
    print("config3x16 e2e %.4f s -> %.3e" % (dt, 16 * cfg.N * cfg.F * 20 / dt))
ref = ffr.run_fastfca(y[3].astype(np.complex128), P[3].astype(np.complex128), l[3].astype(np.float64), v[3].astype(np.float64), iterations=20, stats=False)
print("config3 u=3 c64 vs oracle: P %.2e lam %.2e v %.2e" % (rel(out[0][3], ref.P), rel(out[1][3], ref.lam), rel(out[2][3], ref.v)))
