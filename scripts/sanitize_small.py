"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np

from paper_1805_09498_b200 import ObservationTensor, fastfca, fca, wiener
from paper_1805_09498_b200.workloads import mixture


def run(I, J, F, N, c64=False, plan=None, it=2, rank=4, zf=0.0):
    if plan:
        os.environ["FFCA_FORCE_PLAN"] = plan
    else:
        os.environ.pop("FFCA_FORCE_PLAN", None)
    y, P0, lam0, v0, _ = mixture(3, I, J, F, N, rank, zf)
    if c64:
        y, P0, lam0, v0 = y.astype(np.complex64), P0.astype(np.complex64), lam0.astype(np.float32), v0.astype(np.float32)
    r = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=it,
                            record_likelihood=True)
    wiener.mmse_images_fastfca(r.params, r.stats)
    _ = r.stats.mu
    print("ok", I, J, F, N, c64, plan, flush=True)


run(3, 3, 9, 40, c64=True)                 # c64 I=J=3: 2-bin CTAs, frame-pair records
run(3, 3, 9, 41, c64=True)                 # odd frame count: the half-filled last pair
run(3, 3, 9, 41, c64=True, plan="1,2,1")   # frame pairs split over a cluster (odd per-rank counts)
run(3, 3, 300, 30)                         # c128 one-bin CTAs with 16-lane reduction segments
run(3, 3, 7, 40)                           # c128 G=2
run(3, 3, 5, 90, c64=True, plan="1,2,1")   # cluster of 2
run(4, 4, 5, 70, c64=True, plan="1,4,1")   # I=4 cluster of 4
run(3, 2, 5, 50, plan="1,1,0")             # global slab
run(8, 6, 3, 48, c64=True, zf=0.1)         # I=8 group mode
run(8, 6, 3, 64, c64=True, plan="1,2,1")   # I=8 cluster
run(5, 3, 3, 40)                           # generic I=5
os.environ.pop("FFCA_FORCE_PLAN", None)
y, _, _, v0, _ = mixture(4, 3, 3, 5, 30)
S0 = np.broadcast_to(np.eye(3, dtype=complex), (3, 5, 3, 3)).copy()
rf = fca.run_fca(ObservationTensor(y), fca.FcaParams(S0, v0), iterations=2, record_likelihood=True)
_ = rf.stats.phi
m = fca.m_step(rf.stats, fca.FcaParams(S0, v0), 0.0)
fastfca.params_from_covariances(S0 + 0.1, v0)
print("all ok", flush=True)

# output-side tiles (statistics refresh / images: cp.async ring, staged stores, partial tiles),
# initialisers, STFT, SDR and the device pipeline
from paper_1805_09498_b200 import pipeline, scene  # noqa: E402

for c64 in (True, False):
    run(3, 3, 45, 50, c64=c64)   # F=45: one full and one partial 32-bin tile
    run(2, 4, 33, 17, c64=c64)
rng = np.random.default_rng(0)
refs = rng.standard_normal((2, 2, 3000))
for algo in ("fastfca", "fca"):
    for init in ("oracle", "diffuse"):
        pipeline.separate_once(pipeline.PipelineConfig(algorithm=algo, init=init, iterations=2, sources=2,
                                                       frame_length=256, frame_shift=128), refs.sum(axis=0), refs)
print("ok pipeline", flush=True)
