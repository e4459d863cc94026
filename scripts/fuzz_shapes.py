"""One-off shape fuzz against the oracle: mid-length bins across (I, J), both precisions, lean and
likelihood-recording loops, statistics and images.  Prints the worst relative errors and every failure."""
import os, sys, itertools, json
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
from oracle import fastfca_ref as ffr
from paper_1805_09498_b200 import ObservationTensor, fastfca
from paper_1805_09498_b200.workloads import mixture


def rel(a, b):
    return float(np.abs(np.asarray(a) - b).max() / max(np.abs(b).max(), 1e-300))


worst = {"c128": 0.0, "c64": 0.0}
fails = []
shapes = [(2, 2), (3, 3), (4, 4), (3, 2), (1, 2), (5, 3), (6, 6), (8, 6)]
Ns = [65, 97, 129, 160, 257, 384, 449, 500, 641, 700, 1000, 2100]
for (I, J), N in itertools.product(shapes, Ns):
    F = 5 if N < 1500 else 3
    y, P0, lam0, v0, _ = mixture(31 * N + I, I, J, F, N, 4, 0.0)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=2)
    ref_img = ffr.images(ref.P, ref.mu)
    for dt in ("c128", "c64"):
        if dt == "c64":
            a = (y.astype(np.complex64), P0.astype(np.complex64), lam0.astype(np.float32), v0.astype(np.float32))
        else:
            a = (y, P0, lam0, v0)
        tol = 1e-9 if dt == "c128" else 2e-4
        for rec in (False, True):
            run = fastfca.run_fastfca(ObservationTensor(a[0]), fastfca.FastFcaParams(*a[1:]), iterations=2,
                                      record_likelihood=rec)
            errs = [rel(run.params.P, ref.P), rel(run.params.Lam, ref.lam), rel(run.params.v, ref.v),
                    rel(run.stats.mu, ref.mu), rel(fastfca.images_from_state(ObservationTensor(a[0]), run.params), ref_img)]
            e = max(errs)
            worst[dt] = max(worst[dt], e)
            if not e <= tol:
                fails.append({"I": I, "J": J, "N": N, "dt": dt, "rec": rec, "errs": [float(f"{x:.2e}") for x in errs]})
print(json.dumps({"cases": len(shapes) * len(Ns) * 4, "worst": worst, "fails": fails}))
