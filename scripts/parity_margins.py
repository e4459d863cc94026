"""Print the actual parity margins (not just pass/fail) against the reference golden vectors."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np

from paper_1805_09498_b200 import ObservationTensor, fastfca, wiener

g = dict(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden.npz")))


def rel(a, b):
    return float(np.abs(np.asarray(a) - b).max() / np.abs(b).max())


for key in ["g33", "g44", "g86", "g22", "g12", "g23"]:
    for dt in ("c128", "c64"):
        def c(a):
            if dt != "c64":
                return a
            return a.astype(np.complex64) if np.iscomplexobj(a) else a.astype(np.float32)

        run = fastfca.run_fastfca(ObservationTensor(c(g[key + "/y"])),
                                  fastfca.FastFcaParams(c(g[key + "/P0"]), c(g[key + "/lam0"]), c(g[key + "/v0"])),
                                  iterations=int(g[key + "/iters"]), record_likelihood=True)
        ll = np.array([run.loglik_init] + run.loglik_after_em + run.loglik_after_p)
        e = max(rel(run.params.P, g[key + "/P"]), rel(run.params.Lam, g[key + "/lam"]), rel(run.params.v, g[key + "/v"]),
                rel(wiener.mmse_images_fastfca(run.params, run.stats).stft, g[key + "/images"]))
        lle = float(np.abs(ll - g[key + "/ll"]).max() / np.abs(g[key + "/ll"]).max())
        print(f"{key} {dt}: state/images rel {e:.2e}  loglik rel {lle:.2e}", flush=True)
