"""End-to-end parity at each BASELINE.json config's full iteration count (north_star).

For configs 1, 2 and 4 the full-size problem is too large for the numpy oracle to run in a
test, so each test runs the config's exact per-bin shape (I, J, N, rank, zero cells, dtype,
launch plan) over a slice of bins -- bins are independent for the whole run (fastfca.py:338-340,
357-358), so a slice is the same computation as those bins of the full problem -- for the
config's FULL iteration count:

  * complex128 run on the same inputs: log-likelihood after every iteration rel <= 1e-6 of
    the oracle's (fastfca.py:390-398 / fca.py:101-116), state rel <= 1e-9;
  * complex64 run: separated images rel-L2 <= 1e-3 against the fp64 oracle's images
    (wiener.py:38-43 / 32-35), state rel <= 1e-4.

rel = max|a - b| / max|b| (test_fastfca.py:364-366); rel-L2 = ||a - b|| / ||b||.
Reference loops: fastfca.py:401-474 (run_fastfca), fca.py:187-215 (run_fca).
"""

import os

import numpy as np
import pytest

from conftest import rel
from oracle import fca_ref
from oracle import fastfca_ref as ffr
from paper_1805_09498_b200 import ObservationTensor, _lib, fastfca, fca, wiener
from paper_1805_09498_b200.workloads import CONFIGS, mixture

pytestmark = pytest.mark.gpu


def relL2(a, b):
    return float(np.linalg.norm((np.asarray(a) - b).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def plan(dt_code, I, J, N, F):
    out = np.zeros(6, np.int32)
    _lib.load().ffca_plan_loop(0, dt_code, 1, I, J, N, F, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip))
    return {"G": int(out[0]), "C": int(out[1]), "threads": int(out[3]), "resident": bool(out[4])}


def c64(*arrs):
    return [a.astype(np.complex64) if np.iscomplexobj(a) else a.astype(np.float32) for a in arrs]


def ll_hist(run):
    return np.array([run.loglik_init] + run.loglik_after_em + run.loglik_after_p)


_REF = {}


def check_fastfca(cfg, seed, F, fp64=True):
    y, P0, lam0, v0, _ = mixture(seed, cfg.I, cfg.J, F, cfg.N, cfg.rank, cfg.zero_frac)
    T = cfg.iterations
    key = (cfg.name, seed, F)
    if key not in _REF:  # the oracle run is the slow part: once per case
        ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=T, record_likelihood=True)
        _REF[key] = (ref, ffr.images(ref.P, ref.mu))
    ref, ref_img = _REF[key]
    ref_ll = np.array([ref.loglik_init] + ref.loglik_after_em + ref.loglik_after_p)

    if fp64:
        r64 = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=T,
                                  record_likelihood=True)
        ll = ll_hist(r64)
        assert len(ll) == 1 + 2 * T
        assert np.abs(ll - ref_ll).max() <= 1e-6 * np.abs(ref_ll).max()
        assert abs(ll[-1] - ref_ll[-1]) <= 1e-6 * abs(ref_ll[-1])
        for got, want in ((r64.params.P, ref.P), (r64.params.Lam, ref.lam), (r64.params.v, ref.v)):
            assert rel(got, want) <= 1e-9

    y32, P32, l32, v32 = c64(y, P0, lam0, v0)
    r32 = fastfca.run_fastfca(ObservationTensor(y32), fastfca.FastFcaParams(P32, l32, v32), iterations=T)
    assert np.isfinite(r32.params.v).all() and np.isfinite(r32.params.P).all()
    for got, want in ((r32.params.P, ref.P), (r32.params.Lam, ref.lam), (r32.params.v, ref.v)):
        assert rel(got, want) <= 1e-4
    img = wiener.mmse_images_fastfca(r32.params, r32.stats).stft
    assert img.dtype == np.complex64
    assert relL2(img, ref_img) <= 1e-3
    return r32


def plan8(I, J, N, F, lean):
    out = np.zeros(8, np.int32)
    _lib.load().ffca_plan_loop_ex(0, _lib.C64, 1, I, J, N, F, _lib.VF_AUTO, lean, out.ctypes.data_as(_lib._ip))
    return {"G": int(out[0]), "C": int(out[1]), "threads": int(out[3]), "tm": int(out[6]), "tmcols": int(out[7])}


def test_config2_long_recording_full_30_iterations():
    # config 2: I = J = 4, N = 9375, rank-8 NMF, complex64, 30 iterations, on 12 bins; one bin
    # exceeds a CTA's shared memory.  The plain loop keeps the y records in tensor memory (256
    # columns per CTA) and splits a bin over a 4-CTA cluster; shared memory alone (the loop with the
    # likelihood record, or FFCA_NO_TMEM) needs an 8-CTA cluster.  DSMEM reductions in rank order
    # twice per iteration either way; both plans are held to the same tolerances.
    cfg = CONFIGS[2]
    p = plan8(cfg.I, cfg.J, cfg.N, 12, 1)
    assert p["C"] == 4 and p["tm"] == 1 and p["tmcols"] == 256 and p["threads"] == 128
    assert plan8(cfg.I, cfg.J, cfg.N, 12, 0)["C"] == 8 and plan8(cfg.I, cfg.J, cfg.N, 12, 0)["tm"] == 0
    r_tm = check_fastfca(cfg, 2, 12)
    os.environ["FFCA_NO_TMEM"] = "1"
    try:
        assert plan(_lib.C64, cfg.I, cfg.J, cfg.N, 12)["C"] == 8
        r_sm = check_fastfca(cfg, 2, 12, fp64=False)
    finally:
        os.environ.pop("FFCA_NO_TMEM", None)
    assert rel(r_tm.params.P, r_sm.params.P) <= 1e-5 and rel(r_tm.params.v, r_sm.params.v) <= 1e-5


def test_config4_large_array_full_20_iterations():
    # config 4: I = 8, J = 6, N = 4000, 10 % zero (n, f) cells per source, complex64, 20
    # iterations, on 8 bins; the default plan holds each bin in a CTA pair (2 x 2000 frames)
    cfg = CONFIGS[4]
    p = plan(_lib.C64, cfg.I, cfg.J, cfg.N, 8)
    assert p["C"] == 2 and p["resident"] and p["threads"] == 256
    check_fastfca(cfg, 4, 8)


def test_config0_shape_batch_full_20_iterations_matches_single():
    # config 3 = 256 config-0 mixtures: two of them in one batch, full 20 iterations, complex64,
    # against the fp64 oracle per mixture
    cfg = CONFIGS[3]
    T = cfg.iterations
    parts = [mixture(900 + u, cfg.I, cfg.J, cfg.F, cfg.N, cfg.rank) for u in range(2)]
    y, P0, lam0, v0 = (np.stack([p[k] for p in parts]) for k in range(4))
    P, lam, v, ll = fastfca.run_fastfca_batch(*c64(y, P0, lam0, v0), iterations=T, record_likelihood=True)
    for u in range(2):
        ref = ffr.run_fastfca(y[u], P0[u], lam0[u], v0[u], iterations=T, record_likelihood=True, stats=False)
        assert rel(P[u], ref.P) <= 1e-4 and rel(lam[u], ref.lam) <= 1e-4 and rel(v[u], ref.v) <= 1e-4
        assert abs(ll[u, -1] - ref.loglik_after_p[-1]) <= 1e-4 * abs(ref.loglik_after_p[-1])


def test_config1_fca_full_20_iterations():
    # config 1: conventional FCA on the config-0 generator, I = J = 3, F = 513, N = 626,
    # 20 iterations, complex128 (fca.py:187-215); complex64 images against the fp64 oracle
    cfg = CONFIGS[1]
    T = cfg.iterations
    y, _, _, v0, _ = mixture(0, cfg.I, cfg.J, cfg.F, cfg.N, cfg.rank)
    S0 = np.broadcast_to(np.eye(cfg.I, dtype=complex), (cfg.J, cfg.F, cfg.I, cfg.I)).copy()
    ref = fca_ref.run_fca(y, S0, v0, iterations=T, record_likelihood=True)
    run = fca.run_fca(ObservationTensor(y), fca.FcaParams(S0, v0), iterations=T, record_likelihood=True)
    ll = np.array(run.loglik)
    assert len(ll) == T + 1
    assert np.abs(ll - ref.loglik).max() <= 1e-6 * np.abs(ref.loglik).max()
    assert abs(ll[-1] - ref.loglik[-1]) <= 1e-6 * abs(ref.loglik[-1])
    assert rel(run.params.S, ref.S) <= 1e-9 and rel(run.params.v, ref.v) <= 1e-9
    ref_img = wiener_fca_oracle(ref.S, ref.v, y)
    assert relL2(wiener.mmse_images_fca(run.params, ObservationTensor(y)).stft, ref_img) <= 1e-9

    y32, S32, v32 = c64(y, S0, v0)
    r32 = fca.run_fca(ObservationTensor(y32), fca.FcaParams(S32, v32), iterations=T)
    assert rel(r32.params.S, ref.S) <= 1e-4 and rel(r32.params.v, ref.v) <= 1e-4
    img = wiener.mmse_images_fca(r32.params, ObservationTensor(y32)).stft
    assert img.dtype == np.complex64
    assert relL2(img, ref_img) <= 1e-3


def wiener_fca_oracle(S, v, y):
    """Images (J, I, N, F) = mu of one more E-step at the final state (wiener.py:32-35)."""
    mu, _ = fca_ref.e_step(S, v, y)  # (J, N, F, I)
    return np.ascontiguousarray(np.transpose(mu, (0, 3, 1, 2)))
