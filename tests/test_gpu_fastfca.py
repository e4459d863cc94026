"""GPU parity of the FastFCA-AS path against the CPU oracle and the reference golden vectors.

Tolerances (BASELINE.json north_star):
  per-iteration state check   rel <= 1e-10 (complex128), <= 1e-4 (complex64)
  end to end                  log-likelihood rel <= 1e-6 (fp64); images rel-L2 <= 1e-3 (fp32)
rel = max|a - b| / max|b| (test_fastfca.py:364-366) unless stated.
"""

import os

import numpy as np
import pytest

from conftest import rel
from oracle import fastfca_ref as ffr
from paper_1805_09498_b200 import ObservationTensor, _lib, errors, fastfca, wiener
from paper_1805_09498_b200.workloads import CONFIGS, mixture

pytestmark = pytest.mark.gpu

CASES = ["g33", "g44", "g86", "g22", "g12", "g23"]
TOL = {"c128": 1e-10, "c64": 1e-4}


def relL2(a, b):
    return float(np.linalg.norm((np.asarray(a) - b).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def case(golden, key):
    return {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith(key + "/")}


def cast(dt, *arrs):
    out = []
    for a in arrs:
        if dt == "c64":
            a = a.astype(np.complex64) if np.iscomplexobj(a) else a.astype(np.float32)
        out.append(a)
    return out


@pytest.fixture(autouse=True)
def _plan_env():
    old = os.environ.pop("FFCA_FORCE_PLAN", None)
    yield
    os.environ.pop("FFCA_FORCE_PLAN", None)
    if old is not None:
        os.environ["FFCA_FORCE_PLAN"] = old


# ---------------------------------------------------------------------------
# against the unmodified reference (golden vectors)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("dt", ["c128", "c64"])
@pytest.mark.parametrize("key", CASES)
def test_fused_loop_golden(golden, key, dt):
    g = case(golden, key)
    y, P0, lam0, v0 = cast(dt, g["y"], g["P0"], g["lam0"], g["v0"])
    it = int(g["iters"])
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=it,
                              record_likelihood=True)
    tol = TOL[dt] * (1 if dt == "c128" else 1)
    assert rel(run.params.P, g["P"]) <= tol
    assert rel(run.params.Lam, g["lam"]) <= tol
    assert rel(run.params.v, g["v"]) <= tol
    assert run.counters.inversions == int(g["inversions"]) and run.counters.matmuls == 0
    ll = np.array([run.loglik_init] + run.loglik_after_em + run.loglik_after_p)
    assert np.abs(ll - g["ll"]).max() <= (1e-12 if dt == "c128" else 1e-6) * np.abs(g["ll"]).max()
    assert rel(run.stats.mu, g["mu"]) <= tol
    assert rel(run.stats.phi, g["phi"]) <= tol
    images = wiener.mmse_images_fastfca(run.params, run.stats).stft
    assert rel(images, g["images"]) <= tol


def test_inner_iterations_scalar_floor_golden(golden):
    g = case(golden, "k2")
    run = fastfca.run_fastfca(ObservationTensor(g["y"]), fastfca.FastFcaParams(g["P0"], g["lam0"], g["v0"]),
                              iterations=3, inner_iterations=2, v_floor=0.0)
    assert rel(run.params.P, g["P"]) <= 1e-10
    assert rel(run.params.Lam, g["lam"]) <= 1e-10
    assert rel(run.params.v, g["v"]) <= 1e-10
    assert run.counters.inversions == int(g["inversions"])


def test_unfused_steps_golden(golden):
    g = case(golden, "step")
    y, P, lam, v = g["y"], g["P"], g["lam"], g["v"]
    obs = ObservationTensor(y)
    params = fastfca.FastFcaParams(P, lam, v)
    yt = fastfca.transform_observations(P, obs)
    assert rel(yt, g["yt"]) <= 1e-13
    assert rel(fastfca.mixture_weights(params), g["w"]) <= 1e-14
    st = fastfca.e_step_diag(params, yt)
    assert rel(st.mu, g["mu"]) <= 1e-12 and rel(st.phi, g["phi"]) <= 1e-12
    em = fastfca.m_step_diag(st, params, v_floor=0.05)
    assert rel(em.v, g["v_em"]) <= 1e-12 and rel(em.Lam, g["lam_em"]) <= 1e-12
    Pn = fastfca.fixed_point_update_P(em, obs, inner_iterations=2)
    assert rel(Pn, g["P_new"]) <= 1e-10
    ll = fastfca.log_likelihood(params, obs)
    assert abs(ll - float(g["ll"])) <= 1e-12 * abs(float(g["ll"]))
    assert rel(fastfca.back_transform_means(P, st.mu), g["back"]) <= 1e-12
    one = fastfca.run_fastfca(obs, params, iterations=1, v_floor=0.0)
    assert rel(one.params.P, g["one_iter_P"]) <= 1e-10


# ---------------------------------------------------------------------------
# per-iteration state check (same state fed into one iteration)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("dt", ["c128", "c64"])
@pytest.mark.parametrize("shape", [(3, 3, 40, 200), (4, 4, 12, 300), (8, 6, 6, 160), (2, 3, 9, 77)])
def test_one_iteration_from_state(dt, shape):
    I, J, F, N = shape
    y, P0, lam0, v0, _ = mixture(31 + I, I, J, F, N, 4, 0.0)
    st = ffr.run_fastfca(y, P0, lam0, v0, iterations=3, stats=False)  # a non-trivial state
    y_, P_, l_, v_ = cast(dt, y, st.P, st.lam, st.v)
    # the oracle sees exactly the (possibly rounded) state the GPU sees
    y64, P64, l64, v64 = (a.astype(np.complex128) if np.iscomplexobj(a) else a.astype(np.float64)
                          for a in (y_, P_, l_, v_))
    vf = ffr.power_floor(y64)
    ref = ffr.run_fastfca(y64, P64, l64, v64, iterations=1, v_floor=vf, stats=False)
    run = fastfca.run_fastfca(ObservationTensor(y_), fastfca.FastFcaParams(P_, l_, v_), iterations=1,
                              v_floor=vf)
    tol = TOL[dt]
    assert rel(run.params.v, ref.v) <= tol
    assert rel(run.params.Lam, ref.lam) <= tol
    assert rel(run.params.P, ref.P) <= tol


# ---------------------------------------------------------------------------
# end to end at BASELINE config 0 (full size) and the complex64 path on it
# ---------------------------------------------------------------------------


@pytest.fixture(scope="module")
def config0():
    cfg = CONFIGS[0]
    y, P0, lam0, v0, _ = mixture(0, cfg.I, cfg.J, cfg.F, cfg.N, cfg.rank)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=cfg.iterations, record_likelihood=True)
    return cfg, (y, P0, lam0, v0), ref


def test_end_to_end_config0_fp64(config0):
    cfg, (y, P0, lam0, v0), ref = config0
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0),
                              iterations=cfg.iterations, record_likelihood=True)
    assert abs(run.loglik_after_p[-1] - ref.loglik_after_p[-1]) <= 1e-6 * abs(ref.loglik_after_p[-1])
    lls = np.array(run.loglik_after_p)
    assert np.abs(lls - ref.loglik_after_p).max() <= 1e-10 * abs(ref.loglik_after_p[-1])
    assert rel(run.params.P, ref.P) <= 1e-10
    assert rel(run.params.v, ref.v) <= 1e-10
    images = wiener.mmse_images_fastfca(run.params, run.stats).stft
    assert relL2(images, ffr.images(ref.P, ref.mu)) <= 1e-10


def test_end_to_end_config0_fp32(config0):
    cfg, (y, P0, lam0, v0), ref = config0
    y32, P32, l32, v32 = cast("c64", y, P0, lam0, v0)
    run = fastfca.run_fastfca(ObservationTensor(y32), fastfca.FastFcaParams(P32, l32, v32),
                              iterations=cfg.iterations, record_likelihood=True)
    images = wiener.mmse_images_fastfca(run.params, run.stats).stft
    assert images.dtype == np.complex64
    assert relL2(images, ffr.images(ref.P, ref.mu)) <= 1e-3
    assert abs(run.loglik_after_p[-1] - ref.loglik_after_p[-1]) <= 1e-4 * abs(ref.loglik_after_p[-1])


# ---------------------------------------------------------------------------
# launch-plan coverage: clusters (DSMEM reduction) and the global-slab path
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("plan", ["1,2,1", "1,4,1", "1,8,1", "1,1,0", "1,4,0", "4,1,1", "2,1,1", "1,1,1", "1,1,1,64"])
@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_forced_plans_agree(plan, dt):
    y, P0, lam0, v0, _ = mixture(77, 3, 3, 11, 150, 4, 0.0)
    y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
    base = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=4,
                               record_likelihood=True)
    os.environ["FFCA_FORCE_PLAN"] = plan
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=4,
                              record_likelihood=True)
    tol = 1e-12 if dt == "c128" else 1e-5
    assert rel(run.params.P, base.params.P) <= tol
    assert rel(run.params.v, base.params.v) <= tol
    lltol = 1e-12 if dt == "c128" else 1e-6  # fp32 partial sums are grouped differently per plan
    assert abs(run.loglik_after_p[-1] - base.loglik_after_p[-1]) <= lltol * abs(base.loglik_after_p[-1])


@pytest.mark.parametrize("plan", [None, "1,2,1", "1,4,1", "4,1,1", "2,1,1", "1,1,1"])
@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_packed_slab_gather_agrees(plan, dt):
    # slab images written by the pack pass and bulk-copied into shared memory (the default for the
    # I > 4 one-CTA-per-SM plans; forced here for every resident plan): bitwise the element gather,
    # incl. uneven cluster frame splits (N = 150 over 4 ranks) and groups straddling mixtures
    U, I, J, F, N = 3, 3, 3, 11, 150
    ys, Ps, ls, vs = [], [], [], []
    for u in range(U):
        y, P0, lam0, v0, _ = mixture(80 + u, I, J, F, N, 4, 0.0)
        y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
        ys.append(y); Ps.append(P0); ls.append(lam0); vs.append(v0)
    y, P0, lam0, v0 = (np.stack(a) for a in (ys, Ps, ls, vs))
    if plan:
        os.environ["FFCA_FORCE_PLAN"] = plan
    base = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=4, record_likelihood=True)
    os.environ["FFCA_FORCE_PACK"] = "1"
    try:
        run = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=4, record_likelihood=True)
    finally:
        os.environ.pop("FFCA_FORCE_PACK", None)
    for a, b in zip(run, base):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("IJ", [(5, 2), (6, 3), (7, 4), (8, 6)])
@pytest.mark.parametrize("K", [1, 2])
@pytest.mark.parametrize("plan", [None, "1,2,1,256"])
@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_many_channels_against_oracle(IJ, K, plan, dt):
    # I > 4 kernels: odd I (a diagonal pair with a dummy half in the phase-B units), runtime J
    # (I = 5..7) and the config-4 instantiation (8, 6); K = 2 exercises the in-solve P^-1 of the
    # later inner iterations; "1,2,1,256" is the config-4 plan (CTA pair, 256 threads, the last
    # warp inverting P during phase B).  Likelihood recording covers log|det P| from that warp.
    I, J = IJ
    y, P0, lam0, v0, _ = mixture(40 + I + J, I, J, 3, 160, 4, 0.05)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=3, inner_iterations=K, record_likelihood=True, stats=False)
    y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
    if plan:
        os.environ["FFCA_FORCE_PLAN"] = plan
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=3,
                              inner_iterations=K, record_likelihood=True)
    tol = 1e-10 if dt == "c128" else 1e-4
    assert rel(run.params.P, ref.P) <= tol
    assert rel(run.params.Lam, ref.lam) <= tol
    assert rel(run.params.v, ref.v) <= tol
    ll = np.array([run.loglik_init] + run.loglik_after_em + run.loglik_after_p)
    rll = np.array([ref.loglik_init] + ref.loglik_after_em + ref.loglik_after_p)
    assert np.abs(ll - rll).max() <= (1e-10 if dt == "c128" else 1e-5) * np.abs(rll).max()


@pytest.mark.parametrize("plan", [None, "1,2,1,256", "1,4,1,256"])
@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_many_channels_full_floor_array(plan, dt):
    # I > 4 with a full (J, N, F) floor (vf_mode 2: the floor records ride in the slab, no pack
    # pass), incl. CTA pairs / quads
    I, J = 8, 6
    y, P0, lam0, v0, _ = mixture(71, I, J, 3, 160, 4, 0.05)
    vf = np.random.default_rng(5).uniform(0.0, 0.05, (J, 160, 3)) * v0.mean()
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=3, v_floor=vf, stats=False)
    y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
    if plan:
        os.environ["FFCA_FORCE_PLAN"] = plan
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=3,
                              v_floor=vf)
    tol = 1e-10 if dt == "c128" else 1e-4
    assert rel(run.params.P, ref.P) <= tol
    assert rel(run.params.Lam, ref.lam) <= tol
    assert rel(run.params.v, ref.v) <= tol


def test_long_recording_slice_cluster_path():
    # config-2 shape (I=J=4, N=9375, rank-8 NMF, complex64) on a few bins: the
    # bin is longer than one CTA's shared memory, so a cluster splits the frames
    cfg = CONFIGS[2]
    F = 6
    y, P0, lam0, v0, _ = mixture(2, cfg.I, cfg.J, F, cfg.N, cfg.rank)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=5, stats=False)
    out = (np.zeros(6, np.int32))
    _lib.load().ffca_plan_loop(0, _lib.C64, 1, cfg.I, cfg.J, cfg.N, F, _lib.VF_AUTO,
                               out.ctypes.data_as(_lib._ip))
    assert out[1] > 1  # clustered
    y32, P32, l32, v32 = cast("c64", y, P0, lam0, v0)
    run = fastfca.run_fastfca(ObservationTensor(y32), fastfca.FastFcaParams(P32, l32, v32), iterations=5)
    assert rel(run.params.P, ref.P) <= 1e-4
    assert rel(run.params.Lam, ref.lam) <= 1e-4
    assert rel(run.params.v, ref.v) <= 1e-4


def test_large_array_slice_with_zero_cells():
    # config-4 shape (I=8, J=6, N=4000, 10% zero cells) on a few bins
    cfg = CONFIGS[4]
    F = 4
    y, P0, lam0, v0, _ = mixture(4, cfg.I, cfg.J, F, cfg.N, cfg.rank, cfg.zero_frac)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=3, stats=False)
    run64 = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=3)
    assert rel(run64.params.P, ref.P) <= 1e-10 and rel(run64.params.v, ref.v) <= 1e-10
    y32, P32, l32, v32 = cast("c64", y, P0, lam0, v0)
    run = fastfca.run_fastfca(ObservationTensor(y32), fastfca.FastFcaParams(P32, l32, v32), iterations=3)
    assert np.isfinite(run.params.v).all() and np.isfinite(run.params.P).all()
    assert rel(run.params.P, ref.P) <= 1e-4
    assert rel(run.params.Lam, ref.lam) <= 1e-4
    assert rel(run.params.v, ref.v) <= 1e-4


# ---------------------------------------------------------------------------
# batching, determinism, floors, edge cases, errors
# ---------------------------------------------------------------------------


def test_batch_equals_single_mixtures_bitwise():
    ys, Ps, ls, vs = [], [], [], []
    for s in range(3):
        y, P0, lam0, v0, _ = mixture(100 + s, 3, 3, 13, 50)
        ys.append(y), Ps.append(P0), ls.append(lam0), vs.append(v0)
    Pb, lb, vb, llb = fastfca.run_fastfca_batch(np.stack(ys), np.stack(Ps), np.stack(ls), np.stack(vs),
                                                iterations=4, record_likelihood=True)
    for u in range(3):
        run = fastfca.run_fastfca(ObservationTensor(ys[u]), fastfca.FastFcaParams(Ps[u], ls[u], vs[u]),
                                  iterations=4, record_likelihood=True)
        assert np.array_equal(run.params.P, Pb[u])
        assert np.array_equal(run.params.v, vb[u])
        assert run.loglik_after_p[-1] == llb[u, -1]


def test_deterministic_bitwise():
    y, P0, lam0, v0, _ = mixture(9, 4, 4, 17, 300, 8)
    a = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=6)
    b = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=6)
    assert np.array_equal(a.params.P, b.params.P) and np.array_equal(a.params.v, b.params.v)


@pytest.mark.parametrize("kind", ["bin", "full", "scalar"])
def test_floor_modes(kind):
    y, P0, lam0, v0, _ = mixture(3, 3, 2, 9, 60)
    J, N, F = v0.shape
    if kind == "bin":
        vf = 0.3 * ffr.power_floor(y) * 1e9  # large enough to bind
    elif kind == "full":
        vf = np.random.default_rng(1).uniform(0.0, 0.2, (J, N, F)) * np.abs(y).mean() ** 2
    else:
        vf = 0.05
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=3, v_floor=vf, stats=False)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=3,
                              v_floor=vf)
    assert rel(run.params.v, ref.v) <= 1e-10 and rel(run.params.P, ref.P) <= 1e-10


def test_zero_iterations_keeps_params():
    y, P0, lam0, v0, _ = mixture(4, 2, 2, 3, 5)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=0,
                              record_likelihood=True)
    assert np.array_equal(run.params.P, P0) and np.array_equal(run.params.v, v0)
    assert run.counters.inversions == 0
    assert run.stats.mu.shape == (2, 5, 3, 2)
    assert run.loglik_after_em == [] and run.loglik_after_p == []
    assert abs(run.loglik_init - ffr.log_likelihood(P0, lam0, v0, y)) <= 1e-12 * abs(run.loglik_init)


def test_single_frame_single_channel():
    y, P0, lam0, v0, _ = mixture(6, 1, 2, 4, 1)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=2, stats=False)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=2)
    assert rel(run.params.P, ref.P) <= 1e-10 and rel(run.params.v, ref.v) <= 1e-10


def test_singular_P_raises():
    y, P0, lam0, v0, _ = mixture(8, 2, 2, 3, 10)
    P0[1] = 0.0
    with pytest.raises(errors.SingularP):
        fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=1)


@pytest.mark.parametrize("dt", ["c128", "c64"])
@pytest.mark.parametrize("how", ["zero_row", "zero_col", "repeated_col"])
def test_singular_P_order3(dt, how):
    # I = 3 rows of P^-1 come from the adjugate: an exactly zero determinant raises SingularP.
    # Zero rows / columns raise in the reference too (zero LU pivot); for a repeated column the
    # reference raises only when LAPACK's pivot happens to round to exactly zero (documented
    # divergence).
    y, P0, lam0, v0, _ = mixture(9, 3, 3, 4, 12)
    y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
    if how == "zero_row":
        P0[2, 1, :] = 0.0
    elif how == "zero_col":
        P0[2, :, 0] = 0.0
    else:
        P0[2, :, 2] = P0[2, :, 0]
    with pytest.raises(errors.SingularP):
        fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=1)
    if how != "repeated_col":
        with pytest.raises(ffr.OracleSingular):
            ffr.run_fastfca(y.astype(np.complex128), P0.astype(np.complex128), lam0.astype(np.float64),
                            v0.astype(np.float64), iterations=1)


def test_zero_bin_raises_singular_weighted_covariance():
    y, P0, lam0, v0, _ = mixture(8, 2, 2, 3, 10)
    y[:, :, 2] = 0.0  # B_i = 0 for that bin, stays singular after trace loading
    with pytest.raises(errors.SingularWeightedCovariance):
        fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=1)
    with pytest.raises(ffr.OracleSingular):
        ffr.run_fastfca(y, P0, lam0, v0, iterations=1)


def test_channel_mismatch_raises():
    y, P0, lam0, v0, _ = mixture(8, 3, 2, 3, 10)
    with pytest.raises(errors.DimensionMismatch):
        fastfca.run_fastfca(ObservationTensor(y[:2]), fastfca.FastFcaParams(P0, lam0, v0), iterations=1)


def test_partition_identity_images():
    # sum_j x_j = y (test_wiener.py:56-74; acceptance criterion 8)
    y, P0, lam0, v0, _ = mixture(12, 3, 3, 16, 40)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=5)
    fused = fastfca.images_from_state(ObservationTensor(y), run.params)
    assert np.abs(fused.sum(axis=0) - y).max() <= 1e-8 * np.abs(y).max()
    explicit = wiener.mmse_images_fastfca(run.params, run.stats).stft
    assert np.abs(explicit.sum(axis=0) - y).max() <= 1e-8 * np.abs(y).max()
    assert rel(fused, explicit) <= 1e-12


def test_stats_are_a_snapshot_of_the_final_state():
    # the reference refreshes the statistics eagerly (fastfca.py:466): changing run.params
    # afterwards must not change run.stats; the stats types are dataclasses (fastfca.py:87-96)
    import dataclasses
    y, P0, lam0, v0, _ = mixture(13, 3, 3, 8, 30)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=3)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=3)
    mu0 = run.stats.mu.copy()
    run.params.P[...] = 0.0
    run.params.v *= 2.0
    assert np.array_equal(run.stats.mu, mu0)
    assert rel(run.stats.mu, ref.mu) <= 1e-10 and rel(run.stats.phi, ref.phi) <= 1e-10
    st = dataclasses.replace(run.stats, phi=None)
    assert st.phi is None and set(dataclasses.asdict(run.stats)) == {"mu", "phi"}


def test_batch_stats_match_single_runs():
    y, P0, lam0, v0 = _stack(range(530, 533), 3, 3, 10, 45)
    P, lam, v, ll, mu, phi = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=4, stats=True)
    for u in range(3):
        run = fastfca.run_fastfca(ObservationTensor(y[u]), fastfca.FastFcaParams(P0[u], lam0[u], v0[u]),
                                  iterations=4)
        assert np.array_equal(run.stats.mu, mu[u]) and np.array_equal(run.stats.phi, phi[u])
    os.environ["FFCA_PIPELINE_MIN_BYTES"] = "1"  # chunked host pipeline with the stats outputs
    try:
        got = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=4, stats=True)
    finally:
        os.environ.pop("FFCA_PIPELINE_MIN_BYTES")
    assert np.array_equal(got[4], mu) and np.array_equal(got[5], phi) and np.array_equal(got[2], v)
    one = fastfca.run_fastfca_batch(y[:1], P0[:1], lam0[:1], v0[:1], iterations=4, stats=True)
    os.environ["FFCA_PIPELINE_MIN_BYTES"] = "1"  # one mixture: frequency-block chunks
    try:
        blk = fastfca.run_fastfca_batch(y[:1], P0[:1], lam0[:1], v0[:1], iterations=4, stats=True)
    finally:
        os.environ.pop("FFCA_PIPELINE_MIN_BYTES")
    for a, b in zip(blk, one):
        if a is not None:
            assert np.array_equal(a, b)


def test_launch_count_is_one_kernel():
    y, P0, lam0, v0, _ = mixture(12, 3, 3, 16, 40)
    fastfca.run_fastfca_batch(y[None], P0[None], lam0[None], v0[None], iterations=20)
    assert _lib.launches() == 2  # the whole 20-iteration loop + the per-bin status summary
    fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=20)
    assert _lib.launches() == 3  # + the final statistics refresh (fastfca.py:466)


@pytest.mark.parametrize("shape", [(5, 3, 3, 40, 70), (1, 4, 4, 37, 300)])
def test_pipelined_host_call_is_bitwise_one_launch(shape):
    U, I, J, F, N = shape
    ys, Ps, ls, vs = [], [], [], []
    for u in range(U):
        y, P0, lam0, v0, _ = mixture(200 + u, I, J, F, N, 4)
        ys.append(y), Ps.append(P0), ls.append(lam0), vs.append(v0)
    args = (np.stack(ys), np.stack(Ps), np.stack(ls), np.stack(vs))
    os.environ["FFCA_NO_PIPELINE"] = "1"
    ref = fastfca.run_fastfca_batch(*args, iterations=3, record_likelihood=True)
    os.environ.pop("FFCA_NO_PIPELINE")
    os.environ["FFCA_PIPELINE_MIN_BYTES"] = "1"
    try:
        got = fastfca.run_fastfca_batch(*args, iterations=3, record_likelihood=True)
    finally:
        os.environ.pop("FFCA_PIPELINE_MIN_BYTES")
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_back_transform_stats_reconstruct_and_init_golden(golden):
    g = case(golden, "step")
    params = fastfca.FastFcaParams(g["P"], g["lam"], g["v"])
    st = fastfca.e_step_diag(params, fastfca.transform_observations(g["P"], ObservationTensor(g["y"])))
    mu, phi = fastfca.back_transform_stats(params, st)
    assert rel(mu, g["bt_mu"]) <= 1e-12 and rel(phi, g["bt_phi"]) <= 1e-12
    assert rel(fastfca.reconstruct_spatial_covariances(params), g["S"]) <= 1e-12
    assert rel(fastfca.reconstruct_spatial_covariance(params, 1, 2), g["S01"]) <= 1e-12
    h = case(golden, "init")
    init = fastfca.params_from_covariances(h["S_hat"], h["v_hat"])
    assert rel(init.P, h["P"]) <= 1e-12 and rel(init.Lam, h["Lam"]) <= 1e-12
    with pytest.raises(errors.NotPositiveDefinite):
        fastfca.params_from_covariances(-h["S_hat"], h["v_hat"])


def test_equivalence_to_full_fca_estep(rng):
    # acceptance criterion 2 (test_acceptance.py:132-176): the back-transformed
    # diagonal-path E-step equals the full-matrix E-step on the reconstructed S
    from paper_1805_09498_b200 import fca
    worst = 0.0
    for order in (2, 3, 4):
        for trial in range(6):
            r = np.random.default_rng(1000 * order + trial)
            P = r.standard_normal((4, order, order)) + 1j * r.standard_normal((4, order, order)) + 2 * np.eye(order)
            params = fastfca.FastFcaParams(P, r.uniform(0.5, 2.0, (order, 4, order)),
                                           r.uniform(0.5, 2.0, (order, 8, 4)))
            obs = ObservationTensor(r.standard_normal((order, 8, 4)) + 1j * r.standard_normal((order, 8, 4)))
            st = fastfca.e_step_diag(params, fastfca.transform_observations(P, obs))
            mu, phi = fastfca.back_transform_stats(params, st)
            full = fca.FcaParams(S=fastfca.reconstruct_spatial_covariances(params), v=params.v)
            ref = fca.e_step(full, obs)
            worst = max(worst, np.abs(mu - ref.mu).max(), np.abs(phi - ref.phi).max())
            l1, l2 = fca.log_likelihood(full, obs), fastfca.log_likelihood(params, obs)
            assert abs(l2 - l1) <= 1e-8 * abs(l1)
    assert worst <= 1e-8


def _model_observation(rng, params):
    """y ~ CN(0, sum_j v_j S_j) from the jointly diagonalized model (test_fastfca.py:23-36 pattern)."""
    J, N, F = params.v.shape
    S = fastfca.reconstruct_spatial_covariances(params)
    chol = np.linalg.cholesky(S)
    y = np.zeros((N, F, params.order), dtype=complex)
    for j in range(J):
        z = (rng.standard_normal((N, F, params.order)) + 1j * rng.standard_normal((N, F, params.order))) / np.sqrt(2)
        y += np.sqrt(params.v[j])[..., None] * np.einsum("fab,nfb->nfa", chol[j], z)
    return ObservationTensor(y.transpose(2, 0, 1))


def _rand_params(rng, J, N, F, I):
    P = rng.standard_normal((F, I, I)) + 1j * rng.standard_normal((F, I, I)) + 2.0 * np.eye(I)
    return fastfca.FastFcaParams(P, rng.uniform(0.5, 1.5, (J, F, I)), rng.uniform(0.5, 1.5, (J, N, F)))


def test_em_substep_monotone_and_likelihood_improves(rng):
    # test_fastfca.py:369-386 and acceptance criterion 3
    truth = _rand_params(rng, 3, 48, 4, 3)
    obs = _model_observation(rng, truth)
    init = _rand_params(rng, 3, 48, 4, 3)
    run = fastfca.run_fastfca(obs, init, iterations=15, record_likelihood=True)
    before = [run.loglik_init] + run.loglik_after_p[:-1]
    for prev, new in zip(before, run.loglik_after_em):
        assert new >= prev - 1e-6 * abs(prev)
    assert run.loglik_after_p[-1] > run.loglik_init


def test_fixed_point_stationarity_after_convergence():
    # acceptance criterion 7 (test_acceptance.py:255-295): after 150 iterations
    # one more fixed-point update moves the columns of P by <= 1e-6
    r = np.random.default_rng(77)
    I, J, N, F = 3, 1, 512, 4
    P_true = r.standard_normal((F, I, I)) + 1j * r.standard_normal((F, I, I)) + 2 * np.eye(I)
    truth = fastfca.FastFcaParams(P_true, r.uniform(0.5, 3.0, (J, F, I)), r.uniform(0.3, 3.0, (J, N, F)))
    obs = _model_observation(r, truth)
    init = fastfca.FastFcaParams(P_true + 0.2 * (r.standard_normal(P_true.shape) + 1j * r.standard_normal(P_true.shape)),
                                 truth.Lam * r.uniform(0.7, 1.4, truth.Lam.shape),
                                 truth.v * r.uniform(0.7, 1.4, truth.v.shape))
    run = fastfca.run_fastfca(obs, init, iterations=150)
    upd = fastfca.fixed_point_update_P(run.params, obs)
    resid = (np.linalg.norm(upd - run.params.P, axis=1) / np.linalg.norm(run.params.P, axis=1)).max()
    assert resid <= 1e-6


def test_counters_match_paper_at_benchmark_size():
    # acceptance criterion 1: I=3, F=512 -> exactly 2048 inversions per iteration, 0 matmuls
    y, P0, lam0, v0, _ = mixture(1, 3, 3, 512, 8)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=1)
    assert run.counters.inversions == 2048 and run.counters.matmuls == 0


def test_sharded_driver_device_path_world1():
    # the multi-GPU driver's device compute path (gloo world of 1 on this box)
    import socket

    import torch.distributed as dist

    from paper_1805_09498_b200.multigpu import run_fastfca_sharded
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        parts = [mixture(300 + u, 3, 3, 11, 40) for u in range(2)]
        y, P0, lam0, v0 = (np.stack([p[k] for p in parts]) for k in range(4))
        for mode in ("mixtures", "bins"):
            P, lam, v, ll = run_fastfca_sharded(y, P0, lam0, v0, iterations=3, mode=mode, record_likelihood=True)
            Pr, lr, vr, llr = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=3, record_likelihood=True)
            assert np.array_equal(P, Pr) and np.array_equal(v, vr) and np.allclose(ll, llr, rtol=1e-14)
    finally:
        dist.destroy_process_group()


def _stack(seeds, I, J, F, N, rank=4):
    parts = [mixture(s, I, J, F, N, rank) for s in seeds]
    return tuple(np.stack([p[k] for p in parts]) for k in range(4))


def _plan(dt_code, U, I, J, N, F):
    out = np.zeros(6, np.int32)
    _lib.load().ffca_plan_loop(0, dt_code, U, I, J, N, F, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip))
    return out


def test_c128_results_do_not_depend_on_batch_size():
    # config-0 shape, complex128: the default plan runs one-bin CTAs at every batch size; the
    # 2-bin CTAs (forced here for the batch) must give bitwise the same bins -- the one-bin plan
    # reduces over 16-lane segments exactly like them (the plans used to differ)
    cfg = CONFIGS[0]
    args = _stack(range(500, 504), cfg.I, cfg.J, cfg.F, cfg.N)
    assert _plan(_lib.C128, 1, 3, 3, cfg.N, cfg.F)[0] == 1
    assert _plan(_lib.C128, 4, 3, 3, cfg.N, cfg.F)[0] == 1
    os.environ["FFCA_NO_PIPELINE"] = "1"
    try:
        os.environ["FFCA_FORCE_PLAN"] = "2,1,1"
        try:
            batch = fastfca.run_fastfca_batch(*args, iterations=5, record_likelihood=True)
        finally:
            os.environ.pop("FFCA_FORCE_PLAN")
        for u in (0, 3):
            one = fastfca.run_fastfca_batch(*(a[u:u + 1] for a in args), iterations=5, record_likelihood=True)
            for a, b in zip(one, batch):
                assert np.array_equal(a[0], b[u])
    finally:
        os.environ.pop("FFCA_NO_PIPELINE")


def test_c128_pipelined_chunks_bitwise_one_launch():
    # 3 config-0 mixtures (69 MB) take the host pipeline in chunks of 2 + 1 mixtures: bitwise one launch
    cfg = CONFIGS[0]
    args = _stack(range(510, 513), cfg.I, cfg.J, cfg.F, cfg.N)
    os.environ["FFCA_NO_PIPELINE"] = "1"
    try:
        ref = fastfca.run_fastfca_batch(*args, iterations=4, record_likelihood=True)
    finally:
        os.environ.pop("FFCA_NO_PIPELINE")
    got = fastfca.run_fastfca_batch(*args, iterations=4, record_likelihood=True)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_batch_coerces_mixed_precision_inputs():
    # complex128 y with complex64 / float32 state: the state is promoted to y's precision, and
    # the result equals the all-complex128 call (no host-buffer overrun)
    y, P0, lam0, v0 = _stack(range(520, 522), 3, 3, 9, 40)
    ref = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=3)
    got = fastfca.run_fastfca_batch(y, P0.astype(np.complex64), lam0.astype(np.float32),
                                    v0.astype(np.float32), iterations=3)
    assert got[0].dtype == np.complex128 and got[2].dtype == np.float64
    ref32 = fastfca.run_fastfca_batch(y, P0, lam0, v0.astype(np.float32).astype(np.float64), iterations=3)
    for a, b in zip(got[:3], ref32[:3]):
        assert np.array_equal(a, b)
    assert rel(got[0], ref[0]) <= 1e-4


@pytest.mark.parametrize("shape,dt,plan", [
    ((3, 3, 40, 41), "c64", None),        # frame pairs with a half-filled last pair
    ((3, 3, 40, 41), "c64", "1,2,1"),     # pairs split over a CTA pair (DSMEM partials, parity buffers)
    ((4, 4, 9, 700), "c64", "1,4,1"),     # cluster of 4
    ((3, 3, 300, 30), "c128", None),      # one-bin CTAs, 16-lane segments
    ((8, 6, 3, 160), "c64", "1,2,1,256"), # I > 4 CTA pair, P^-1 warp concurrent with phase B
])
def test_repeated_runs_bitwise_race_canary(shape, dt, plan):
    # compute-sanitizer is closed on the GPU pool (profiles/r2_sanitizer_refused.log), so shared-memory
    # and DSMEM races are probed by repetition: any race between the reductions, the solver
    # publication and the next phase would show up as run-to-run differences
    I, J, F, N = shape
    y, P0, lam0, v0, _ = mixture(61, I, J, F, N, 4, 0.05 if I > 4 else 0.0)
    y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
    if plan:
        os.environ["FFCA_FORCE_PLAN"] = plan
    first = fastfca.run_fastfca_batch(y[None], P0[None], lam0[None], v0[None], iterations=6, record_likelihood=True)
    for _ in range(8):
        again = fastfca.run_fastfca_batch(y[None], P0[None], lam0[None], v0[None], iterations=6,
                                          record_likelihood=True)
        for a, b in zip(first, again):
            assert np.array_equal(a, b)


def test_loading_retry_is_per_bin_documented_divergence(monkeypatch):
    # when one bin's B_i is exactly singular, the reference's batched
    # numpy inverse fails for the whole (F, I, I) stack and retries EVERY bin with the 1e-10 tr(B)
    # loading (fastfca.py:184-194); the device retries the failing bin only.  Pin both halves: the
    # device equals a per-bin-retry restatement, and differs from the whole-batch one only in the
    # bins that did not need loading, by the loading's size.
    y, P0, lam0, v0, _ = mixture(14, 3, 2, 5, 40)
    y[2, :, 1] = 0.0  # channel 2 silent in bin 1: B_i(f=1) has an exactly zero row / column
    run = fastfca.run_fastfca_batch(y[None], P0[None], lam0[None], v0[None], iterations=1)
    whole = ffr.run_fastfca(y, P0, lam0, v0, iterations=1, stats=False)

    def per_bin(B):
        out = np.empty_like(B)
        for f in range(B.shape[0]):
            try:
                out[f] = np.linalg.inv(B[f])
            except np.linalg.LinAlgError:
                tr = np.real(np.trace(B[f]))
                out[f] = np.linalg.inv(B[f] + ffr.B_REGULARIZATION * tr * np.eye(B.shape[-1]))
        return out

    monkeypatch.setattr(ffr, "_inv_loaded", per_bin)
    local = ffr.run_fastfca(y, P0, lam0, v0, iterations=1, stats=False)
    P = run[0][0]
    assert rel(P, local.P) <= 1e-10  # the device's per-bin semantics
    assert rel(P[1], whole.P[1]) <= 1e-10  # the singular bin: loaded in both
    others = [0, 2, 3, 4]
    d = np.abs(P[others] - whole.P[others]).max() / np.abs(whole.P[others]).max()
    assert 0.0 < d <= 1e-8  # the whole-batch retry also loaded the healthy bins (by ~1e-10 tr)


@pytest.mark.parametrize("dt,shape", [("c64", (3, 3, 40, 90)), ("c128", (3, 3, 40, 90)), ("c64", (4, 4, 6, 700)),
                                      ("c64", (8, 6, 3, 160))])
def test_lean_instantiation_matches_general(dt, shape):
    # the plain loop runs lean (FAST) instantiations with the likelihood / floor-array / P-only paths
    # compiled out.  They are separate compilations of the same arithmetic, so nvcc may contract a
    # different a*b + c*d into an FMA: the state agrees with the general kernel (FFCA_NO_FAST=1, or a
    # call that records the likelihood) to rounding, not necessarily bitwise
    I, J, F, N = shape
    y, P0, lam0, v0, _ = mixture(91, I, J, F, N, 4, 0.05 if I > 4 else 0.0)
    y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
    args = (y[None], P0[None], lam0[None], v0[None])
    fast = fastfca.run_fastfca_batch(*args, iterations=5)
    rec = fastfca.run_fastfca_batch(*args, iterations=5, record_likelihood=True)
    os.environ["FFCA_NO_FAST"] = "1"
    try:
        general = fastfca.run_fastfca_batch(*args, iterations=5)
    finally:
        os.environ.pop("FFCA_NO_FAST")
    tol = 1e-12 if dt == "c128" else 1e-5
    for a, b, c in zip(fast[:3], rec[:3], general[:3]):
        assert rel(a, c) <= tol and rel(b, c) <= tol


def test_c128_lean_results_do_not_depend_on_batch_size():
    # the bitwise batch-size independence of the complex128 plans also holds for the lean kernels
    cfg = CONFIGS[0]
    args = _stack(range(540, 544), cfg.I, cfg.J, cfg.F, cfg.N)
    os.environ["FFCA_NO_PIPELINE"] = "1"
    try:
        batch = fastfca.run_fastfca_batch(*args, iterations=5)
        one = fastfca.run_fastfca_batch(*(a[2:3] for a in args), iterations=5)
    finally:
        os.environ.pop("FFCA_NO_PIPELINE")
    for a, b in zip(one[:3], batch[:3]):
        assert np.array_equal(a[0], b[2])
