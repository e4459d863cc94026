"""Generate golden vectors by running the UNMODIFIED reference (fcasep).

Run in the build container, where the read-only reference is mounted:

    python tests/golden/make_golden.py

It imports ``fcasep`` from /root/reference/pkg/src, runs the hot-path entry
points on small seeded inputs and writes ``tests/golden/golden.npz``.  The
fixture is committed; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from fcasep import fastfca, fca, wiener  # noqa: E402
from fcasep.stft import ObservationTensor  # noqa: E402

from paper_1805_09498_b200.workloads import mixture  # noqa: E402


def rand_state(rng, J, N, F, I):
    P = rng.standard_normal((F, I, I)) + 1j * rng.standard_normal((F, I, I)) + 2.0 * np.eye(I)
    lam = rng.uniform(0.5, 1.5, (J, F, I))
    v = rng.uniform(0.5, 1.5, (J, N, F))
    return P, lam, v


def main():
    out = {}

    # --- fused loop on generator mixtures (I, J, F, N, iters, rank, zero_frac, seed)
    cases = {
        "g33": (3, 3, 16, 40, 5, 4, 0.0, 11),
        "g44": (4, 4, 9, 64, 4, 8, 0.0, 12),
        "g86": (8, 6, 5, 48, 3, 8, 0.1, 13),
        "g22": (2, 2, 7, 30, 6, 4, 0.0, 14),
        "g12": (1, 2, 6, 25, 4, 4, 0.0, 15),
        "g23": (2, 3, 5, 33, 3, 4, 0.0, 16),
    }
    for key, (I, J, F, N, it, r, zf, seed) in cases.items():
        y, P0, lam0, v0, _ = mixture(seed, I, J, F, N, r, zf)
        obs = ObservationTensor(y)
        run = fastfca.run_fastfca(obs, fastfca.FastFcaParams(P0, lam0, v0), iterations=it,
                                  record_likelihood=True)
        images = wiener.mmse_images_fastfca(run.params, run.stats).stft
        out[f"{key}/y"] = y
        out[f"{key}/P0"], out[f"{key}/lam0"], out[f"{key}/v0"] = P0, lam0, v0
        out[f"{key}/iters"] = np.array(it)
        out[f"{key}/P"], out[f"{key}/lam"], out[f"{key}/v"] = run.params.P, run.params.Lam, run.params.v
        out[f"{key}/mu"], out[f"{key}/phi"] = run.stats.mu, run.stats.phi
        out[f"{key}/images"] = images
        out[f"{key}/inversions"] = np.array(run.counters.inversions)
        out[f"{key}/ll"] = np.array([run.loglik_init] + run.loglik_after_em + run.loglik_after_p)
        out[f"{key}/vfloor"] = fca.power_floor(obs)

    # --- K = 2 inner iterations, scalar v_floor
    I, J, F, N = 3, 2, 6, 20
    rng = np.random.default_rng(7)
    P, lam, v = rand_state(rng, J, N, F, I)
    y = rng.standard_normal((I, N, F)) + 1j * rng.standard_normal((I, N, F))
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P, lam, v), iterations=3,
                              inner_iterations=2, v_floor=0.0)
    out.update({"k2/y": y, "k2/P0": P, "k2/lam0": lam, "k2/v0": v, "k2/P": run.params.P,
                "k2/lam": run.params.Lam, "k2/v": run.params.v,
                "k2/inversions": np.array(run.counters.inversions)})

    # --- unfused step functions on a random state (test_fastfca.py style)
    I, J, F, N = 3, 3, 5, 12
    rng = np.random.default_rng(8)
    P, lam, v = rand_state(rng, J, N, F, I)
    y = rng.standard_normal((I, N, F)) + 1j * rng.standard_normal((I, N, F))
    obs = ObservationTensor(y)
    params = fastfca.FastFcaParams(P, lam, v)
    yt = fastfca.transform_observations(P, obs)
    st = fastfca.e_step_diag(params, yt)
    em = fastfca.m_step_diag(st, params, v_floor=0.05)
    Pn = fastfca.fixed_point_update_P(em, obs, inner_iterations=2)
    out.update({
        "step/y": y, "step/P": P, "step/lam": lam, "step/v": v,
        "step/yt": yt, "step/w": fastfca.mixture_weights(params),
        "step/mu": st.mu, "step/phi": st.phi,
        "step/v_em": em.v, "step/lam_em": em.Lam, "step/P_new": Pn,
        "step/ll": np.array(fastfca.log_likelihood(params, obs)),
        "step/back": fastfca.back_transform_means(P, st.mu),
        "step/S": fastfca.reconstruct_spatial_covariances(params),
        "step/one_iter_P": fastfca.run_fastfca(obs, params, iterations=1, v_floor=0.0).params.P,
    })

    # --- back-transformed stats, reconstruction, whitening init
    mu_b, phi_b = fastfca.back_transform_stats(params, st)
    rngw = np.random.default_rng(9)
    a = rngw.standard_normal((3, 5, 3, 3)) + 1j * rngw.standard_normal((3, 5, 3, 3))
    S_hat = a @ np.conj(np.swapaxes(a, -1, -2)) + np.eye(3)
    S_hat = 0.5 * (S_hat + np.conj(np.swapaxes(S_hat, -1, -2)))
    v_hat = rngw.uniform(0.5, 2.0, (3, 7, 5))
    init = fastfca.params_from_covariances(S_hat, v_hat)
    out.update({
        "init/S_hat": S_hat, "init/v_hat": v_hat, "init/P": init.P, "init/Lam": init.Lam,
        "step/bt_mu": mu_b, "step/bt_phi": phi_b,
        "step/S01": fastfca.reconstruct_spatial_covariance(params, 1, 2),
    })

    # --- STFT filterbank (the caller of the path)
    from fcasep.stft import StftConfig, analyze, synthesize
    rngs = np.random.default_rng(10)
    audio = rngs.standard_normal((2, 6 * 1024 + 300))
    cfg = StftConfig()
    tens = analyze(audio, cfg)
    out.update({"stft/audio": audio, "stft/obs": tens.data, "stft/resynth": synthesize(tens, cfg),
                "stft/small_obs": analyze(audio[:, :2048], StftConfig(256, 128)).data})

    # --- conventional FCA
    I, J, F, N = 3, 3, 6, 24
    y, P0, lam0, v0, _ = mixture(21, I, J, F, N)
    obs = ObservationTensor(y)
    S0 = np.broadcast_to(np.eye(I, dtype=complex), (J, F, I, I)).copy()
    rf = fca.run_fca(obs, fca.FcaParams(S0, v0), iterations=4, record_likelihood=True)
    e = fca.e_step(fca.FcaParams(S0, v0), obs)
    m = fca.m_step(e, fca.FcaParams(S0, v0), fca.power_floor(obs))
    out.update({
        "fca/y": y, "fca/S0": S0, "fca/v0": v0, "fca/iters": np.array(4),
        "fca/S": rf.params.S, "fca/v": rf.params.v, "fca/mu": rf.stats.mu, "fca/phi": rf.stats.phi,
        "fca/ll": np.array(rf.loglik), "fca/inversions": np.array(rf.counters.inversions),
        "fca/matmuls": np.array(rf.counters.matmuls),
        "fca/e_mu": e.mu, "fca/e_phi": e.phi, "fca/m_S": m.S, "fca/m_v": m.v,
        "fca/images": wiener.mmse_images_fca(rf.params, obs).stft,
    })

    # --- initialisers (scene.oracle_covariances / diffuse_covariances), with degenerate bins
    from fcasep import scene
    rngi = np.random.default_rng(31)
    J, I, N, F = 2, 3, 40, 9
    refs = (rngi.standard_normal((J, I, N, F)) + 1j * rngi.standard_normal((J, I, N, F))) * \
        rngi.uniform(0.1, 3.0, (J, 1, N, F))
    refs[:, :, :, 2] = 0.0          # silent bin: floor 1e-300, identity loading
    refs[1, :, :, 5] = 0.0          # one silent source in a live bin
    refs[0, :, 7, :] = 0.0          # a silent frame
    obs_i = ObservationTensor(refs.sum(axis=0))
    So, vo = scene.oracle_covariances(refs, obs_i)
    Sd2, vd2 = scene.diffuse_covariances(obs_i, 2, 7)
    Sd3, vd3 = scene.diffuse_covariances(obs_i, 3, 8)
    out.update({
        "scene/refs": refs, "scene/y": obs_i.data, "scene/oracle_S": So, "scene/oracle_v": vo,
        "scene/diffuse2_S": Sd2, "scene/diffuse2_v": vd2, "scene/diffuse3_S": Sd3, "scene/diffuse3_v": vd3,
    })

    # --- the whole in-memory pipeline (cli.separate_once): synthetic scene -> separated audio
    from fcasep import cli
    built = scene.synth_mixture(scene.SceneSpec(n_sources=2, n_channels=2, duration=0.4, seed=9))
    out.update({"pipe/mixture": built.mixture, "pipe/references": built.references})
    for algo in ("fastfca", "fca"):
        for init in ("oracle", "diffuse"):
            rc = cli.RunConfig(algorithm=algo, iterations=5, init=init, sources=2, seed=4,
                               frame_length=256, frame_shift=128)
            images, report, _run = cli.separate_once(rc, built.mixture, built.references)
            out[f"pipe/{algo}_{init}_audio"] = images.audio
            out[f"pipe/{algo}_{init}_sdr"] = np.array(report.sdr_per_source)

    # --- synthetic scene generator (scene.synth_mixture), used by the acceptance tests
    sc = scene.synth_mixture(scene.SceneSpec(n_sources=2, n_channels=3, duration=0.25, seed=5))
    out.update({"scenegen/mixture": sc.mixture, "scenegen/references": sc.references})

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
