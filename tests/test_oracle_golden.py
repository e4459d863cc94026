"""Pin the CPU oracle against golden vectors produced by the unmodified reference.

CPU-only (no GPU marker).  The oracle must reproduce the reference to within
re-ordered fp64 rounding before anything is checked against it.
"""

import numpy as np
import pytest

from conftest import rel
from oracle import fastfca_ref as ffr
from oracle import fca_ref, pipeline_ref, scene_ref, stft_ref

CASES = ["g33", "g44", "g86", "g22", "g12", "g23"]


@pytest.mark.parametrize("key", CASES)
def test_fused_loop_matches_reference(golden, key):
    g = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith(key + "/")}
    run = ffr.run_fastfca(g["y"], g["P0"], g["lam0"], g["v0"], iterations=int(g["iters"]),
                          record_likelihood=True)
    assert rel(run.P, g["P"]) <= 1e-12
    assert rel(run.lam, g["lam"]) <= 1e-12
    assert rel(run.v, g["v"]) <= 1e-12
    assert rel(run.mu, g["mu"]) <= 1e-12
    assert rel(run.phi, g["phi"]) <= 1e-12
    assert run.inversions == int(g["inversions"])
    ll = np.array([run.loglik_init] + run.loglik_after_em + run.loglik_after_p)
    assert np.abs(ll - g["ll"]).max() <= 1e-12 * np.abs(g["ll"]).max()
    assert rel(ffr.images(run.P, run.mu), g["images"]) <= 1e-12
    assert rel(ffr.power_floor(g["y"]), g["vfloor"]) <= 1e-14


def test_inner_iterations_and_scalar_floor(golden):
    g = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("k2/")}
    run = ffr.run_fastfca(g["y"], g["P0"], g["lam0"], g["v0"], iterations=3, inner_iterations=2,
                          v_floor=0.0, stats=False)
    assert rel(run.P, g["P"]) <= 1e-12
    assert rel(run.lam, g["lam"]) <= 1e-12
    assert rel(run.v, g["v"]) <= 1e-12
    assert run.inversions == int(g["inversions"])


def test_unfused_steps(golden):
    g = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("step/")}
    y, P, lam, v = g["y"], g["P"], g["lam"], g["v"]
    yt = ffr.transform(P, y)
    assert rel(yt, g["yt"]) <= 1e-14
    assert rel(ffr.weights(v, lam), g["w"]) <= 1e-14
    mu, phi = ffr.e_step_diag(P, lam, v, yt)
    assert rel(mu, g["mu"]) <= 1e-13 and rel(phi, g["phi"]) <= 1e-13
    v_em, lam_em = ffr.m_step_diag(mu, phi, lam, 0.05)
    assert rel(v_em, g["v_em"]) <= 1e-13 and rel(lam_em, g["lam_em"]) <= 1e-13
    Pn, cnt = ffr.fixed_point_update_P(P, lam_em, v_em, y, inner_iterations=2)
    assert rel(Pn, g["P_new"]) <= 1e-12
    assert cnt == (3 + 1) * 5 * 2
    assert abs(ffr.log_likelihood(P, lam, v, y) - float(g["ll"])) <= 1e-12 * abs(float(g["ll"]))
    assert rel(ffr.back_transform_means(P, mu), g["back"]) <= 1e-12
    assert rel(ffr.reconstruct_spatial_covariances(P, lam), g["S"]) <= 1e-12
    one = ffr.run_fastfca(y, P, lam, v, iterations=1, v_floor=0.0, stats=False)
    assert rel(one.P, g["one_iter_P"]) <= 1e-12


def test_back_transform_stats_and_init(golden):
    g = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("step/")}
    mu, phi = ffr.e_step_diag(g["P"], g["lam"], g["v"], ffr.transform(g["P"], g["y"]))
    bmu, bphi = ffr.back_transform_stats(g["P"], mu, phi)
    assert rel(bmu, g["bt_mu"]) <= 1e-12 and rel(bphi, g["bt_phi"]) <= 1e-12
    assert rel(ffr.reconstruct_spatial_covariances(g["P"], g["lam"])[1, 2], g["S01"]) <= 1e-12
    h = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("init/")}
    P, lam, _ = ffr.params_from_covariances(h["S_hat"], h["v_hat"])
    assert rel(P, h["P"]) <= 1e-12 and rel(lam, h["Lam"]) <= 1e-12


def test_fca_baseline(golden):
    g = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("fca/")}
    run = fca_ref.run_fca(g["y"], g["S0"], g["v0"], iterations=int(g["iters"]), record_likelihood=True)
    assert rel(run.S, g["S"]) <= 1e-12
    assert rel(run.v, g["v"]) <= 1e-12
    assert rel(run.mu, g["mu"]) <= 1e-12
    assert rel(run.phi, g["phi"]) <= 1e-12
    assert np.abs(np.array(run.loglik) - g["ll"]).max() <= 1e-12 * np.abs(g["ll"]).max()
    assert run.inversions == int(g["inversions"]) and run.matmuls == int(g["matmuls"])
    mu, phi = fca_ref.e_step(g["S0"], g["v0"], g["y"])
    assert rel(mu, g["e_mu"]) <= 1e-13 and rel(phi, g["e_phi"]) <= 1e-13
    S, v = fca_ref.m_step(mu, phi, g["S0"], ffr.power_floor(g["y"]))
    assert rel(S, g["m_S"]) <= 1e-13 and rel(v, g["m_v"]) <= 1e-13
    mu_f, _ = fca_ref.e_step(run.S, run.v, g["y"])
    assert rel(np.transpose(mu_f, (0, 3, 1, 2)), g["images"]) <= 1e-12


def test_oracle_singular_P_raises():
    y = np.ones((2, 3, 2), complex)
    P = np.zeros((2, 2, 2), complex)
    with pytest.raises(ffr.OracleSingular):
        ffr.run_fastfca(y, P, np.ones((1, 2, 2)), np.ones((1, 3, 2)), iterations=1)


def test_stft_oracle_matches_reference(golden):
    g = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("stft/")}
    obs = stft_ref.analyze(g["audio"])
    assert rel(obs, g["obs"]) <= 1e-13
    assert rel(stft_ref.synthesize(obs), g["resynth"]) <= 1e-13
    assert rel(stft_ref.analyze(g["audio"][:, :2048], 256, 128), g["small_obs"]) <= 1e-13


def test_scene_initialisers_match_reference(golden):
    g = {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("scene/")}
    S, v = scene_ref.oracle_covariances(g["refs"], g["y"])
    assert rel(S, g["oracle_S"]) <= 1e-13 and rel(v, g["oracle_v"]) <= 1e-14
    # the silent bin falls back to identity loading, exactly as the reference
    assert np.array_equal(S[:, 2], np.broadcast_to(np.eye(3), S[:, 2].shape))
    for J, seed in ((2, 7), (3, 8)):
        S, v = scene_ref.diffuse_covariances(g["y"], J, seed)
        assert rel(S, g[f"diffuse{J}_S"]) <= 1e-13 and rel(v, g[f"diffuse{J}_v"]) <= 1e-14


@pytest.mark.parametrize("algo", ["fastfca", "fca"])
@pytest.mark.parametrize("init", ["oracle", "diffuse"])
def test_pipeline_oracle_matches_reference(golden, algo, init):
    # cli.separate_once on a synthetic scene (scene.synth_mixture, seed 9), 5 iterations
    audio, sdrs, _ = pipeline_ref.separate_once(golden["pipe/mixture"], golden["pipe/references"], algo, init,
                                                sources=2, iterations=5, seed=4, L=256, shift=128)
    assert rel(audio, golden[f"pipe/{algo}_{init}_audio"]) <= 1e-13
    assert np.allclose(sdrs, golden[f"pipe/{algo}_{init}_sdr"], rtol=0, atol=1e-10)


def test_scene_generator_matches_reference(golden):
    mix, refs = scene_ref.synth_mixture(n_sources=2, n_channels=3, duration=0.25, seed=5)
    assert rel(mix, golden["scenegen/mixture"]) <= 1e-13
    assert rel(refs, golden["scenegen/references"]) <= 1e-13
