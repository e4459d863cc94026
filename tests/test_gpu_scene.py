"""GPU initialisers (scene.oracle_covariances / diffuse_covariances, scene.py:195-271)
vs the reference golden vectors and the CPU oracle; edge cases follow test_scene.py:130-201."""

import numpy as np
import pytest

from conftest import rel
from oracle import fastfca_ref as ffr
from oracle import fca_ref, scene_ref
from paper_1805_09498_b200 import _lib, errors, fastfca, fca, scene
from paper_1805_09498_b200.stft import ObservationTensor, StftConfig, analyze

pytestmark = pytest.mark.gpu


def case(golden):
    return {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("scene/")}


def test_oracle_covariances_golden(golden):
    g = case(golden)
    S, v = scene.oracle_covariances(g["refs"], ObservationTensor(g["y"]))
    assert S.shape == g["oracle_S"].shape and v.shape == g["oracle_v"].shape
    assert rel(S, g["oracle_S"]) <= 1e-12 and rel(v, g["oracle_v"]) <= 1e-14
    # silent bin -> identity (trace 0 -> loading 1.0), silent source in a live bin -> identity too
    assert np.array_equal(S[:, 2], np.broadcast_to(np.eye(3), S[:, 2].shape))
    assert np.array_equal(S[1, 5], np.eye(3))
    assert np.array_equal(v, g["oracle_v"]) or rel(v, g["oracle_v"]) <= 1e-15
    assert _lib.load().ffca_last_launch_count() >= 1


@pytest.mark.parametrize("J,seed", [(2, 7), (3, 8)])
def test_diffuse_covariances_golden(golden, J, seed):
    g = case(golden)
    S, v = scene.diffuse_covariances(ObservationTensor(g["y"]), J, seed)
    assert rel(S, g[f"diffuse{J}_S"]) <= 1e-12 and rel(v, g[f"diffuse{J}_v"]) <= 1e-14


def test_complex64_inputs():
    rng = np.random.default_rng(3)
    J, I, N, F = 3, 4, 200, 33
    refs = rng.standard_normal((J, I, N, F)) + 1j * rng.standard_normal((J, I, N, F))
    y = refs.sum(axis=0)
    S_ref, v_ref = scene_ref.oracle_covariances(refs, y)
    S, v = scene.oracle_covariances(refs.astype(np.complex64), ObservationTensor(y.astype(np.complex64)))
    assert S.dtype == np.complex64 and v.dtype == np.float32
    assert rel(S, S_ref) <= 2e-6 and rel(v, v_ref) <= 2e-6
    S, v = scene.diffuse_covariances(ObservationTensor(y.astype(np.complex64)), J, 11)
    S_ref, v_ref = scene_ref.diffuse_covariances(y, J, 11)
    assert rel(S, S_ref) <= 2e-6 and rel(v, v_ref) <= 2e-6


@pytest.mark.parametrize("I,J", [(1, 2), (2, 2), (3, 3), (4, 4), (6, 8), (8, 6)])
def test_against_oracle_all_orders(I, J):
    rng = np.random.default_rng(100 + I * 10 + J)
    N, F = 150, 17
    refs = (rng.standard_normal((J, I, N, F)) + 1j * rng.standard_normal((J, I, N, F))) * \
        rng.uniform(0.01, 10.0, (J, 1, N, F))
    y = refs.sum(axis=0)
    obs = ObservationTensor(y)
    S, v = scene.oracle_covariances(refs, obs)
    S_ref, v_ref = scene_ref.oracle_covariances(refs, y)
    assert rel(S, S_ref) <= 1e-12 and rel(v, v_ref) <= 1e-14
    S, v = scene.diffuse_covariances(obs, J, 5)
    S_ref, v_ref = scene_ref.diffuse_covariances(y, J, 5)
    assert rel(S, S_ref) <= 1e-12 and rel(v, v_ref) <= 1e-14
    np.linalg.cholesky(S)  # PD


def test_diffuse_deterministic_and_seeded():
    # test_scene.py:178-188
    rng = np.random.default_rng(21)
    y = rng.standard_normal((3, 60, 20)) + 1j * rng.standard_normal((3, 60, 20))
    obs = ObservationTensor(y)
    a = scene.init_diffuse(obs, 2, seed=7, algorithm="fca")
    b = scene.init_diffuse(obs, 2, seed=7, algorithm="fca")
    assert np.array_equal(a.S, b.S) and np.array_equal(a.v, b.v)
    np.linalg.cholesky(a.S)
    c = scene.init_diffuse(obs, 2, seed=8, algorithm="fca")
    assert not np.array_equal(a.S, c.S)


def test_init_oracle_both_algorithms_finite():
    # test_scene.py:163-174: FCA params PD, both likelihoods finite
    rng = np.random.default_rng(9)
    cfg = StftConfig(frame_length=256, frame_shift=128)
    images = rng.standard_normal((2, 2, 16000))  # (J, I, S) source images
    mixture = images.sum(axis=0)
    obs = analyze(mixture, cfg)
    refs = scene.reference_tensors(images, cfg)
    assert refs.shape == (2,) + obs.data.shape
    p = scene.init_oracle(refs, obs, "fca")
    np.linalg.cholesky(p.S)
    assert np.isfinite(fca.log_likelihood(p, obs))
    f = scene.init_oracle(refs, obs, "fastfca")
    assert np.isfinite(fastfca.log_likelihood(f, obs))
    with pytest.raises(ValueError):
        scene.init_oracle(refs, obs, "nope")


def test_fca_monotone_from_diffuse_init():
    # test_scene.py:191-200
    rng = np.random.default_rng(33)
    cfg = StftConfig(frame_length=256, frame_shift=128)
    obs = analyze(rng.standard_normal((2, 12800)), cfg)
    init = scene.init_diffuse(obs, 2, seed=3, algorithm="fca")
    run = fca.run_fca(obs, init, iterations=10, record_likelihood=True)
    hist = np.array(run.loglik)
    assert (np.diff(hist) >= -1e-6 * np.abs(hist[:-1])).all()
    # and the oracle FCA from the same start agrees
    ref = fca_ref.run_fca(obs.data, init.S, init.v, iterations=10)
    assert rel(run.params.S, ref.S) <= 1e-8


def test_errors():
    y = np.ones((2, 10, 4), complex)
    with pytest.raises(errors.DimensionMismatch):
        scene.oracle_covariances(np.ones((2, 2, 10, 5), complex), ObservationTensor(y))
    with pytest.raises(errors.DimensionMismatch):
        scene.diffuse_covariances(ObservationTensor(y), 0, 1)


def test_matches_oracle_whitening_chain():
    # init_oracle(..., "fastfca") == params_from_covariances(oracle S_hat)
    rng = np.random.default_rng(77)
    J, I, N, F = 3, 3, 80, 12
    refs = rng.standard_normal((J, I, N, F)) + 1j * rng.standard_normal((J, I, N, F))
    y = refs.sum(axis=0)
    p = scene.init_oracle(refs, ObservationTensor(y), "fastfca")
    S_ref, v_ref = scene_ref.oracle_covariances(refs, y)
    P_ref, lam_ref, _ = ffr.params_from_covariances(S_ref, v_ref)
    assert rel(p.P, P_ref) <= 1e-11 and rel(p.Lam, lam_ref) <= 1e-11 and rel(p.v, v_ref) <= 1e-14
