"""Device-resident separation pipeline (cli.separate_once, cli.py:217-260) vs the reference's
own output on a synthetic scene, plus SDR / resynthesis helpers (evalkit.py:68-93, wiener.py:46-53)."""

import numpy as np
import pytest

from conftest import rel
from oracle import pipeline_ref, stft_ref
from paper_1805_09498_b200 import _lib, errors, evalkit, pipeline, wiener
from paper_1805_09498_b200.stft import StftConfig

pytestmark = pytest.mark.gpu


def cfg(algo, init, **kw):
    return pipeline.PipelineConfig(algorithm=algo, iterations=5, init=init, sources=2, seed=4, frame_length=256,
                                   frame_shift=128, **kw)


@pytest.mark.parametrize("algo", ["fastfca", "fca"])
@pytest.mark.parametrize("init", ["oracle", "diffuse"])
def test_pipeline_matches_reference(golden, algo, init):
    res = pipeline.separate_once(cfg(algo, init), golden["pipe/mixture"], golden["pipe/references"])
    g = golden[f"pipe/{algo}_{init}_audio"]
    assert res.images.audio.shape == g.shape
    assert rel(res.images.audio, g) <= 1e-9
    assert np.allclose(res.sdr_per_source, golden[f"pipe/{algo}_{init}_sdr"], rtol=0, atol=1e-6)
    assert res.estimator_seconds > 0 and res.rtf == res.estimator_seconds / 0.4
    J, I, N, F = res.images.stft.shape
    if algo == "fastfca":
        assert res.counters.inversions == 5 * (I + 1) * F and res.counters.matmuls == 0
    else:
        assert res.counters.inversions == 5 * (J + N) * F and res.counters.matmuls == 5 * 2 * J * N * F


def test_pipeline_complex64(golden):
    res = pipeline.separate_once(cfg("fastfca", "oracle", complex64=True), golden["pipe/mixture"],
                                 golden["pipe/references"])
    assert res.images.audio.dtype == np.float32
    assert rel(res.images.audio, golden["pipe/fastfca_oracle_audio"]) <= 1e-3
    assert np.allclose(res.sdr_per_source, golden["pipe/fastfca_oracle_sdr"], atol=0.05)


def test_pipeline_bitwise_reproducible(golden):
    # the reference's reproducibility test (test_cli.py:109-135): identical inputs -> identical outputs
    a = pipeline.separate_once(cfg("fastfca", "diffuse"), golden["pipe/mixture"], golden["pipe/references"])
    b = pipeline.separate_once(cfg("fastfca", "diffuse"), golden["pipe/mixture"], golden["pipe/references"])
    assert np.array_equal(a.images.audio, b.images.audio) and a.sdr_per_source == b.sdr_per_source


def test_pipeline_larger_scene_against_oracle():
    rng = np.random.default_rng(12)
    refs = rng.standard_normal((3, 3, 24000))
    mix = refs.sum(axis=0)
    c = pipeline.PipelineConfig(iterations=8, init="oracle", sources=3)
    res = pipeline.separate_once(c, mix, refs)
    audio, sdrs, _ = pipeline_ref.separate_once(mix, refs, "fastfca", "oracle", sources=3, iterations=8)
    assert rel(res.images.audio, audio) <= 1e-9
    assert np.allclose(res.sdr_per_source, sdrs, atol=1e-6)


def test_pipeline_errors(golden):
    with pytest.raises(ValueError):
        pipeline.separate_once(cfg("fastfca", "oracle"), golden["pipe/mixture"], None)
    with pytest.raises(errors.TooShort):
        pipeline.separate_once(cfg("fastfca", "diffuse"), np.zeros((2, 100)))
    with pytest.raises(errors.DimensionMismatch):
        pipeline.separate_once(cfg("fastfca", "oracle"), golden["pipe/mixture"], golden["pipe/references"][:, :, :-1])
    with pytest.raises(ValueError):
        pipeline.PipelineConfig(algorithm="nmf")


def test_compute_sdr_and_resynthesis():
    rng = np.random.default_rng(2)
    ref = rng.standard_normal((2, 5000))
    est = ref + 0.1 * rng.standard_normal((2, 5000))
    assert abs(evalkit.compute_sdr(ref, est) - pipeline_ref.compute_sdr(ref, est)) <= 1e-9
    assert evalkit.compute_sdr(ref, ref) == evalkit.SDR_CAP_DB
    with pytest.raises(errors.LengthMismatch):
        evalkit.compute_sdr(ref, est[:, :-1])
    with pytest.raises(errors.ZeroReference):
        evalkit.compute_sdr(np.zeros((2, 10)), est[:, :10])
    stft = rng.standard_normal((2, 3, 20, 128)) + 1j * rng.standard_normal((2, 3, 20, 128))
    out = wiener.resynthesize_images(wiener.SeparatedImages(stft=stft), StftConfig(256, 128))
    want = stft_ref.synthesize(stft.reshape(6, 20, 128), 256, 128).reshape(2, 3, -1)
    assert rel(out.audio, want) <= 1e-12
    assert evalkit.rtf_value(2.0, 8.0) == 0.25
