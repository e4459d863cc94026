"""GPU STFT filterbank (the caller of the estimation path) vs the reference golden vectors."""

import numpy as np
import pytest

from conftest import rel
from oracle import stft_ref
from paper_1805_09498_b200 import errors
from paper_1805_09498_b200.stft import ObservationTensor, StftConfig, analyze, interior_slice, synthesize

pytestmark = pytest.mark.gpu


def case(golden):
    return {k.split("/", 1)[1]: v for k, v in golden.items() if k.startswith("stft/")}


def test_analyze_synthesize_golden(golden):
    g = case(golden)
    obs = analyze(g["audio"])
    assert obs.data.shape == g["obs"].shape and obs.data.dtype == np.complex128
    assert rel(obs.data, g["obs"]) <= 1e-12
    assert rel(synthesize(obs), g["resynth"]) <= 1e-12
    assert rel(analyze(g["audio"][:, :2048], StftConfig(256, 128)).data, g["small_obs"]) <= 1e-12


def test_round_trip_acceptance_6():
    # acceptance criterion 6 (test_acceptance.py:241-252): interior relative RMS <= 1e-10
    rng = np.random.default_rng(5150)
    audio = rng.standard_normal((3, 8 * 16000))
    cfg = StftConfig()
    rebuilt = synthesize(analyze(audio, cfg), cfg)
    sl = interior_slice(min(audio.shape[1], rebuilt.shape[1]), cfg)
    err = np.sqrt(np.mean((rebuilt[:, sl] - audio[:, sl]) ** 2)) / np.sqrt(np.mean(audio[:, sl] ** 2))
    assert err <= 1e-10


def test_float32_path_and_shapes():
    rng = np.random.default_rng(1)
    audio = rng.standard_normal((2, 5000)).astype(np.float32)
    obs = analyze(audio)
    assert obs.data.dtype == np.complex64 and obs.data.shape == (2, (5000 - 1024) // 512 + 1, 512)
    ref = stft_ref.analyze(audio.astype(np.float64))
    assert rel(obs.data, ref) <= 1e-5
    back = synthesize(obs)
    assert back.dtype == np.float32
    assert rel(back, stft_ref.synthesize(ref)) <= 1e-5


def test_errors():
    with pytest.raises(errors.TooShort):
        analyze(np.zeros((2, 100)))
    with pytest.raises(errors.ChannelLengthMismatch):
        analyze([np.zeros(2048), np.zeros(2049)])
    with pytest.raises(errors.DimensionMismatch):
        analyze(np.zeros((2, 2, 2048)))
    with pytest.raises(errors.DimensionMismatch):
        synthesize(ObservationTensor(np.zeros((1, 3, 100), complex)))
    with pytest.raises(ValueError):
        StftConfig(1024, 256)
