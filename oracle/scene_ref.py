"""CPU restatement of the reference's initialisers -- TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/fcasep/scene.py:195-247 (``_load_pd``,
``oracle_covariances``, ``diffuse_covariances``) and fca.py:82-89
(``power_floor``).  Arrays are numpy, float64 / complex128; the observation
tensor is the plain (I, N, F) array.  Pinned against the reference's outputs
in tests/golden/golden.npz (``scene/*``, made by tests/golden/make_golden.py).
"""

from __future__ import annotations

import numpy as np

from .fastfca_ref import power_floor

INIT_LOADING = 1e-9  # scene.py:197


def load_pd(S):
    """S + relative diagonal loading; identity loading for trace <= 0.  scene.py:200-204."""
    I = S.shape[-1]
    scale = np.trace(S, axis1=-2, axis2=-1).real / I
    loading = np.where(scale > 0, INIT_LOADING * scale, 1.0)
    return S + loading[..., None, None] * np.eye(I)


def oracle_covariances(refs, y):
    """refs (J, I, N, F), y (I, N, F) -> S_hat (J, F, I, I), v_hat (J, N, F).  scene.py:207-223."""
    I, N = refs.shape[1], refs.shape[2]
    p = (np.abs(refs) ** 2).sum(axis=1) / I  # (J, N, F)
    v_hat = np.maximum(p, power_floor(y))
    S = np.einsum("janf,jbnf,jnf->jfab", refs, refs.conj(), 1.0 / v_hat) / N
    return load_pd(S), v_hat


def perturbations(I, J, seed):
    """Seeded trace-normalised PD matrices W_j in the reference's draw order.  scene.py:232-239."""
    rng = np.random.default_rng(seed)
    W = np.empty((J, I, I), np.complex128)
    for j in range(J):
        A = rng.standard_normal((I, I)) + 1j * rng.standard_normal((I, I))
        Wj = A @ A.conj().T
        W[j] = Wj * (I / np.trace(Wj).real)
    return W


def diffuse_covariances(y, J, seed):
    """y (I, N, F) -> S_hat (J, F, I, I), v_hat (J, N, F).  scene.py:226-247."""
    I, N, F = y.shape
    avg = np.einsum("anf,bnf->fab", y, y.conj()) / N
    scale = np.maximum(np.trace(avg, axis1=-2, axis2=-1).real / I, 1e-300)
    W = perturbations(I, J, seed)
    S = avg[None] + 0.5 * scale[None, :, None, None] * W[:, None]
    power = (np.abs(y) ** 2).sum(axis=0) / I
    v_hat = np.maximum(np.broadcast_to(power / J, (J, N, F)), power_floor(y))
    return load_pd(S), np.ascontiguousarray(v_hat)


# ---------------------------------------------------------------------------
# Synthetic scenes (scene.py:64-189), restated so that the acceptance tests can
# build the reference's benchmark scenes without the reference installed.
# Pinned against scene.synth_mixture output (golden ``scenegen/*``).
# ---------------------------------------------------------------------------
SPEED_OF_SOUND = 343.0  # scene.py:29


def synth_sources(n_sources, duration, sample_rate, rng):
    """Band-shaped nonstationary noise, unit RMS + -50 dB floor, (J, T).  scene.py:64-90."""
    import scipy.signal

    T = int(round(duration * sample_rate))
    nyq = sample_rate / 2.0
    out = np.empty((n_sources, T))
    freqs = np.fft.rfftfreq(T, 1.0 / sample_rate)
    for j in range(n_sources):
        shape = np.full_like(freqs, 0.02)
        for _ in range(3):
            c = rng.uniform(0.05, 0.6) * nyq
            w = rng.uniform(0.02, 0.08) * nyq
            shape += np.exp(-0.5 * ((freqs - c) / w) ** 2)
        carrier = np.fft.irfft(np.fft.rfft(rng.standard_normal(T)) * shape, n=T)
        grain = max(1, int(0.08 * sample_rate))
        steps = rng.rayleigh(1.0, T // grain + 2)
        env = np.repeat(steps, grain)[:T]
        win = np.hanning(2 * grain + 1)
        env = scipy.signal.fftconvolve(env, win / win.sum(), mode="same")
        s = carrier * env
        s = s / np.sqrt(np.mean(s ** 2))
        s += 10 ** (-50 / 20) * rng.standard_normal(T)
        out[j] = s
    return out


def synth_rirs(n_sources, n_channels, sample_rate, rng, rt60_ms=300.0, tail_gain=0.3, base_delay=32,
               mic_spacing=0.05, source_distance=1.5):
    """Direct path + exponentially decaying noise tail, (J, I, L).  scene.py:93-121."""
    rt60 = max(1.0, rt60_ms * 1e-3 * sample_rate)
    L = int(base_delay + 1.5 * rt60) + 8
    rirs = np.zeros((n_sources, n_channels, L))
    mic_x = (np.arange(n_channels) - (n_channels - 1) / 2) * mic_spacing
    angles = np.linspace(-60.0, 60.0, n_sources) + rng.uniform(-10.0, 10.0, n_sources)
    for j in range(n_sources):
        th = np.deg2rad(angles[j])
        src = source_distance * np.array([np.sin(th), np.cos(th)])
        d = np.hypot(src[0] - mic_x, src[1])
        delays = base_delay + np.round((d - d.min()) / SPEED_OF_SOUND * sample_rate)
        gains = d.min() / d
        decay = 10.0 ** (-3.0 * np.arange(L) / rt60)
        for i in range(n_channels):
            k = int(delays[i])
            rirs[j, i, k] = gains[i]
            tail = rng.standard_normal(L - k - 1)
            rirs[j, i, k + 1:] += tail_gain * gains[i] * tail * decay[1:L - k]
    return rirs


def mix_scene(dry, rirs):
    """x_j = rir_j * s_j per channel, truncated; y = sum_j x_j.  scene.py:156-189."""
    import scipy.signal

    J, I, T = rirs.shape[0], rirs.shape[1], dry.shape[1]
    refs = np.empty((J, I, T))
    for j in range(J):
        for i in range(I):
            refs[j, i] = scipy.signal.fftconvolve(dry[j], rirs[j, i])[:T]
    return refs.sum(axis=0), refs


def synth_mixture(n_sources=3, n_channels=3, duration=8.0, sample_rate=16000, seed=0, rt60_ms=300.0,
                  tail_gain=0.3):
    """(mixture (I, T), references (J, I, T)) of scene.synth_mixture(SceneSpec(...)).  scene.py:179-188."""
    rng = np.random.default_rng(seed)
    dry = synth_sources(n_sources, duration, sample_rate, rng)
    rirs = synth_rirs(n_sources, n_channels, sample_rate, rng, rt60_ms, tail_gain)
    return mix_scene(dry, rirs)
