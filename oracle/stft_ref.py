"""numpy restatement of the STFT filterbank (checker only).  stft.py:96-134.

sqrt-Hann analysis/synthesis pair at 50% overlap; F = L/2 bins with the DC
and Nyquist coefficients packed into bin 0 (stft.py:7-13).
"""

from __future__ import annotations

import numpy as np


def window(L: int) -> np.ndarray:
    return np.sin(np.pi * np.arange(L) / L)


def analyze(audio: np.ndarray, L: int = 1024, shift: int = 512) -> np.ndarray:
    """(I, S) -> (I, N, L/2) complex, N = (S - L) // shift + 1.  stft.py:96-112."""
    audio = np.atleast_2d(np.asarray(audio, dtype=np.float64))
    N = (audio.shape[1] - L) // shift + 1
    idx = np.arange(N)[:, None] * shift + np.arange(L)[None, :]
    spec = np.fft.rfft(audio[:, idx] * window(L), axis=-1)
    out = spec[..., : L // 2].copy()
    out[..., 0] = spec[..., 0].real + 1j * spec[..., -1].real
    return out


def synthesize(obs: np.ndarray, L: int = 1024, shift: int = 512) -> np.ndarray:
    """(I, N, L/2) -> (I, (N-1)*shift + L) by windowed overlap-add.  stft.py:115-134."""
    I, N, F = obs.shape
    spec = np.zeros((I, N, F + 1), dtype=np.complex128)
    spec[..., :F] = obs
    spec[..., 0] = obs[..., 0].real
    spec[..., F] = obs[..., 0].imag
    frames = np.fft.irfft(spec, n=L, axis=-1) * window(L)
    out = np.zeros((I, (N - 1) * shift + L))
    for n in range(N):
        out[:, n * shift: n * shift + L] += frames[:, n]
    return out
