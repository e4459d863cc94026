"""Observation tensor and STFT filterbank (stft.py:32-146) on the B200.

``ObservationTensor`` is the input contract of the hot path.  ``analyze`` /
``synthesize`` are the caller of the path, run on the
device: framing + sqrt-Hann window, cuFFT batched R2C / C2R, the reference's
DC/Nyquist packing into bin 0, deterministic overlap-add.

Dtype policy (documented extension): complex64 data stays complex64 and runs
the fp32 kernels; anything else is coerced to complex128 as the reference
does (stft.py:63).  float32 audio analyses to complex64.  WAV I/O is out of
scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ChannelLengthMismatch, DimensionMismatch, TooShort


def _coerce(data) -> np.ndarray:
    arr = np.asarray(data)
    if arr.dtype == np.complex64:
        return np.ascontiguousarray(arr)
    return np.ascontiguousarray(arr, dtype=np.complex128)


@dataclass(frozen=True)
class StftConfig:
    frame_length: int = 1024
    frame_shift: int = 512
    window: str = "sqrt_hann"
    sample_rate: int = 16000

    def __post_init__(self):
        if self.window != "sqrt_hann":
            raise ValueError(f"unsupported window {self.window!r}")
        if self.frame_length % self.frame_shift != 0:
            raise ValueError("frame_shift must divide frame_length")
        if 2 * self.frame_shift != self.frame_length:
            raise ValueError("sqrt-Hann pair requires frame_shift == frame_length/2")

    @property
    def bins(self) -> int:
        return self.frame_length // 2

    def analysis_window(self) -> np.ndarray:
        t = np.arange(self.frame_length)
        return np.sin(np.pi * t / self.frame_length)


@dataclass
class ObservationTensor:
    """Complex STFT coefficients indexed (channel, frame, bin)."""

    data: np.ndarray  # (I, N, F) complex128 (or complex64)
    check_finite: bool = True

    def __post_init__(self):
        self.data = _coerce(self.data)
        if self.data.ndim != 3:
            raise DimensionMismatch(f"tensor must be (I, N, F), got {self.data.shape}")
        # stft.py:66-67 -- an O(T) host pass; callers that guarantee finiteness
        # (e.g. the benchmark) may skip it with check_finite=False.
        if self.check_finite and not np.isfinite(self.data).all():
            raise ValueError("tensor has non-finite entries")

    @property
    def channels(self) -> int:
        return self.data.shape[0]

    @property
    def frames(self) -> int:
        return self.data.shape[1]

    @property
    def bins(self) -> int:
        return self.data.shape[2]


def _as_channel_matrix(audio) -> np.ndarray:
    if isinstance(audio, (list, tuple)):
        lengths = {len(np.asarray(ch)) for ch in audio}
        if len(lengths) > 1:
            raise ChannelLengthMismatch(f"channel lengths differ: {sorted(lengths)}")
        audio = np.stack([np.asarray(ch) for ch in audio])
    audio = np.asarray(audio)
    if audio.dtype != np.float32:
        audio = audio.astype(np.float64)
    if audio.ndim == 1:
        audio = audio[None, :]
    if audio.ndim != 2:
        raise DimensionMismatch(f"audio must be (channels, samples), got {audio.shape}")
    return np.ascontiguousarray(audio)


def analyze(audio, cfg: StftConfig = StftConfig()) -> ObservationTensor:
    """Multichannel time signal -> observation tensor (I, N, F).  stft.py:96-112."""
    audio = _as_channel_matrix(audio)
    L, shift = cfg.frame_length, cfg.frame_shift
    if audio.shape[1] < L:
        raise TooShort(f"need at least {L} samples, got {audio.shape[1]}")
    lib = _lib.require_gpu()
    c64 = audio.dtype == np.float32
    I, S = audio.shape
    N = (S - L) // shift + 1
    out = np.empty((I, N, cfg.bins), np.complex64 if c64 else np.complex128)
    _lib.check(lib.ffca_stft_analyze(_lib.device(), None, _lib.MEM_HOST, _lib.C64 if c64 else _lib.C128, I, S, L,
                                     shift, _lib.ptr(audio), _lib.ptr(out)), "ffca_stft_analyze")
    return ObservationTensor(out, check_finite=False)


def synthesize(tensor: ObservationTensor, cfg: StftConfig = StftConfig()) -> np.ndarray:
    """Observation tensor -> multichannel signal by windowed overlap-add.  stft.py:115-134."""
    if tensor.bins != cfg.bins:
        raise DimensionMismatch(f"tensor has {tensor.bins} bins, config implies {cfg.bins}")
    lib = _lib.require_gpu()
    data = tensor.data
    c64 = data.dtype == np.complex64
    I, N, _ = data.shape
    L, shift = cfg.frame_length, cfg.frame_shift
    out = np.empty((I, (N - 1) * shift + L), np.float32 if c64 else np.float64)
    _lib.check(lib.ffca_stft_synthesize(_lib.device(), None, _lib.MEM_HOST, _lib.C64 if c64 else _lib.C128, I, N, L,
                                        shift, _lib.ptr(data), _lib.ptr(out)), "ffca_stft_synthesize")
    return out


def interior_slice(n_samples: int, cfg: StftConfig) -> slice:
    """Sample range with full window overlap, where reconstruction is exact.  stft.py:137-139."""
    return slice(cfg.frame_length, n_samples - cfg.frame_length)
