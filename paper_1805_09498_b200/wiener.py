"""Source-image recovery (multichannel Wiener filter) -- wiener.py:20-53 on the GPU.

WAV output (wiener.py:56-79) is file I/O and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fastfca, fca
from .stft import ObservationTensor, StftConfig, synthesize


@dataclass
class SeparatedImages:
    """Per-source multichannel source-image estimates."""

    stft: np.ndarray  # (J, I, N, F) complex
    audio: np.ndarray | None = None

    @property
    def sources(self) -> int:
        return self.stft.shape[0]


def mmse_images_fca(params: fca.FcaParams, obs: ObservationTensor) -> SeparatedImages:
    """Wiener estimates from full-matrix parameters (a final E-step's means).  wiener.py:32-35.

    The device writes the means directly in the (J, I, N, F) image layout.
    """
    return SeparatedImages(stft=fca.e_step(params, obs, images_layout=True).mu)


def mmse_images_fastfca(params: fastfca.FastFcaParams, stats: fastfca.TransformedStats) -> SeparatedImages:
    """Wiener estimates x_j = P^{-H} mu_tilde_j.  wiener.py:38-43.

    One device pass: P^{-H} per bin, then the back-solve written straight in
    the (J, I, N, F) image layout.  Statistics still in device memory (the
    ``run_fastfca`` snapshot) are used in place; only the images come back.  (``fastfca.images_from_state`` fuses the
    refresh too, for callers that never need mu_tilde.)
    """
    mu_t = stats.device_tensor("mu") if isinstance(stats, fastfca.TransformedStats) else None
    return SeparatedImages(stft=fastfca.back_transform_means(params.P, stats.mu if mu_t is None else mu_t,
                                                             images_layout=True))


def resynthesize_images(images: SeparatedImages, cfg: StftConfig = StftConfig()) -> SeparatedImages:
    """Time-domain audio for every source by overlap-add synthesis.  wiener.py:46-53.

    All J x I image channels go through one batched device synthesis call.
    """
    J, I, N, F = images.stft.shape
    flat = ObservationTensor(np.ascontiguousarray(images.stft).reshape(J * I, N, F), check_finite=False)
    audio = synthesize(flat, cfg)
    return SeparatedImages(stft=images.stft, audio=audio.reshape(J, I, -1))
