"""Source-image recovery (multichannel Wiener filter) -- wiener.py:20-43 on the GPU.

Resynthesis / WAV output are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fastfca, fca
from .stft import ObservationTensor


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

    When ``stats`` is the lazy refresh returned by ``run_fastfca`` for these
    params, the device computes the images straight from (y, P, Lambda, v)
    in one pass (mu_tilde is never materialised).
    """
    src = getattr(stats, "_source", None)
    if src is not None and stats._mu is None and src[1] is params:
        return SeparatedImages(stft=fastfca.images_from_state(src[0], params))
    return SeparatedImages(stft=fastfca.back_transform_means(params.P, stats.mu, images_layout=True))
