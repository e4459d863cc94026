"""Observation tensor: the input contract of the hot path (stft.py:56-79).

Dtype policy (documented extension): complex64 data stays complex64 and runs
the fp32 device path; anything else is coerced to complex128 exactly as the
reference does (stft.py:63).  The STFT filterbank itself is out of scope
(SURVEY.md §2 row 6, §8(f) "next" #1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatch


def _coerce(data) -> np.ndarray:
    arr = np.asarray(data)
    if arr.dtype == np.complex64:
        return np.ascontiguousarray(arr)
    return np.ascontiguousarray(arr, dtype=np.complex128)


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
