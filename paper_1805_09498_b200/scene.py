"""Initial parameters for the estimators, computed on the device.

Drop-in for the initialisation half of the reference's ``fcasep.scene``
(scene.py:191-275): ``oracle_covariances``, ``diffuse_covariances``,
``init_oracle``, ``init_diffuse`` and ``reference_tensors``, same names,
argument meaning, layouts and errors.  The scene *synthesis* half
(synth_sources, synth_rirs, mix_scene, file loading) is out of scope
(SURVEY.md §8(f)).

The per-bin reductions (power-normalised outer products over frames, the
average observed covariance, diagonal loading) run in one CUDA kernel
(``ffca_init_covariances``, csrc/bins.cu); the power floor is
``fca.power_floor`` on the device.  The only host arithmetic is drawing the
J seeded I x I perturbations W_j from the reference's RNG stream
(``numpy.random.default_rng(seed)``, scene.py:232-239): J * I * I numbers,
identical to the reference bit for bit.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import DimensionMismatch
from .fca import FcaParams, power_floor
from .stft import ObservationTensor, StftConfig, analyze

# scene.py:195-197: relative diagonal loading that keeps initial covariances PD.
INIT_LOADING = 1e-9

_ORACLE, _DIFFUSE = 0, 1


def _code(c64: bool) -> int:
    return _lib.C64 if c64 else _lib.C128


def _floor_2d(obs: ObservationTensor) -> np.ndarray:
    return np.ascontiguousarray(power_floor(obs).reshape(1, -1))


def _perturbations(order: int, n_sources: int, seed: int) -> np.ndarray:
    """W_j = A A^H scaled to trace I, A complex Gaussian, in the reference's draw order (scene.py:232-239)."""
    rng = np.random.default_rng(seed)
    W = np.empty((n_sources, order, order), np.complex128)
    for j in range(n_sources):
        A = rng.standard_normal((order, order)) + 1j * rng.standard_normal((order, order))
        Wj = A @ A.conj().T
        Wj *= order / np.trace(Wj).real
        W[j] = Wj
    return W


def _run(mode: int, x: np.ndarray, obs: ObservationTensor, J: int, W=None):
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    I, N, F = obs.data.shape
    cdt = np.complex64 if c64 else np.complex128
    x = np.ascontiguousarray(x, dtype=cdt)
    floor = _floor_2d(obs)
    S = np.empty((J, F, I, I), cdt)
    v = np.empty((J, N, F), np.float32 if c64 else np.float64)
    Wd = None if W is None else np.ascontiguousarray(W, dtype=cdt)
    _lib.check(lib.ffca_init_covariances(_lib.device(), None, _lib.MEM_HOST, _code(c64), mode, 1, I, J, N, F,
                                         _lib.ptr(x), _lib.ptr(floor), _lib.ptr(Wd), _lib.ptr(S), _lib.ptr(v)),
               "ffca_init_covariances")
    return S, v


def oracle_covariances(refs: np.ndarray, obs: ObservationTensor) -> tuple[np.ndarray, np.ndarray]:
    """Spatial covariances and powers from reference source-image STFTs.  scene.py:207-223.

    ``refs`` is (J, I, N, F).  v_hat = max(||x_j||^2 / I, power_floor), S_hat the
    power-normalised outer products averaged over frames, diagonally loaded.
    Returns S_hat (J, F, I, I), v_hat (J, N, F).
    """
    refs = np.asarray(refs)
    if refs.ndim != 4 or refs.shape[1:] != obs.data.shape:
        raise DimensionMismatch(f"refs shape {refs.shape} does not match observations {obs.data.shape}")
    return _run(_ORACLE, refs, obs, refs.shape[0])


def diffuse_covariances(obs: ObservationTensor, n_sources: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Blind fallback: average observed covariance + seeded PD perturbation per source.  scene.py:226-247."""
    if n_sources < 1:
        raise DimensionMismatch(f"n_sources must be >= 1, got {n_sources}")
    W = _perturbations(obs.channels, n_sources, seed)
    return _run(_DIFFUSE, obs.data, obs, n_sources, W)


def init_oracle(refs: np.ndarray, obs: ObservationTensor, algorithm: str = "fca"):
    """Oracle initialisation from reference source images.  scene.py:250-259."""
    S_hat, v_hat = oracle_covariances(refs, obs)
    return _params(S_hat, v_hat, algorithm)


def init_diffuse(obs: ObservationTensor, n_sources: int, seed: int, algorithm: str = "fca"):
    """Seeded diffuse initialisation (deterministic for a given seed).  scene.py:262-271."""
    S_hat, v_hat = diffuse_covariances(obs, n_sources, seed)
    return _params(S_hat, v_hat, algorithm)


def _params(S_hat, v_hat, algorithm):
    if algorithm == "fca":
        return FcaParams(S=S_hat, v=v_hat)
    if algorithm == "fastfca":
        from .fastfca import params_from_covariances

        return params_from_covariances(S_hat, v_hat)
    raise ValueError(f"unknown algorithm {algorithm!r}")


def reference_tensors(references, cfg: StftConfig) -> np.ndarray:
    """STFTs of all reference source images, (J, I, N, F).  scene.py:274-276.

    ``references`` is a sequence of (I, S) source images (the reference takes a
    Scene and reads ``scene.references``; either is accepted here).
    """
    refs = getattr(references, "references", references)
    return np.stack([analyze(ref, cfg).data for ref in refs])
