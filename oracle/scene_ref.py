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
