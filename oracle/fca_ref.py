"""numpy restatement of the conventional FCA EM baseline (checker only).

Layouts follow the reference (fca.py:9-11): S (J, F, I, I), v (J, N, F),
y (I, N, F), posterior means (J, N, F, I), covariances (J, N, F, I, I).
"""

from __future__ import annotations

import math

import numpy as np

from .fastfca_ref import OracleSingular, hermitize, power_floor

S_REGULARIZATION = 1e-10  # fca.py:29


def log_likelihood(S, v, y) -> float:
    """L1 = sum over (n,f) of log N(y; 0, sum_j v_j S_j).  fca.py:101-116."""
    yv = np.transpose(y, (1, 2, 0))
    mix = np.einsum("jnf,jfab->nfab", v, S)
    _, ld = np.linalg.slogdet(mix)
    if not np.isfinite(ld).all():
        raise OracleSingular("NotPositiveDefinite", "mixture covariance is singular")
    inv = np.linalg.inv(mix)
    quad = np.real(np.einsum("nfa,nfab,nfb->nf", np.conj(yv), inv, yv))
    N, F, order = yv.shape
    return float(-N * F * order * math.log(math.pi) - ld.sum() - quad.sum())


def e_step(S, v, y):
    """(mu, phi) of the full-matrix E-step.  fca.py:119-144."""
    yv = np.transpose(y, (1, 2, 0))
    R = v[..., None, None] * S[:, None]  # (J, N, F, I, I)
    try:
        mix_inv = np.linalg.inv(R.sum(axis=0))
    except np.linalg.LinAlgError as exc:
        raise OracleSingular("NotPositiveDefinite", str(exc)) from exc
    gain = np.matmul(R, mix_inv)
    mu = np.matmul(gain, yv[..., None])[..., 0]
    phi = hermitize(R - np.matmul(gain, R))
    return mu, phi


def invert_spatial(S):
    """Inverse with Cholesky-failure loading 1e-10 tr/I.  fca.py:147-158."""
    try:
        np.linalg.cholesky(S)
    except np.linalg.LinAlgError:
        tr = np.real(np.einsum("jfii->jf", S)) / S.shape[-1]
        S = S + (S_REGULARIZATION * tr)[..., None, None] * np.eye(S.shape[-1])
    try:
        return np.linalg.inv(S)
    except np.linalg.LinAlgError as exc:
        raise OracleSingular("NotPositiveDefinite", str(exc)) from exc


def m_step(mu, phi, S, v_floor=0.0):
    """(S', v') with v from the old S first.  fca.py:161-184."""
    S_inv = invert_spatial(S)
    T = mu[..., :, None] * np.conj(mu[..., None, :]) + phi
    order = S.shape[-1]
    v_new = np.real(np.einsum("jfab,jnfba->jnf", S_inv, T)) / order
    v_new = np.maximum(v_new, v_floor)
    S_new = hermitize(np.einsum("jnf,jnfab->jfab", 1.0 / v_new, T) / v_new.shape[1])
    return S_new, v_new


class FcaRunResult:
    def __init__(self, S, v, mu, phi, inversions, matmuls, loglik):
        self.S, self.v, self.mu, self.phi = S, v, mu, phi
        self.inversions, self.matmuls, self.loglik = inversions, matmuls, loglik


def run_fca(y, S0, v0, iterations=20, v_floor=None, record_likelihood=False):
    """EM sweeps; stats from the last E-step.  fca.py:187-215."""
    if v_floor is None:
        v_floor = power_floor(y)
    S, v = np.asarray(S0, np.complex128), np.asarray(v0, np.float64)
    J, N, F = v.shape
    hist = [log_likelihood(S, v, y)] if record_likelihood else None
    mu = phi = None
    inv = mm = 0
    for _ in range(iterations):
        mu, phi = e_step(S, v, y)
        inv += N * F
        mm += 2 * J * N * F
        S, v = m_step(mu, phi, S, v_floor)
        inv += J * F
        if record_likelihood:
            hist.append(log_likelihood(S, v, y))
    return FcaRunResult(S, v, mu, phi, inv, mm, hist)
