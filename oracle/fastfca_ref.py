"""numpy restatement of the FastFCA-AS estimator (checker only, see __init__).

Array conventions follow the reference's public layouts:
  y    (I, N, F) complex      -- ``stft.ObservationTensor.data`` (stft.py:56-67)
  P    (F, I, I) complex      -- fastfca.py:54
  lam  (J, F, I) real         -- fastfca.py:55
  v    (J, N, F) real         -- fastfca.py:56
Internally the loop works bin-major ((F, N, I) etc.), as the reference's
fused loop does (fastfca.py:428-436).

Each function cites the reference lines whose arithmetic it restates.
"""

from __future__ import annotations

import math

import numpy as np

LAMBDA_FLOOR_RTOL = 1e-12  # fastfca.py:43
WEIGHT_FLOOR = 1e-300  # fastfca.py:45
B_REGULARIZATION = 1e-10  # fastfca.py:47
V_FLOOR_RTOL = 1e-10  # fca.py:27
LOG_PI = math.log(math.pi)


class OracleSingular(Exception):
    """Raised where the reference raises SingularP / SingularWeightedCovariance."""

    def __init__(self, kind: str, msg: str = ""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def power_floor(y: np.ndarray) -> np.ndarray:
    """Per-bin v floor, (F,).  fca.py:82-89."""
    p = np.abs(y) ** 2
    return np.maximum(V_FLOOR_RTOL * p.mean(axis=(0, 1)), 1e-300)


def transform(P: np.ndarray, y: np.ndarray) -> np.ndarray:
    """y_t[n, f, b] = sum_a conj(P[f, a, b]) y[a, n, f]  -> (N, F, I).

    fastfca.py:113-116."""
    return np.einsum("fab,anf->nfb", np.conj(P), y)


def weights(v: np.ndarray, lam: np.ndarray) -> np.ndarray:
    """w[n, f, i] = max(sum_j v[j,n,f] lam[j,f,i], 1e-300).  fastfca.py:138-141."""
    return np.maximum(np.einsum("jnf,jfi->nfi", v, lam), WEIGHT_FLOOR)


def e_step_diag(P, lam, v, y_t):
    """Transformed posterior (mu_t, phi_t), each (J, N, F, I).  fastfca.py:144-157."""
    w = weights(v, lam)
    a = v[:, :, :, None] * lam[:, None, :, :]
    g = a / w[None]
    mu = g * y_t[None]
    phi = np.maximum(a * (1.0 - g), 0.0)
    return mu, phi


def m_step_diag(mu, phi, lam, v_floor=0.0):
    """(v', lam') from transformed stats.  fastfca.py:160-181."""
    order = lam.shape[-1]
    m2 = mu.real ** 2 + mu.imag ** 2 + phi
    v_new = np.maximum(np.einsum("jnfi,jfi->jnf", m2, 1.0 / lam) / order, v_floor)
    lam_new = np.einsum("jnf,jnfi->jfi", 1.0 / v_new, m2) / v_new.shape[1]
    lam_new = np.maximum(lam_new, LAMBDA_FLOOR_RTOL * lam_new.max(axis=-1, keepdims=True))
    return v_new, lam_new


def _inv(m: np.ndarray, kind: str) -> np.ndarray:
    try:
        return np.linalg.inv(m)
    except np.linalg.LinAlgError as exc:
        raise OracleSingular(kind, str(exc)) from exc


def _inv_loaded(B: np.ndarray) -> np.ndarray:
    """Inverse with one trace-loaded retry.  fastfca.py:184-194."""
    try:
        return np.linalg.inv(B)
    except np.linalg.LinAlgError:
        tr = np.real(np.trace(B, axis1=-2, axis2=-1))
        eye = np.eye(B.shape[-1])
        return _inv(B + (B_REGULARIZATION * tr)[..., None, None] * eye, "SingularWeightedCovariance")


def weighted_covariances(y, v, lam, hermitian=True):
    """B[i, f] = (1/N) sum_n y y^H / w_i, (I, F, I, I).  fastfca.py:214-224 / 352-358."""
    w = weights(v, lam)  # (N, F, I)
    N = y.shape[1]
    B = np.einsum("anf,bnf,nfi->ifab", y, np.conj(y), 1.0 / w) / N
    if hermitian:
        B = hermitize(B)
    return B


def p_columns(P, B, inner_iterations=1):
    """Column-wise fixed-point map [P]_i <- B_i^{-1} [P^{-H}]_i, K times.

    fastfca.py:225-237 / 359-370.  Returns (P', inversions counted)."""
    order = P.shape[-1]
    count = 0
    for _ in range(inner_iterations):
        Pinv = _inv(P, "SingularP")
        count += P.shape[0]
        PinvH = np.conj(np.swapaxes(Pinv, -1, -2))
        out = np.empty_like(P)
        for i in range(order):
            Bi = _inv_loaded(B[i])
            count += P.shape[0]
            out[:, :, i] = np.einsum("fab,fb->fa", Bi, PinvH[:, :, i])
        P = out
    return P, count


def fixed_point_update_P(P, lam, v, y, inner_iterations=1):
    """Unfused P update.  fastfca.py:197-237."""
    B = weighted_covariances(y, v, lam, hermitian=True)
    return p_columns(P, B, inner_iterations)


def log_likelihood(P, lam, v, y) -> float:
    """L2 in the transformed basis.  fastfca.py:240-255."""
    y_t = transform(P, y)
    w = weights(v, lam)
    sign, ld = np.linalg.slogdet(P)
    ld = np.real(ld)
    if not np.isfinite(ld).all():
        raise OracleSingular("SingularP", "basis transform is singular")
    q = y_t.real ** 2 + y_t.imag ** 2
    N, F, order = y_t.shape
    return float(-N * F * order * LOG_PI - np.log(w).sum() - (q / w).sum() + 2.0 * N * ld.sum())


def back_transform_means(P, mu_t):
    """Solve P^H x = mu_t per bin; (J, N, F, I) in and out.  fastfca.py:258-273."""
    PH = np.conj(np.swapaxes(P, -1, -2))
    out = np.empty_like(mu_t)
    for f in range(P.shape[0]):
        try:
            out[:, :, f, :] = np.linalg.solve(PH[f], mu_t[:, :, f, :].reshape(-1, P.shape[-1]).T).T.reshape(
                mu_t.shape[0], mu_t.shape[1], -1)
        except np.linalg.LinAlgError as exc:
            raise OracleSingular("SingularP", str(exc)) from exc
    return out


def images(P, mu_t):
    """Wiener images (J, I, N, F).  wiener.py:38-43."""
    return back_transform_means(P, mu_t).transpose(0, 3, 1, 2)


def hermitize(a):
    """Lower triangle mirrored, real diagonal.  matcore.py:39-51."""
    lo = np.tril(a, -1)
    out = lo + np.conj(np.swapaxes(lo, -1, -2))
    idx = np.arange(a.shape[-1])
    out[..., idx, idx] = np.real(a[..., idx, idx])
    return out


def reconstruct_spatial_covariances(P, lam):
    """S_j = P^{-H} diag(lam_j) P^{-1}, hermitized, (J, F, I, I).  fastfca.py:119-126."""
    Pinv = _inv(P, "SingularP")
    S = np.einsum("fia,jfi,fib->jfab", np.conj(Pinv), lam, Pinv)
    return hermitize(S)


# ---------------------------------------------------------------------------
# the fused bin-major loop (fastfca.py:312-474)
# ---------------------------------------------------------------------------


def em_sweep_binmajor(q, v, lam, order, vfl):
    """One fused E+M sweep on (F,N,*) arrays.  fastfca.py:323-346.

    q (F,N,I) = |P^H y|^2 ; v (F,N,J) ; lam (F,J,I) ; vfl broadcastable (F,N,J).
    """
    w = np.maximum(np.matmul(v, lam), WEIGHT_FLOOR)
    iw = 1.0 / w
    qiw2 = (q * iw) * iw
    lamT = np.swapaxes(lam, 1, 2)
    r1 = np.matmul(iw, lamT)
    r2 = np.matmul(qiw2, lamT)
    step = (r1 - r2) * v * v / order
    v_new = np.maximum(v - step, vfl)
    ratio = v / v_new
    s0 = ratio.sum(axis=1)  # (F, J)
    d = qiw2 - iw
    s1 = np.matmul(np.swapaxes(ratio * v, 1, 2), d)  # (F, J, I)
    N = v.shape[1]
    lam_new = lam * (s0[:, :, None] / N) + lam * lam * (s1 / N)
    lam_new = np.maximum(lam_new, LAMBDA_FLOOR_RTOL * lam_new.max(axis=-1, keepdims=True))
    return v_new, lam_new


def b_accumulate_binmajor(y_fni, v, lam, y_fin=None, yc_fni=None):
    """B (I, F, I, I) without hermitization, as in the fused loop.  fastfca.py:352-358.

    B_i = (y * (1/w_i)) y^H / N as one batched (F: I x N @ N x I) product per i, the
    reference's own GEMM formulation (a three-operand einsum here ran ~2x slower than the
    reference).  y_fin (F, I, N) and yc_fni = conj(y_fni) are loop invariants the caller
    may pass precomputed.
    """
    w = np.maximum(np.matmul(v, lam), WEIGHT_FLOOR)  # (F, N, I)
    N = y_fni.shape[1]
    if y_fin is None:
        y_fin = np.ascontiguousarray(np.transpose(y_fni, (0, 2, 1)))
    if yc_fni is None:
        yc_fni = np.conj(y_fni)
    iw_fin = np.ascontiguousarray(np.transpose(1.0 / w, (0, 2, 1)))  # (F, I, N)
    order = y_fni.shape[-1]
    B = np.empty((order, y_fni.shape[0], order, order), dtype=np.complex128)
    for i in range(order):
        B[i] = np.matmul(y_fin * iw_fin[:, i, None, :], yc_fni) / N
    return B


def _loglik_binmajor(q, v, lam, P):
    """fastfca.py:390-398."""
    w = np.maximum(np.matmul(v, lam), WEIGHT_FLOOR)
    _, ld = np.linalg.slogdet(P)
    N = q.shape[1]
    tot = -N * P.shape[0] * P.shape[-1] * LOG_PI
    tot -= np.log(w).sum() + (q / w).sum()
    tot += 2.0 * N * np.real(ld).sum()
    return float(tot)


class FusedRun:
    """Result of ``run_fastfca``; same fields as the reference's FastFcaRun (fastfca.py:99-106)."""

    def __init__(self, P, lam, v, mu, phi, inversions, ll_init, ll_em, ll_p):
        self.P, self.lam, self.v = P, lam, v
        self.mu, self.phi = mu, phi
        self.inversions = inversions
        self.loglik_init, self.loglik_after_em, self.loglik_after_p = ll_init, ll_em, ll_p


def run_fastfca(y, P0, lam0, v0, iterations=20, inner_iterations=1, v_floor=None,
                record_likelihood=False, stats=True):
    """Hybrid loop.  fastfca.py:401-474.  y is (I,N,F)."""
    if v_floor is None:
        v_floor = power_floor(y)
    order = P0.shape[-1]
    y_fni = np.ascontiguousarray(np.transpose(y, (2, 1, 0)))
    y_fin = np.ascontiguousarray(np.transpose(y, (2, 0, 1)))
    yc_fni = np.conj(y_fni)
    v = np.ascontiguousarray(np.transpose(v0, (2, 1, 0))).astype(np.float64)
    lam = np.ascontiguousarray(np.transpose(lam0, (1, 0, 2))).astype(np.float64)
    P = np.array(P0, dtype=np.complex128)
    vfl = np.ascontiguousarray(
        np.transpose(np.broadcast_to(np.asarray(v_floor, dtype=np.float64), v0.shape), (2, 1, 0)))

    def q_of(Pm):
        yt = np.matmul(y_fni, np.conj(Pm))
        return yt.real ** 2 + yt.imag ** 2

    ll0, lle, llp = None, None, None
    if record_likelihood:
        ll0, lle, llp = _loglik_binmajor(q_of(P), v, lam, P), [], []
    count = 0
    for _ in range(iterations):
        v, lam = em_sweep_binmajor(q_of(P), v, lam, order, vfl)
        if record_likelihood:
            lle.append(_loglik_binmajor(q_of(P), v, lam, P))
        B = b_accumulate_binmajor(y_fni, v, lam, y_fin, yc_fni)
        P, c = p_columns(P, B, inner_iterations)
        count += c
        if record_likelihood:
            llp.append(_loglik_binmajor(q_of(P), v, lam, P))
    lam_pub = np.ascontiguousarray(np.transpose(lam, (1, 0, 2)))
    v_pub = np.ascontiguousarray(np.transpose(v, (2, 1, 0)))
    mu = phi = None
    if stats:
        mu, phi = stats_refresh(P, lam_pub, v_pub, y)
    return FusedRun(P, lam_pub, v_pub, mu, phi, count, ll0, lle, llp)


def stats_refresh(P, lam, v, y):
    """Final transformed stats, (J,N,F,I) each.  fastfca.py:373-387."""
    return e_step_diag(P, lam, v, transform(P, y))


def back_transform_stats(P, mu_t, phi_t):
    """(mu (J,N,F,I), phi (J,N,F,I,I)) in the microphone basis.  fastfca.py:276-287."""
    mu = back_transform_means(P, mu_t)
    A = np.linalg.inv(np.conj(np.swapaxes(P, -1, -2)))
    phi = np.einsum("fai,jnfi,fbi->jnfab", A, phi_t, np.conj(A))
    return mu, hermitize(phi)


def params_from_covariances(S_hat, v):
    """Whitening init: P = (chol(sum_j S_j)^H)^-1, lam = diag(P^H S_j P).  fastfca.py:290-309."""
    total = S_hat.sum(axis=0)
    try:
        low = np.linalg.cholesky(total)
    except np.linalg.LinAlgError as exc:
        raise OracleSingular("NotPositiveDefinite", str(exc)) from exc
    P = np.linalg.inv(np.conj(np.swapaxes(low, -1, -2)))
    lam = np.real(np.einsum("fai,jfab,fbi->jfi", np.conj(P), S_hat, P))
    lam = np.maximum(lam, LAMBDA_FLOOR_RTOL * lam.max(axis=-1, keepdims=True))
    return P, lam, np.asarray(v, dtype=np.float64)
