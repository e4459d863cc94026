"""FastFCA-AS estimator -- drop-in for ``fcasep.fastfca`` on the B200.

Same public names, signatures and array layouts as the reference module
(/root/reference/pkg/src/fcasep/fastfca.py); every numeric function runs on
the GPU through libffca_b200.so (include/ffca.h).  There is no CPU path.

Layouts: P (F, I, I) complex, Lam (J, F, I) real, v (J, N, F) real,
transformed statistics (J, N, F, I).  complex64 inputs stay complex64 and use
the fp32 kernels (documented extension; the reference upcasts,
fastfca.py:59-61).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatch, NotPositiveDefinite, SingularP
from .evalkit import OpCounters
from .stft import ObservationTensor

LAMBDA_FLOOR_RTOL = 1e-12  # fastfca.py:43
WEIGHT_FLOOR = 1e-300  # fastfca.py:45 (fp32 path: 1e-30)
B_REGULARIZATION = 1e-10  # fastfca.py:47
LOG_PI = math.log(math.pi)


def _as_c(a, c64: bool):
    return np.ascontiguousarray(a, dtype=np.complex64 if c64 else np.complex128)


def _as_r(a, c64: bool):
    return np.ascontiguousarray(a, dtype=np.float32 if c64 else np.float64)


@dataclass
class FastFcaParams:
    P: np.ndarray  # (F, I, I) complex, non-singular per bin
    Lam: np.ndarray  # (J, F, I) positive diagonal entries
    v: np.ndarray  # (J, N, F) positive real

    def __post_init__(self):
        c64 = np.asarray(self.P).dtype == np.complex64
        self.P = _as_c(self.P, c64)
        self.Lam = _as_r(self.Lam, c64)
        self.v = _as_r(self.v, c64)
        if self.P.ndim != 3 or self.P.shape[-1] != self.P.shape[-2]:
            raise DimensionMismatch(f"P must be (F, I, I), got {self.P.shape}")
        if self.Lam.ndim != 3 or self.Lam.shape[1:] != (self.P.shape[0], self.P.shape[-1]):
            raise DimensionMismatch(f"Lam must be (J, F, I), got {self.Lam.shape}")
        if self.v.ndim != 3 or self.v.shape[0] != self.Lam.shape[0]:
            raise DimensionMismatch(f"v must be (J, N, F), got {self.v.shape}")
        if self.v.shape[2] != self.P.shape[0]:
            raise DimensionMismatch("P and v disagree on the number of bins")

    @property
    def sources(self) -> int:
        return self.Lam.shape[0]

    @property
    def bins(self) -> int:
        return self.P.shape[0]

    @property
    def order(self) -> int:
        return self.P.shape[-1]

    def copy(self) -> "FastFcaParams":
        return FastFcaParams(self.P.copy(), self.Lam.copy(), self.v.copy())


class TransformedStats:
    """Posterior statistics in the transformed basis (fastfca.py:87-96).

    ``mu`` (J, N, F, I) complex holds P^H mu_j and ``phi`` (J, N, F, I) real the
    diagonal of P^H Phi_j P.  Statistics returned by ``run_fastfca`` are
    materialised lazily on first access (one device pass over y); until then
    ``mmse_images_fastfca`` computes images straight from the final state
    without forming mu_t.
    """

    def __init__(self, mu=None, phi=None, *, source=None):
        self._mu = mu
        self._phi = phi
        self._source = source  # (ObservationTensor, FastFcaParams) when lazy

    def _materialize(self):
        obs, params = self._source
        mu, phi = _stats(obs, params, want_mu=self._mu is None, want_phi=self._phi is None)
        if self._mu is None:
            self._mu = mu
        if self._phi is None:
            self._phi = phi

    @property
    def mu(self) -> np.ndarray:
        if self._mu is None and self._source is not None:
            self._materialize()
        return self._mu

    @mu.setter
    def mu(self, value):
        self._mu = value

    @property
    def phi(self) -> np.ndarray:
        if self._phi is None and self._source is not None:
            self._materialize()
        return self._phi

    @phi.setter
    def phi(self, value):
        self._phi = value

    @property
    def is_lazy(self) -> bool:
        return self._source is not None and (self._mu is None or self._phi is None)


@dataclass
class FastFcaRun:
    params: FastFcaParams
    stats: TransformedStats
    counters: OpCounters
    loglik_init: float | None = None
    loglik_after_em: list[float] | None = None
    loglik_after_p: list[float] | None = None


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def _check_obs(obs: ObservationTensor, params: FastFcaParams):
    if obs.channels != params.order:
        raise DimensionMismatch(f"tensor has {obs.channels} channels, params expect {params.order}")
    if params.v.shape[1:] != (obs.frames, obs.bins):
        raise DimensionMismatch(f"v is {params.v.shape}, observations have N={obs.frames}, F={obs.bins}")


def _floor_args(v_floor, J, N, F, c64):
    """Map the reference's v_floor argument (fastfca.py:406,421-424,435-436) to a C-ABI mode."""
    if v_floor is None:
        return _lib.VF_AUTO, 0.0, None
    arr = np.asarray(v_floor, dtype=np.float64)
    if arr.ndim == 0:
        return _lib.VF_SCALAR, float(arr), None
    if arr.shape in ((F,), (1, F), (1, 1, F)):
        return _lib.VF_BIN, 0.0, _as_r(arr.reshape(F), c64)
    full = np.broadcast_to(arr, (J, N, F))
    return _lib.VF_FULL, 0.0, _as_r(full, c64)


def _stats(obs, params, want_mu=True, want_phi=True):
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    code = _lib.C64 if c64 else _lib.C128
    J, N, F = params.v.shape
    I = params.order
    mu = np.empty((J, N, F, I), np.complex64 if c64 else np.complex128) if want_mu else None
    phi = np.empty((J, N, F, I), np.float32 if c64 else np.float64) if want_phi else None
    P, lam, v = _as_c(params.P, c64), _as_r(params.Lam, c64), _as_r(params.v, c64)
    rc = lib.ffca_fastfca_stats(_lib.device(), None, _lib.MEM_HOST, code, 1, I, J, N, F,
                                _lib.ptr(obs.data), _lib.ptr(P), _lib.ptr(lam), _lib.ptr(v),
                                _lib.ptr(mu), _lib.ptr(phi))
    _lib.check(rc, "ffca_fastfca_stats")
    return mu, phi


# ---------------------------------------------------------------------------
# the fused estimation loop
# ---------------------------------------------------------------------------


def run_fastfca(
    obs: ObservationTensor,
    init: FastFcaParams,
    iterations: int = 20,
    inner_iterations: int = 1,
    v_floor: float | np.ndarray | None = None,
    record_likelihood: bool = False,
) -> FastFcaRun:
    """Hybrid estimation loop on the GPU (fastfca.py:401-474).

    One EM sweep on (v, Lambda), then the fixed-point update of P, per outer
    iteration -- the whole loop is one kernel launch.  Returns the final
    parameters, lazily refreshed transformed statistics and counters; with
    ``record_likelihood`` the likelihood at init, after every EM sweep and
    after every P update.
    """
    if obs.channels != init.order:
        raise DimensionMismatch(f"tensor has {obs.channels} channels, params expect {init.order}")
    _check_obs(obs, init)
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    code = _lib.C64 if c64 else _lib.C128
    J, N, F = init.v.shape
    I = init.order
    y = obs.data
    P0, lam0, v0 = _as_c(init.P, c64), _as_r(init.Lam, c64), _as_r(init.v, c64)
    mode, vf_scalar, vf_arr = _floor_args(v_floor, J, N, F, c64)
    P = np.empty_like(P0)
    lam = np.empty_like(lam0)
    v = np.empty_like(v0)
    nev = 1 + 2 * int(iterations)
    ll = np.empty((1, nev)) if record_likelihood else None
    rc = lib.ffca_fastfca_run(_lib.device(), None, _lib.MEM_HOST, code, 1, I, J, N, F,
                              _lib.ptr(y), _lib.ptr(P0), _lib.ptr(lam0), _lib.ptr(v0),
                              mode, vf_scalar, _lib.ptr(vf_arr), int(iterations), int(inner_iterations),
                              1 if record_likelihood else 0, _lib.ptr(P), _lib.ptr(lam), _lib.ptr(v),
                              _lib.ptr(ll), None, None)
    _lib.check(rc, "ffca_fastfca_run")
    params = FastFcaParams(P=P, Lam=lam, v=v)
    counters = OpCounters()
    counters.add_inversions(int(iterations) * (I + 1) * F * int(inner_iterations))
    run = FastFcaRun(params=params, stats=TransformedStats(source=(obs, params)), counters=counters)
    if record_likelihood:
        T = int(iterations)
        run.loglik_init = float(ll[0, 0])
        run.loglik_after_em = [float(x) for x in ll[0, 1:2 * T + 1:2]]
        run.loglik_after_p = [float(x) for x in ll[0, 2:2 * T + 1:2]]
    return run


def run_fastfca_batch(y, P0, lam0, v0, iterations=20, inner_iterations=1, v_floor=None,
                      record_likelihood=False, mem=None, stream=None):
    """Batched extension: U independent mixtures in one launch.

    y (U, I, N, F), P0 (U, F, I, I), lam0 (U, J, F, I), v0 (U, J, N, F);
    v_floor None (per-mixture power floor) / scalar / (U, F).  Returns
    (P, lam, v, ll (U, 1+2T) or None).  Numpy arrays only.
    """
    lib = _lib.require_gpu()
    c64 = y.dtype == np.complex64
    code = _lib.C64 if c64 else _lib.C128
    U, I, N, F = y.shape
    J = v0.shape[1]
    if P0.shape != (U, F, I, I) or lam0.shape != (U, J, F, I) or v0.shape != (U, J, N, F):
        raise DimensionMismatch("batched shapes disagree")
    if v_floor is None:
        mode, vfs, vfa = _lib.VF_AUTO, 0.0, None
    elif np.ndim(v_floor) == 0:
        mode, vfs, vfa = _lib.VF_SCALAR, float(v_floor), None
    else:
        mode, vfs, vfa = _lib.VF_BIN, 0.0, _as_r(np.reshape(v_floor, (U, F)), c64)
    P, lam, v = np.empty_like(P0), np.empty_like(lam0), np.empty_like(v0)
    ll = np.empty((U, 1 + 2 * iterations)) if record_likelihood else None
    rc = lib.ffca_fastfca_run(_lib.device(), stream, _lib.MEM_HOST, code, U, I, J, N, F,
                              _lib.ptr(y), _lib.ptr(P0), _lib.ptr(lam0), _lib.ptr(v0), mode, vfs,
                              _lib.ptr(vfa), iterations, inner_iterations, 1 if record_likelihood else 0,
                              _lib.ptr(P), _lib.ptr(lam), _lib.ptr(v), _lib.ptr(ll), None, None)
    _lib.check(rc, "ffca_fastfca_run")
    return P, lam, v, ll
