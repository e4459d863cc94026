"""Conventional full-rank FCA EM baseline -- drop-in for ``fcasep.fca`` on the B200.

Same names, signatures and layouts as the reference module
(/root/reference/pkg/src/fcasep/fca.py): S (J, F, I, I) complex, v (J, N, F)
real, posterior means (J, N, F, I), covariances (J, N, F, I, I).  Every
numeric function is a device call into libffca_b200.so; the whole EM loop of
``run_fca`` is one bin-resident kernel launch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lazy import DeviceArray, LazyHostFields
from .errors import DimensionMismatch, NotPositiveDefinite
from .evalkit import OpCounters
from .stft import ObservationTensor

V_FLOOR_RTOL = 1e-10  # fca.py:27
S_REGULARIZATION = 1e-10  # fca.py:29


def _as_c(a, c64):
    return np.ascontiguousarray(a, dtype=np.complex64 if c64 else np.complex128)


def _as_r(a, c64):
    return np.ascontiguousarray(a, dtype=np.float32 if c64 else np.float64)


def _code(c64):
    return _lib.C64 if c64 else _lib.C128


@dataclass
class FcaParams:
    S: np.ndarray  # (J, F, I, I) complex, Hermitian PD per (j, f)
    v: np.ndarray  # (J, N, F) positive real

    def __post_init__(self):
        c64 = np.asarray(self.S).dtype == np.complex64
        self.S = _as_c(self.S, c64)
        self.v = _as_r(self.v, c64)
        if self.S.ndim != 4 or self.S.shape[-1] != self.S.shape[-2]:
            raise DimensionMismatch(f"S must be (J, F, I, I), got {self.S.shape}")
        if self.v.ndim != 3 or self.v.shape[0] != self.S.shape[0]:
            raise DimensionMismatch(f"v must be (J, N, F), got {self.v.shape}")
        if self.v.shape[2] != self.S.shape[1]:
            raise DimensionMismatch("S and v disagree on the number of bins")

    @property
    def sources(self) -> int:
        return self.S.shape[0]

    @property
    def bins(self) -> int:
        return self.S.shape[1]

    @property
    def order(self) -> int:
        return self.S.shape[-1]

    def copy(self) -> "FcaParams":
        return FcaParams(self.S.copy(), self.v.copy())


@dataclass
class PosteriorStats(LazyHostFields):
    """Posterior means (J, N, F, I) and covariances (J, N, F, I, I) (fca.py:63-66).

    ``run_fca`` returns the last sweep's E-step (at the penultimate parameters,
    which the loop kernel writes out), computed on the device right after the
    loop and kept there until a field is first read on the host (then copied to
    numpy once; see ``_lazy``).
    """

    _LAZY = ("mu", "phi")
    mu: np.ndarray
    phi: np.ndarray


@dataclass
class FcaRun:
    params: FcaParams
    stats: PosteriorStats | None
    counters: OpCounters
    loglik: list[float] | None = None


def _check(params: FcaParams, obs: ObservationTensor):
    if obs.channels != params.order:
        raise DimensionMismatch(f"tensor has {obs.channels} channels, params expect {params.order}")
    if params.v.shape[1:] != (obs.frames, obs.bins):
        raise DimensionMismatch(f"v is {params.v.shape}, observations have N={obs.frames}, F={obs.bins}")


def _floor_args(v_floor, J, N, F, c64):
    if v_floor is None:
        return _lib.VF_AUTO, 0.0, None
    arr = np.asarray(v_floor, dtype=np.float64)
    if arr.ndim == 0:
        return _lib.VF_SCALAR, float(arr), None
    if arr.shape in ((F,), (1, F), (1, 1, F)):
        return _lib.VF_BIN, 0.0, _as_r(arr.reshape(F), c64)
    return _lib.VF_FULL, 0.0, _as_r(np.broadcast_to(arr, (J, N, F)), c64)


def power_floor(obs: ObservationTensor) -> np.ndarray:
    """Per-bin floor max(1e-10 mean_{i,n} |y|^2, 1e-300), (F,).  fca.py:82-89."""
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    I, N, F = obs.data.shape
    out = np.empty(F)
    _lib.check(lib.ffca_power_floor(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, N, F,
                                    _lib.ptr(obs.data), _lib.ptr(out)), "ffca_power_floor")
    return out


def mix_covariance(params: FcaParams, n: int, f: int) -> np.ndarray:
    """sum_j v_j(n,f) S_j(f) at one point (fca.py:92-94); a host-side accessor, not on the path."""
    return np.einsum("j,jab->ab", params.v[:, n, f], params.S[:, f])


def log_likelihood(params: FcaParams, obs: ObservationTensor) -> float:
    """L1 = sum over (n, f) of log N(y; 0, sum_j v_j S_j).  fca.py:101-116."""
    _check(params, obs)
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    ll = np.empty(1)
    _lib.check(lib.ffca_fca_loglik(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                   _lib.ptr(obs.data), _lib.ptr(_as_c(params.S, c64)), _lib.ptr(_as_r(params.v, c64)),
                                   _lib.ptr(ll), None), "ffca_fca_loglik")
    if not np.isfinite(ll[0]):
        raise NotPositiveDefinite("mixture covariance is singular")
    return float(ll[0])


def e_step(params: FcaParams, obs: ObservationTensor, counters: OpCounters | None = None,
           images_layout: bool = False) -> PosteriorStats:
    """Posterior means and covariances.  fca.py:119-144."""
    _check(params, obs)
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    mu = np.empty((J, I, N, F) if images_layout else (J, N, F, I), obs.data.dtype)
    phi = None if images_layout else np.empty((J, N, F, I, I), obs.data.dtype)
    _lib.check(lib.ffca_fca_estep(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                  _lib.ptr(obs.data), _lib.ptr(_as_c(params.S, c64)), _lib.ptr(_as_r(params.v, c64)),
                                  _lib.ptr(mu), _lib.ptr(phi), 1 if images_layout else 0, None), "ffca_fca_estep")
    if counters is not None:
        counters.add_inversions(N * F)
        counters.add_matmuls(2 * J * N * F)
    return PosteriorStats(mu=mu, phi=phi)


def m_step(stats: PosteriorStats, params: FcaParams, v_floor: float | np.ndarray = 0.0,
           counters: OpCounters | None = None) -> FcaParams:
    """v from the old S, then S from the new v.  fca.py:161-184."""
    lib = _lib.require_gpu()
    c64 = params.S.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    mode, vfs, vfa = _floor_args(v_floor, J, N, F, c64)
    if mode == _lib.VF_AUTO:
        raise ValueError("m_step needs an explicit v_floor")
    S_new = np.empty_like(params.S)
    v_new = np.empty_like(params.v)
    _lib.check(lib.ffca_fca_mstep(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                  _lib.ptr(_as_c(stats.mu, c64)), _lib.ptr(_as_c(stats.phi, c64)),
                                  _lib.ptr(params.S), mode, vfs, _lib.ptr(vfa), _lib.ptr(S_new), _lib.ptr(v_new), None),
               "ffca_fca_mstep")
    if counters is not None:
        counters.add_inversions(J * F)
    return FcaParams(S=S_new, v=v_new)


def run_fca(
    obs: ObservationTensor,
    init: FcaParams,
    iterations: int = 20,
    v_floor: float | np.ndarray | None = None,
    record_likelihood: bool = False,
) -> FcaRun:
    """E and M steps for ``iterations`` sweeps in one device launch.  fca.py:187-215.

    ``stats`` are those of the last sweep's E-step (at the penultimate
    parameters); None when iterations == 0, in which case
    ``params is init`` as in the reference.
    """
    _check(init, obs)
    counters = OpCounters()
    J, N, F = init.v.shape
    I = init.order
    if iterations == 0:
        hist = [log_likelihood(init, obs)] if record_likelihood else None
        return FcaRun(params=init, stats=None, counters=counters, loglik=hist)
    import torch
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    code = _code(c64)
    S0, v0 = _as_c(init.S, c64), _as_r(init.v, c64)
    mode, vfs, vfa = _floor_args(v_floor, J, N, F, c64)
    # y, the initial state and every result live on the device between the loop and the final
    # E-step (one H2D of y); S, v (and the likelihood) come back, the statistics stay in HBM
    dev = torch.device("cuda", _lib.device())

    def up(a):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    dy, dS0, dv0, dvfa = up(obs.data), up(S0), up(v0), up(vfa)
    dS, dv, dSp, dvp = torch.empty_like(dS0), torch.empty_like(dv0), torch.empty_like(dS0), torch.empty_like(dv0)
    dll = torch.empty((1, 1 + iterations), dtype=torch.float64, device=dev) if record_likelihood else None
    ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    _lib.check(lib.ffca_fca_run(dev.index, None, _lib.MEM_DEVICE, code, 1, I, J, N, F, ptr(dy), ptr(dS0), ptr(dv0),
                                mode, vfs, ptr(dvfa), int(iterations), 1 if record_likelihood else 0, ptr(dS),
                                ptr(dv), ptr(dSp), ptr(dvp), ptr(dll), None), "ffca_fca_run")
    counters.add_inversions(iterations * (J + N) * F)
    counters.add_matmuls(iterations * 2 * J * N * F)
    # fca.py:211: the last sweep's E-step statistics, at the penultimate parameters
    mu = torch.empty((J, N, F, I), dtype=dy.dtype, device=dev)
    phi = torch.empty((J, N, F, I, I), dtype=dy.dtype, device=dev)
    _lib.check(lib.ffca_fca_estep(dev.index, None, _lib.MEM_DEVICE, code, 1, I, J, N, F, ptr(dy), ptr(dSp), ptr(dvp),
                                  ptr(mu), ptr(phi), 0, None), "ffca_fca_estep")
    stats = PosteriorStats(mu=DeviceArray(mu), phi=DeviceArray(phi))
    S, v = dS.cpu().numpy(), dv.cpu().numpy()
    ll = dll.cpu().numpy() if record_likelihood else None
    hist = [float(x) for x in ll[0]] if record_likelihood else None
    return FcaRun(params=FcaParams(S=S, v=v), stats=stats, counters=counters, loglik=hist)


def run_fca_batch(y, S0, v0, iterations=20, v_floor=None, record_likelihood=False, stream=None, out=None):
    """Batched extension: U mixtures (U, I, N, F) in one launch; returns (S, v, ll)."""
    lib = _lib.require_gpu()
    c64 = y.dtype == np.complex64
    U, I, N, F = y.shape
    J = v0.shape[1]
    if v_floor is None:
        mode, vfs, vfa = _lib.VF_AUTO, 0.0, None
    else:
        mode, vfs, vfa = _lib.VF_SCALAR, float(v_floor), None
    S, v = out if out is not None else (np.empty_like(S0), np.empty_like(v0))
    ll = np.empty((U, 1 + iterations)) if record_likelihood else None
    _lib.check(lib.ffca_fca_run(_lib.device(), stream, _lib.MEM_HOST, _code(c64), U, I, J, N, F, _lib.ptr(y),
                                _lib.ptr(S0), _lib.ptr(v0), mode, vfs, _lib.ptr(vfa), int(iterations),
                                1 if record_likelihood else 0, _lib.ptr(S), _lib.ptr(v), None, None, _lib.ptr(ll),
                                None), "ffca_fca_run")
    return S, v, ll
