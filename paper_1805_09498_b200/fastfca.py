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
from ._lazy import DeviceArray, LazyHostFields
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


@dataclass
class TransformedStats(LazyHostFields):
    """Posterior statistics in the transformed basis (fastfca.py:87-96).

    ``mu`` (J, N, F, I) complex holds P^H mu_j and ``phi`` (J, N, F, I) real the
    diagonal of P^H Phi_j P.  ``run_fastfca`` computes them at the final state in
    the same device call as the loop (fastfca.py:466), so they are a snapshot:
    later changes to ``run.params`` do not touch them.  The snapshot stays in
    device memory until a field is first read on the host (then it is copied
    to numpy once, and from then on is a plain array): a device consumer such
    as ``wiener.mmse_images_fastfca`` uses it in place, so the statistics
    never cross PCIe in the reference's estimate -> images flow (cli.py:227-233).
    ``dataclasses.replace / asdict``, equality and pickling see numpy arrays.
    """

    _LAZY = ("mu", "phi")
    mu: np.ndarray
    phi: np.ndarray


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


def _device_stats_buffers(U, J, N, F, I, c64):
    """Device tensors for the statistics (U, J, N, F, I) on the library's device."""
    import torch
    dev = torch.device("cuda", _lib.device())
    return (torch.empty((U, J, N, F, I), dtype=torch.complex64 if c64 else torch.complex128, device=dev),
            torch.empty((U, J, N, F, I), dtype=torch.float32 if c64 else torch.float64, device=dev))


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
    iteration -- the whole loop is one kernel launch, followed by the statistics
    refresh in the same call.  Returns the final parameters, the transformed
    statistics at the final state and counters; with
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
    mu, phi = _device_stats_buffers(1, J, N, F, I, c64)
    nev = 1 + 2 * int(iterations)
    ll = np.empty((1, nev)) if record_likelihood else None
    # the loop and the final statistics refresh (fastfca.py:466) in one device call; the
    # statistics stay in device memory (TransformedStats copies them on first host access)
    rc = lib.ffca_fastfca_run_stats(_lib.device(), None, _lib.MEM_HOST_STATS_DEVICE, code, 1, I, J, N, F,
                                    _lib.ptr(y), _lib.ptr(P0), _lib.ptr(lam0), _lib.ptr(v0),
                                    mode, vf_scalar, _lib.ptr(vf_arr), int(iterations), int(inner_iterations),
                                    1 if record_likelihood else 0, _lib.ptr(P), _lib.ptr(lam), _lib.ptr(v),
                                    _lib.ptr(ll), None, None, mu.data_ptr(), phi.data_ptr())
    _lib.check(rc, "ffca_fastfca_run_stats")
    params = FastFcaParams(P=P, Lam=lam, v=v)
    counters = OpCounters()
    counters.add_inversions(int(iterations) * (I + 1) * F * int(inner_iterations))
    stats = TransformedStats(mu=DeviceArray(mu[0]), phi=DeviceArray(phi[0]))
    run = FastFcaRun(params=params, stats=stats, counters=counters)
    if record_likelihood:
        T = int(iterations)
        run.loglik_init = float(ll[0, 0])
        run.loglik_after_em = [float(x) for x in ll[0, 1:2 * T + 1:2]]
        run.loglik_after_p = [float(x) for x in ll[0, 2:2 * T + 1:2]]
    return run


def run_fastfca_batch(y, P0, lam0, v0, iterations=20, inner_iterations=1, v_floor=None,
                      record_likelihood=False, stream=None, out=None, stats=False, stats_out=None):
    """Batched extension: U independent mixtures in one launch.

    y (U, I, N, F), P0 (U, F, I, I), lam0 (U, J, F, I), v0 (U, J, N, F);
    v_floor None (per-mixture power floor) / scalar / (U, F).  Returns
    (P, lam, v, ll (U, 1+2T) or None); with ``stats`` also (mu, phi), each
    (U, J, N, F, I) -- run_fastfca's final refresh for every mixture.  Numpy
    arrays in and out; with ``stats="device"`` the statistics are returned as
    device (torch) tensors instead and never cross PCIe (``stats_out`` may then
    be a pair of such tensors to fill).
    """
    y = np.asarray(y)
    if not np.iscomplexobj(y) or y.ndim != 4:
        raise DimensionMismatch(f"y must be a complex (U, I, N, F) array, got {y.dtype} {y.shape}")
    c64 = y.dtype == np.complex64
    code = _lib.C64 if c64 else _lib.C128
    # every array in the precision the kernel runs in (y's): the C ABI reads them as such
    y = _as_c(y, c64)
    P0, lam0, v0 = _as_c(P0, c64), _as_r(lam0, c64), _as_r(v0, c64)
    U, I, N, F = y.shape
    J = v0.shape[1] if v0.ndim == 4 else -1
    if P0.shape != (U, F, I, I) or lam0.shape != (U, J, F, I) or v0.shape != (U, J, N, F):
        raise DimensionMismatch("batched shapes disagree")
    if out is not None:
        out = tuple(out)
        if len(out) != 3:
            raise ValueError("out must be (P, lam, v)")
        for o, ref, name in zip(out, (P0, lam0, v0), ("P", "lam", "v")):
            if (not isinstance(o, np.ndarray) or o.shape != ref.shape or o.dtype != ref.dtype
                    or not o.flags.c_contiguous or not o.flags.writeable):
                raise ValueError(f"out {name} must be a writeable C-contiguous {ref.dtype} array of shape {ref.shape}")
    if v_floor is None:
        mode, vfs, vfa = _lib.VF_AUTO, 0.0, None
    elif np.ndim(v_floor) == 0:
        mode, vfs, vfa = _lib.VF_SCALAR, float(v_floor), None
    else:
        mode, vfs, vfa = _lib.VF_BIN, 0.0, _as_r(np.reshape(v_floor, (U, F)), c64)
    P, lam, v = out if out is not None else (np.empty_like(P0), np.empty_like(lam0), np.empty_like(v0))
    ll = np.empty((U, 1 + 2 * iterations)) if record_likelihood else None
    mu = phi = None
    stats_dev = isinstance(stats, str) and stats == "device"
    if stats_dev:
        if stats_out is not None:
            mu, phi = stats_out
            for o, shape, cplx in ((mu, (U, J, N, F, I), True), (phi, (U, J, N, F, I), False)):
                if (not hasattr(o, "data_ptr") or not o.is_cuda or tuple(o.shape) != shape or not o.is_contiguous()
                        or o.is_complex() != cplx or o.element_size() != (y.itemsize if cplx else v0.itemsize)):
                    raise ValueError(f"stats_out must be contiguous CUDA tensors of shape {shape} in y's precision")
        else:
            mu, phi = _device_stats_buffers(U, J, N, F, I, c64)
    elif stats:
        if stats_out is not None:
            mu, phi = stats_out
            for o, shape, dt in ((mu, (U, J, N, F, I), y.dtype), (phi, (U, J, N, F, I), v0.dtype)):
                if (not isinstance(o, np.ndarray) or o.shape != shape or o.dtype != dt or not o.flags.c_contiguous
                        or not o.flags.writeable):
                    raise ValueError(f"stats_out must be writeable C-contiguous {dt} arrays of shape {shape}")
        else:
            mu, phi = np.empty((U, J, N, F, I), y.dtype), np.empty((U, J, N, F, I), v0.dtype)
    lib = _lib.require_gpu()
    rc = lib.ffca_fastfca_run_stats(_lib.device(), stream, _lib.MEM_HOST_STATS_DEVICE if stats_dev else _lib.MEM_HOST,
                                    code, U, I, J, N, F,
                                    _lib.ptr(y), _lib.ptr(P0), _lib.ptr(lam0), _lib.ptr(v0), mode, vfs,
                                    _lib.ptr(vfa), iterations, inner_iterations, 1 if record_likelihood else 0,
                                    _lib.ptr(P), _lib.ptr(lam), _lib.ptr(v), _lib.ptr(ll), None, None,
                                    mu.data_ptr() if stats_dev else _lib.ptr(mu),
                                    phi.data_ptr() if stats_dev else _lib.ptr(phi))
    _lib.check(rc, "ffca_fastfca_run_stats")
    if stats:
        return P, lam, v, ll, mu, phi
    return P, lam, v, ll


# ---------------------------------------------------------------------------
# unfused public steps (each one a device call)
# ---------------------------------------------------------------------------


def _code(c64):
    return _lib.C64 if c64 else _lib.C128


def transform_observations(P: np.ndarray, obs: ObservationTensor) -> np.ndarray:
    """y_tilde(n,f) = P(f)^H y(n,f), returned as (N, F, I).  fastfca.py:113-116."""
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    I, N, F = obs.data.shape
    P = _as_c(P, c64)
    if P.shape != (F, I, I):
        raise DimensionMismatch(f"P must be (F, I, I) = {(F, I, I)}, got {P.shape}")
    out = np.empty((N, F, I), obs.data.dtype)
    _lib.check(lib.ffca_transform(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, N, F,
                                  _lib.ptr(obs.data), _lib.ptr(P), _lib.ptr(out)), "ffca_transform")
    return out


def mixture_weights(params: FastFcaParams) -> np.ndarray:
    """w_i(n,f) = max(sum_j v_j Lambda_j,ii, floor) as (N, F, I).  fastfca.py:138-141."""
    lib = _lib.require_gpu()
    c64 = params.P.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    out = np.empty((N, F, I), np.float32 if c64 else np.float64)
    _lib.check(lib.ffca_mixture_weights(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                        _lib.ptr(params.Lam), _lib.ptr(params.v), _lib.ptr(out)),
               "ffca_mixture_weights")
    return out


def e_step_diag(params: FastFcaParams, y_t: np.ndarray) -> TransformedStats:
    """mu_t = (a/w) y_t, phi_t = max(a - a^2/w, 0), entrywise.  fastfca.py:144-157."""
    lib = _lib.require_gpu()
    c64 = params.P.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    yt = _as_c(y_t, c64)
    if yt.shape != (N, F, I):
        raise DimensionMismatch(f"y_t must be (N, F, I) = {(N, F, I)}, got {yt.shape}")
    mu = np.empty((J, N, F, I), yt.dtype)
    phi = np.empty((J, N, F, I), np.float32 if c64 else np.float64)
    _lib.check(lib.ffca_fastfca_estep_yt(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                         _lib.ptr(yt), _lib.ptr(params.Lam), _lib.ptr(params.v),
                                         _lib.ptr(mu), _lib.ptr(phi)), "ffca_fastfca_estep_yt")
    return TransformedStats(mu=mu, phi=phi)


def m_step_diag(stats: TransformedStats, params: FastFcaParams,
                v_floor: float | np.ndarray = 0.0) -> FastFcaParams:
    """v then Lambda from transformed statistics; P untouched.  fastfca.py:160-181."""
    lib = _lib.require_gpu()
    c64 = params.P.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    mu, phi = _as_c(stats.mu, c64), _as_r(stats.phi, c64)
    mode, vfs, vfa = _floor_args(v_floor, J, N, F, c64)
    if mode == _lib.VF_AUTO:
        raise ValueError("m_step_diag needs an explicit v_floor")
    v_new = np.empty((J, N, F), np.float32 if c64 else np.float64)
    lam_new = np.empty((J, F, I), v_new.dtype)
    _lib.check(lib.ffca_mstep_diag(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                   _lib.ptr(mu), _lib.ptr(phi), _lib.ptr(params.Lam), mode, vfs, _lib.ptr(vfa),
                                   _lib.ptr(v_new), _lib.ptr(lam_new)), "ffca_mstep_diag")
    return FastFcaParams(P=params.P, Lam=lam_new, v=v_new)


def fixed_point_update_P(params: FastFcaParams, obs: ObservationTensor, inner_iterations: int = 1,
                         counters: OpCounters | None = None) -> np.ndarray:
    """Column-wise fixed-point map, ``inner_iterations`` times.  fastfca.py:197-237."""
    _check_obs(obs, params)
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    P = _as_c(params.P, c64)
    out = np.empty_like(P)
    _lib.check(lib.ffca_fixed_point_update_P(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                             _lib.ptr(obs.data), _lib.ptr(P), _lib.ptr(_as_r(params.Lam, c64)),
                                             _lib.ptr(_as_r(params.v, c64)), int(inner_iterations),
                                             _lib.ptr(out), None), "ffca_fixed_point_update_P")
    if counters is not None:
        counters.add_inversions((I + 1) * F * int(inner_iterations))
    return out


def log_likelihood(params: FastFcaParams, obs: ObservationTensor) -> float:
    """Observed log likelihood in the transformed basis.  fastfca.py:240-255."""
    _check_obs(obs, params)
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    ll = np.empty(1)
    _lib.check(lib.ffca_fastfca_loglik(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                       _lib.ptr(obs.data), _lib.ptr(_as_c(params.P, c64)),
                                       _lib.ptr(_as_r(params.Lam, c64)), _lib.ptr(_as_r(params.v, c64)),
                                       _lib.ptr(ll), None), "ffca_fastfca_loglik")
    if not np.isfinite(ll[0]):
        raise SingularP("basis transform is singular")
    return float(ll[0])


def _back_transform_device(P: np.ndarray, mu_t, images_layout: bool) -> np.ndarray:
    """back_transform_means with mu_tilde already in device memory (a torch CUDA tensor)."""
    import torch
    lib = _lib.require_gpu()
    c64 = mu_t.dtype == torch.complex64
    J, N, F, I = mu_t.shape
    P = _as_c(P, c64)
    if P.shape != (F, I, I):
        raise DimensionMismatch(f"P must be (F, I, I) = {(F, I, I)}, got {P.shape}")
    dP = torch.from_numpy(np.ascontiguousarray(P)).to(mu_t.device)
    out = torch.empty((J, I, N, F) if images_layout else (J, N, F, I), dtype=mu_t.dtype, device=mu_t.device)
    mu_t = mu_t.contiguous()
    _lib.check(lib.ffca_back_transform(mu_t.device.index, None, _lib.MEM_DEVICE, _code(c64), 1, I, J, N, F,
                                       dP.data_ptr(), mu_t.data_ptr(), out.data_ptr(), 1 if images_layout else 0,
                                       None), "ffca_back_transform")
    return out.cpu().numpy()


def back_transform_means(P: np.ndarray, mu_t: np.ndarray, images_layout: bool = False) -> np.ndarray:
    """Solve P^H mu = mu_tilde per bin; (J, N, F, I) in and out.  fastfca.py:258-273."""
    if hasattr(mu_t, "is_cuda") and mu_t.is_cuda:
        return _back_transform_device(P, mu_t, images_layout)
    lib = _lib.require_gpu()
    c64 = np.asarray(mu_t).dtype == np.complex64
    mu_t = _as_c(mu_t, c64)
    P = _as_c(P, c64)
    J, N, F, I = mu_t.shape
    if P.shape != (F, I, I):
        raise DimensionMismatch(f"P must be (F, I, I) = {(F, I, I)}, got {P.shape}")
    out = np.empty((J, I, N, F) if images_layout else (J, N, F, I), mu_t.dtype)
    _lib.check(lib.ffca_back_transform(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                       _lib.ptr(P), _lib.ptr(mu_t), _lib.ptr(out), 1 if images_layout else 0,
                                       None), "ffca_back_transform")
    return out


def images_from_state(obs: ObservationTensor, params: FastFcaParams) -> np.ndarray:
    """Fused stats refresh + Wiener back-solve: images (J, I, N, F) from the final state."""
    lib = _lib.require_gpu()
    c64 = obs.data.dtype == np.complex64
    J, N, F = params.v.shape
    I = params.order
    out = np.empty((J, I, N, F), obs.data.dtype)
    _lib.check(lib.ffca_fastfca_images(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                       _lib.ptr(obs.data), _lib.ptr(_as_c(params.P, c64)),
                                       _lib.ptr(_as_r(params.Lam, c64)), _lib.ptr(_as_r(params.v, c64)),
                                       _lib.ptr(out), None), "ffca_fastfca_images")
    return out


def back_transform_stats(params: FastFcaParams, stats: TransformedStats):
    """(mu (J,N,F,I), phi (J,N,F,I,I)) in the microphone basis.  fastfca.py:276-287."""
    lib = _lib.require_gpu()
    c64 = params.P.dtype == np.complex64
    mu = back_transform_means(params.P, stats.mu)
    phi_t = _as_r(stats.phi, c64)
    J, N, F, I = phi_t.shape
    out = np.empty((J, N, F, I, I), np.complex64 if c64 else np.complex128)
    _lib.check(lib.ffca_back_transform_phi(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, N, F,
                                           _lib.ptr(_as_c(params.P, c64)), _lib.ptr(phi_t), _lib.ptr(out), None),
               "ffca_back_transform_phi")
    return mu, out


def reconstruct_spatial_covariances(params: FastFcaParams) -> np.ndarray:
    """All S_j(f) = P^{-H} Lambda_j P^{-1}, (J, F, I, I), hermitized.  fastfca.py:119-126."""
    lib = _lib.require_gpu()
    c64 = params.P.dtype == np.complex64
    J, F, I = params.Lam.shape
    S = np.empty((J, F, I, I), params.P.dtype)
    _lib.check(lib.ffca_reconstruct_covariances(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, F,
                                                _lib.ptr(params.P), _lib.ptr(params.Lam), _lib.ptr(S), None),
               "ffca_reconstruct_covariances")
    return S


def reconstruct_spatial_covariance(params: FastFcaParams, j: int, f: int) -> np.ndarray:
    """S_j(f) for one source and bin.  fastfca.py:129-135."""
    one = FastFcaParams(P=params.P[f:f + 1], Lam=params.Lam[j:j + 1, f:f + 1], v=params.v[j:j + 1, :, f:f + 1])
    return reconstruct_spatial_covariances(one)[0, 0]


def params_from_covariances(S_hat: np.ndarray, v: np.ndarray) -> FastFcaParams:
    """Whitening initialization from spatial covariance estimates.  fastfca.py:290-309."""
    lib = _lib.require_gpu()
    S_hat = np.asarray(S_hat)
    c64 = S_hat.dtype == np.complex64
    S_hat = _as_c(S_hat, c64)
    J, F, I, _ = S_hat.shape
    P = np.empty((F, I, I), S_hat.dtype)
    lam = np.empty((J, F, I), np.float32 if c64 else np.float64)
    _lib.check(lib.ffca_params_from_covariances(_lib.device(), None, _lib.MEM_HOST, _code(c64), 1, I, J, F,
                                                _lib.ptr(S_hat), _lib.ptr(P), _lib.ptr(lam), None),
               "ffca_params_from_covariances")
    return FastFcaParams(P=P, Lam=lam, v=_as_r(v, c64))
