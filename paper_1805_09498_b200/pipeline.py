"""Device-resident separation pipeline: audio in, separated source images out.

Mirrors the reference's in-memory pipeline ``cli.separate_once``
(cli.py:217-260) and the per-trial body of ``cli.cmd_bench`` (cli.py:292-340):

    analyze -> initialise (oracle / diffuse) -> estimator (fastfca / fca)
            -> Wiener images -> overlap-add synthesis -> SDR per source

with every stage a call into libffca_b200.so on device memory (torch tensors
are only the allocator): the mixture and the reference images cross PCIe once
on the way in, the images / audio / parameters once on the way out, and no
intermediate (observations, covariances, P, Lambda, v, images) ever visits the
host.  The estimator is timed on the device with CUDA events, the scope the
reference times with ``time.perf_counter`` around ``_run_estimator``
(cli.py:226-229), giving the same real-time factor definition
(evalkit.rtf_value).  File I/O, CSV reports and manifests (cli.py:262-389)
stay out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DimensionMismatch, TooShort
from .evalkit import OpCounters, sdr_from_energies
from .fastfca import FastFcaParams
from .fca import FcaParams
from .scene import _perturbations
from .stft import StftConfig, _as_channel_matrix
from .wiener import SeparatedImages


@dataclass
class PipelineConfig:
    """The estimator / filterbank fields of the reference's ``RunConfig`` (cli.py:41-80)."""

    algorithm: str = "fastfca"
    iterations: int = 20
    inner_k: int = 1
    init: str = "oracle"
    seed: int = 0
    sources: int = 3
    frame_length: int = 1024
    frame_shift: int = 512
    sample_rate: int = 16000
    complex64: bool = False  # extension: run the fp32 kernels end to end

    def __post_init__(self):
        # cli.py:68-76
        if self.iterations < 0:
            raise ValueError("iterations must be >= 0")
        if self.inner_k < 1:
            raise ValueError("inner_k must be >= 1")
        if self.algorithm not in ("fca", "fastfca"):
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.init not in ("oracle", "diffuse"):
            raise ValueError(f"unknown init {self.init!r}")

    def stft_config(self) -> StftConfig:
        return StftConfig(frame_length=self.frame_length, frame_shift=self.frame_shift,
                          sample_rate=self.sample_rate)


@dataclass
class PipelineResult:
    images: SeparatedImages  # stft (J, I, N, F) and audio (J, I, S_out)
    params: object  # FastFcaParams or FcaParams after the run
    counters: OpCounters
    estimator_seconds: float  # device time of the estimator call alone
    duration: float  # mixture length in seconds
    sdr_per_source: list = field(default_factory=list)

    @property
    def rtf(self) -> float:
        return self.estimator_seconds / self.duration

    def report(self) -> dict:
        """The fields of the reference's per-run manifest summary (cli.py:243-258)."""
        return {"rtf": self.rtf, "sdr_per_source": list(self.sdr_per_source),
                "sdr_mean": float(np.mean(self.sdr_per_source)) if self.sdr_per_source else float("nan"),
                "counters": self.counters.as_dict()}


def separate_once(cfg: PipelineConfig, mixture, references=None) -> PipelineResult:
    """Full separation on in-memory audio, device-resident end to end (cli.py:217-260).

    ``mixture`` is (I, S) (or a list of channels); ``references`` the (J, I, S)
    source images (needed for ``init="oracle"``, optional otherwise; when
    given the SDR per source is computed).
    """
    import torch

    lib = _lib.require_gpu()
    di = _lib.device()
    dev = torch.device("cuda", di)
    sp = torch.cuda.current_stream(dev).cuda_stream
    code = _lib.C64 if cfg.complex64 else _lib.C128
    rdt, cdt = (torch.float32, torch.complex64) if cfg.complex64 else (torch.float64, torch.complex128)
    ndt_c = np.complex64 if cfg.complex64 else np.complex128
    MEM = _lib.MEM_DEVICE

    def P(t):
        return None if t is None else t.data_ptr()

    mix = _as_channel_matrix(mixture)
    I, S = mix.shape
    L, sh = cfg.frame_length, cfg.frame_shift
    if S < L:
        raise TooShort(f"signal has {S} samples, frame needs {L}")
    N, F = (S - L) // sh + 1, L // 2
    refs = None
    if references is not None:
        refs = np.asarray(references, dtype=np.float64)
        if refs.ndim != 3 or refs.shape[1:] != (I, S):
            raise DimensionMismatch(f"references {refs.shape} do not match the mixture ({I}, {S})")
    if cfg.init == "oracle" and refs is None:
        raise ValueError("oracle init needs reference source images")  # cli.py:195-197
    J = refs.shape[0] if cfg.init == "oracle" else cfg.sources

    # analysis of the mixture and (one batched call) of all J*I reference channels
    mix_d = torch.from_numpy(mix).to(dev, rdt)
    y = torch.empty((I, N, F), dtype=cdt, device=dev)
    _lib.check(lib.ffca_stft_analyze(di, sp, MEM, code, I, S, L, sh, P(mix_d), P(y)), "ffca_stft_analyze")
    refs_d = X = None
    if refs is not None:
        Jr = refs.shape[0]
        refs_d = torch.from_numpy(refs.reshape(Jr * I, S)).to(dev, rdt)
        X = torch.empty((Jr, I, N, F), dtype=cdt, device=dev)
        _lib.check(lib.ffca_stft_analyze(di, sp, MEM, code, Jr * I, S, L, sh, P(refs_d), P(X)), "ffca_stft_analyze")

    # initial covariances (scene.py:207-247)
    floor = torch.empty((1, F), dtype=torch.float64, device=dev)
    _lib.check(lib.ffca_power_floor(di, sp, MEM, code, 1, I, N, F, P(y), P(floor)), "ffca_power_floor")
    S_hat = torch.empty((J, F, I, I), dtype=cdt, device=dev)
    v_hat = torch.empty((J, N, F), dtype=rdt, device=dev)
    if cfg.init == "oracle":
        _lib.check(lib.ffca_init_covariances(di, sp, MEM, code, 0, 1, I, J, N, F, P(X), P(floor), None, P(S_hat),
                                             P(v_hat)), "ffca_init_covariances")
    else:
        W = torch.from_numpy(_perturbations(I, J, cfg.seed).astype(ndt_c)).to(dev)
        _lib.check(lib.ffca_init_covariances(di, sp, MEM, code, 1, 1, I, J, N, F, P(y), P(floor), P(W), P(S_hat),
                                             P(v_hat)), "ffca_init_covariances")

    # estimator (timed alone, as cli.py:226-229) + Wiener images
    images = torch.empty((J, I, N, F), dtype=cdt, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    counters = OpCounters()
    it = int(cfg.iterations)
    if cfg.algorithm == "fastfca":
        P0 = torch.empty((F, I, I), dtype=cdt, device=dev)
        lam0 = torch.empty((J, F, I), dtype=rdt, device=dev)
        _lib.check(lib.ffca_params_from_covariances(di, sp, MEM, code, 1, I, J, F, P(S_hat), P(P0), P(lam0), None),
                   "ffca_params_from_covariances")
        Pm, lam, v = torch.empty_like(P0), torch.empty_like(lam0), torch.empty_like(v_hat)
        e0.record()
        _lib.check(lib.ffca_fastfca_run(di, sp, MEM, code, 1, I, J, N, F, P(y), P(P0), P(lam0), P(v_hat),
                                        _lib.VF_AUTO, 0.0, None, it, int(cfg.inner_k), 0, P(Pm), P(lam), P(v),
                                        None, None, None), "ffca_fastfca_run")
        e1.record()
        _lib.check(lib.ffca_fastfca_images(di, sp, MEM, code, 1, I, J, N, F, P(y), P(Pm), P(lam), P(v), P(images),
                                           None), "ffca_fastfca_images")
        counters.add_inversions(it * (I + 1) * F * int(cfg.inner_k))
        out_params = (Pm, lam, v)
    else:
        Sm, v = torch.empty_like(S_hat), torch.empty_like(v_hat)
        e0.record()
        _lib.check(lib.ffca_fca_run(di, sp, MEM, code, 1, I, J, N, F, P(y), P(S_hat), P(v_hat), _lib.VF_AUTO, 0.0,
                                    None, it, 0, P(Sm), P(v), None, None, None, None), "ffca_fca_run")
        e1.record()
        _lib.check(lib.ffca_fca_estep(di, sp, MEM, code, 1, I, J, N, F, P(y), P(Sm), P(v), P(images), None, 1,
                                      None), "ffca_fca_estep")
        counters.add_inversions(it * (J + N) * F)
        counters.add_matmuls(it * 2 * J * N * F)
        out_params = (Sm, v)

    # overlap-add of all J*I image channels in one call, then SDR energies
    S_out = (N - 1) * sh + L
    audio = torch.empty((J, I, S_out), dtype=rdt, device=dev)
    _lib.check(lib.ffca_stft_synthesize(di, sp, MEM, code, J * I, N, L, sh, P(images), P(audio)),
               "ffca_stft_synthesize")
    sdrs = []
    if refs_d is not None and refs.shape[0] == J:
        en = torch.empty((J, 2), dtype=torch.float64, device=dev)
        _lib.check(lib.ffca_sdr_energies(di, sp, MEM, code, J, I, S, S_out, P(refs_d), P(audio), P(en)),
                   "ffca_sdr_energies")
        sdrs = sdr_from_energies(en.cpu().numpy())
    torch.cuda.synchronize(dev)
    est_s = e0.elapsed_time(e1) / 1e3

    host = [t.cpu().numpy() for t in out_params]
    params = FastFcaParams(P=host[0], Lam=host[1], v=host[2]) if cfg.algorithm == "fastfca" else \
        FcaParams(S=host[0], v=host[1])
    sep = SeparatedImages(stft=images.cpu().numpy(), audio=audio.cpu().numpy())
    return PipelineResult(images=sep, params=params, counters=counters, estimator_seconds=est_s,
                          duration=S / cfg.sample_rate, sdr_per_source=sdrs)
