"""Seeded synthetic mixtures for the BASELINE.json configurations.

The reference measures on synthetic scenes (no public dataset; SURVEY.md
§8(d)).  This generator follows BASELINE.json's description with a fixed draw
order per mixture (rng = numpy.random.default_rng(seed)):

  1. A (J, F, I, I) ~ CN(0, 1)            R_j(f) = A A^H + 0.01 I
  2. W (J, F, r), H (J, r, N) ~ Gamma(0.5, 1);  v_j = (W_j H_j)^T -> (J, N, F)
  3. (sparse only) per-source mask U(0,1) < frac  -> v = 0 there
  4. z (J, N, F, I) ~ CN(0, I);  c_j = sqrt(v_j) chol(R_j) z;  y = sum_j c_j  (I, N, F)
  5. init: P = I, lam = 1, v0 = mean_i |y_i|^2 / J * U(0.9, 1.1)

Everything is generated in float64 and cast at the end for complex64 configs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SQRT_HALF = np.sqrt(0.5)


@dataclass(frozen=True)
class Config:
    name: str
    I: int
    J: int
    F: int
    N: int
    iterations: int
    dtype: str  # "c128" | "c64"
    mixtures: int = 1
    rank: int = 4
    zero_frac: float = 0.0
    algorithm: str = "fastfca"

    @property
    def points(self) -> int:
        return self.mixtures * self.N * self.F

    @property
    def point_iterations(self) -> int:
        return self.points * self.iterations


CONFIGS = {
    0: Config("config0: FastFCA-AS I=J=3 F=513 N=626 c128 20it", 3, 3, 513, 626, 20, "c128"),
    1: Config("config1: FCA I=J=3 F=513 N=626 c128 20it", 3, 3, 513, 626, 20, "c128", algorithm="fca"),
    2: Config("config2: FastFCA-AS I=J=4 F=1025 N=9375 c64 30it", 4, 4, 1025, 9375, 30, "c64", rank=8),
    3: Config("config3: FastFCA-AS 256 x (I=J=3 F=513 N=626) c64 20it", 3, 3, 513, 626, 20, "c64",
              mixtures=256),
    4: Config("config4: FastFCA-AS I=8 J=6 F=2049 N=4000 c64 20it 10% zero cells", 8, 6, 2049, 4000, 20,
              "c64", rank=8, zero_frac=0.1),
}


def _cn(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * SQRT_HALF


def mixture(seed: int, I: int, J: int, F: int, N: int, rank: int = 4, zero_frac: float = 0.0):
    """One seeded mixture.  Returns (y (I,N,F) c128, P0, lam0, v0, v_true)."""
    rng = np.random.default_rng(seed)
    A = _cn(rng, (J, F, I, I))
    R = A @ np.conj(np.swapaxes(A, -1, -2)) + 0.01 * np.eye(I)
    W = rng.gamma(0.5, 1.0, (J, F, rank))
    H = rng.gamma(0.5, 1.0, (J, rank, N))
    v_true = np.ascontiguousarray(np.swapaxes(W @ H, 1, 2))  # (J, N, F)
    if zero_frac > 0.0:
        v_true[rng.random((J, N, F)) < zero_frac] = 0.0
    L = np.linalg.cholesky(R)  # (J, F, I, I)
    z = _cn(rng, (J, N, F, I))
    c = np.sqrt(v_true)[..., None] * np.einsum("jfab,jnfb->jnfa", L, z)
    y = np.ascontiguousarray(np.transpose(c.sum(axis=0), (2, 0, 1)))  # (I, N, F)
    P0 = np.broadcast_to(np.eye(I, dtype=np.complex128), (F, I, I)).copy()
    lam0 = np.ones((J, F, I))
    power = (y.real ** 2 + y.imag ** 2).mean(axis=0)  # (N, F)
    v0 = (power / J)[None] * rng.uniform(0.9, 1.1, (J, N, F))
    return y, P0, lam0, v0, v_true


def make(cfg: Config, seed0: int = 0, mixtures: int | None = None):
    """Stacked inputs for a config: y (U,I,N,F), P (U,F,I,I), lam (U,J,F,I), v (U,J,N,F)."""
    U = cfg.mixtures if mixtures is None else mixtures
    cdt = np.complex64 if cfg.dtype == "c64" else np.complex128
    rdt = np.float32 if cfg.dtype == "c64" else np.float64
    y = np.empty((U, cfg.I, cfg.N, cfg.F), cdt)
    P = np.empty((U, cfg.F, cfg.I, cfg.I), cdt)
    lam = np.empty((U, cfg.J, cfg.F, cfg.I), rdt)
    v = np.empty((U, cfg.J, cfg.N, cfg.F), rdt)
    for u in range(U):
        yu, Pu, lu, vu, _ = mixture(seed0 + u, cfg.I, cfg.J, cfg.F, cfg.N, cfg.rank, cfg.zero_frac)
        y[u], P[u], lam[u], v[u] = yu, Pu, lu, vu
    return y, P, lam, v


def make_torch_range(cfg: Config, seed0: int, u0: int, u1: int, device):
    """Mixtures u0..u1-1 of a config, mixture u drawn from its own torch generator (seed0 + u).

    Every mixture depends only on its index, so shards of the mixture axis generated on
    different ranks (bench.py --gpus N) are exactly the corresponding slices of the
    single-GPU batch.  Same recipe and layouts as ``make_torch``.
    """
    import torch

    parts = [make_torch(cfg, seed0 + u, 1, device) for u in range(u0, u1)]
    if not parts:
        cdt = torch.complex64 if cfg.dtype == "c64" else torch.complex128
        rdt = torch.float32 if cfg.dtype == "c64" else torch.float64
        I, J, F, N = cfg.I, cfg.J, cfg.F, cfg.N
        return (torch.empty((0, I, N, F), dtype=cdt, device=device), torch.empty((0, F, I, I), dtype=cdt, device=device),
                torch.empty((0, J, F, I), dtype=rdt, device=device), torch.empty((0, J, N, F), dtype=rdt, device=device))
    out = tuple(torch.cat([p[k] for p in parts]) for k in range(4))
    del parts
    return out


def make_torch(cfg: Config, seed: int, mixtures: int, device, chunk: int = 32):
    """The same recipe drawn with torch on the GPU (fast for the 256-mixture config).

    Used by bench.py only; the draws differ from ``make`` (different RNG) but
    follow the identical distributions.  Returns device tensors in the
    reference layouts with a leading mixture axis, cast to the config dtype.
    """
    import torch

    I, J, F, N, r = cfg.I, cfg.J, cfg.F, cfg.N, cfg.rank
    cdt = torch.complex64 if cfg.dtype == "c64" else torch.complex128
    rdt = torch.float32 if cfg.dtype == "c64" else torch.float64
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    y = torch.empty((mixtures, I, N, F), dtype=cdt, device=device)
    v0 = torch.empty((mixtures, J, N, F), dtype=rdt, device=device)
    eye = torch.eye(I, dtype=torch.complex128, device=device)

    def cn(shape):
        re = torch.randn(shape, dtype=torch.float64, device=device, generator=gen)
        im = torch.randn(shape, dtype=torch.float64, device=device, generator=gen)
        return torch.complex(re, im) * SQRT_HALF

    def gamma(shape):
        # Gamma(shape 1/2, scale 1) is exactly Z^2 / 2 with Z ~ N(0, 1)
        z = torch.randn(shape, dtype=torch.float64, device=device, generator=gen)
        return 0.5 * z * z

    for u0 in range(0, mixtures, chunk):
        U = min(chunk, mixtures - u0)
        A = cn((U, J, F, I, I))
        R = A @ A.conj().transpose(-1, -2) + 0.01 * eye
        L = torch.linalg.cholesky(R)
        W = gamma((U, J, F, r))
        H = gamma((U, J, r, N))
        vt = (W @ H).transpose(-1, -2).contiguous()  # (U, J, N, F)
        if cfg.zero_frac > 0:
            mask = torch.rand((U, J, N, F), dtype=torch.float64, device=device, generator=gen) < cfg.zero_frac
            vt = vt.masked_fill(mask, 0.0)
        yy = torch.zeros((U, N, F, I), dtype=torch.complex128, device=device)
        for j in range(J):
            z = cn((U, N, F, I))
            yy += torch.sqrt(vt[:, j])[..., None] * torch.einsum("ufab,unfb->unfa", L[:, j], z)
        yi = yy.permute(0, 3, 1, 2).contiguous()  # (U, I, N, F)
        y[u0:u0 + U] = yi.to(cdt)
        power = (yi.real ** 2 + yi.imag ** 2).mean(dim=1)  # (U, N, F)
        jit = 0.9 + 0.2 * torch.rand((U, J, N, F), dtype=torch.float64, device=device, generator=gen)
        v0[u0:u0 + U] = ((power / J)[:, None] * jit).to(rdt)
        del A, R, L, W, H, vt, yy, yi
    P0 = torch.eye(I, dtype=cdt, device=device).expand(mixtures, F, I, I).contiguous()
    lam0 = torch.ones((mixtures, J, F, I), dtype=rdt, device=device)
    return y, P0, lam0, v0
