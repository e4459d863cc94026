"""Multi-GPU driver: shard independent bins / mixtures, one process per GPU.

Frequency bins are independent for the whole FastFCA-AS run (every reduction
is over frames at a fixed bin, fastfca.py:338-340,357-358), so
the work partitions with **no data-path collective**: each rank runs the
single-GPU path on its shard and the only exchange is the final gather of
the estimates.

Shard modes:
  "mixtures"  contiguous blocks of the mixture axis (config 3, batched utterances)
  "bins"      contiguous F-blocks of every mixture (configs 2 and 4, long recordings)
Shard boundaries are fixed (`shard_range`), so results are bitwise equal to
the single-GPU run.
"""

from __future__ import annotations

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `total` items for `rank` of `world` (sizes differ by <= 1)."""
    return total * rank // world, total * (rank + 1) // world


def _device_compute(y, P0, lam0, v0, iterations, inner_iterations, v_floor, record_likelihood=False):
    from .fastfca import run_fastfca_batch

    P, lam, v, ll = run_fastfca_batch(y, P0, lam0, v0, iterations=iterations,
                                      inner_iterations=inner_iterations, v_floor=v_floor,
                                      record_likelihood=record_likelihood)
    return (P, lam, v, ll) if record_likelihood else (P, lam, v)


def _all_gather_concat(arr: np.ndarray, axis: int, group, world: int, device):
    """All-gather numpy shards (possibly unequal along `axis`) and concatenate them."""
    import torch
    import torch.distributed as dist

    sizes = torch.tensor([arr.shape[axis]], dtype=torch.int64, device=device)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [int(s.item()) for s in all_sizes]
    mx = max(all_sizes)
    pad = [(0, 0)] * arr.ndim
    pad[axis] = (0, mx - arr.shape[axis])
    padded = np.ascontiguousarray(np.pad(arr, pad))
    if np.iscomplexobj(padded):
        t = torch.from_numpy(padded.view(padded.real.dtype)).to(device)
    else:
        t = torch.from_numpy(padded).to(device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    parts = []
    for o, n in zip(outs, all_sizes):
        a = o.cpu().numpy()
        if np.iscomplexobj(arr):
            a = a.view(arr.dtype)
        parts.append(np.take(a, np.arange(n), axis=axis))
    return np.concatenate(parts, axis=axis)


def run_fastfca_sharded(y, P0, lam0, v0, iterations=20, inner_iterations=1, v_floor=None, mode="mixtures",
                        group=None, compute=None, device=None, record_likelihood=False):
    """Run the batched estimator with this rank's shard and all-gather the result.

    y (U, I, N, F), P0 (U, F, I, I), lam0 (U, J, F, I), v0 (U, J, N, F) are the
    full inputs on every rank (host numpy).  `compute` defaults to the device
    path (`fastfca.run_fastfca_batch`); it has the signature
    compute(y, P0, lam0, v0, iterations, inner_iterations, v_floor[, record_likelihood])
    -> (P, lam, v[, ll]).  Returns (P, lam, v) for all mixtures / bins on every
    rank, plus the per-mixture log-likelihood history (U, 1+2T) when
    ``record_likelihood``: concatenated over mixture shards, or summed over
    F-block shards (each block's partial already carries its share of the
    -N F I ln(pi) constant) with one all-reduce.
    """
    import torch.distributed as dist

    compute = compute or _device_compute
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if device is None:
        device = "cpu" if dist.get_backend(group) == "gloo" else f"cuda:{rank % max(1, _ndev())}"
    U, I, N, F = y.shape
    if mode == "mixtures":
        lo, hi = shard_range(U, rank, world)
        vf = v_floor if (v_floor is None or np.ndim(v_floor) == 0) else np.asarray(v_floor)[lo:hi]
        res = compute(y[lo:hi], P0[lo:hi], lam0[lo:hi], v0[lo:hi], iterations, inner_iterations, vf,
                      *((True,) if record_likelihood else ()))
        axes = (0, 0, 0)
    elif mode == "bins":
        lo, hi = shard_range(F, rank, world)
        vf = v_floor if (v_floor is None or np.ndim(v_floor) == 0) else np.asarray(v_floor)[..., lo:hi]
        res = compute(np.ascontiguousarray(y[..., lo:hi]), np.ascontiguousarray(P0[:, lo:hi]),
                      np.ascontiguousarray(lam0[:, :, lo:hi]), np.ascontiguousarray(v0[..., lo:hi]),
                      iterations, inner_iterations, vf, *((True,) if record_likelihood else ()))
        axes = (1, 2, 3)
    else:
        raise ValueError(f"unknown shard mode {mode!r}")
    out = tuple(_all_gather_concat(np.asarray(a), ax, group, world, device) for a, ax in zip(res[:3], axes))
    if not record_likelihood:
        return out
    ll = np.asarray(res[3], dtype=np.float64)
    if mode == "mixtures":
        ll = _all_gather_concat(ll, 0, group, world, device)
    else:
        import torch

        t = torch.from_numpy(np.ascontiguousarray(ll)).to(device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        ll = t.cpu().numpy()
    return out + (ll,)


def _ndev() -> int:
    try:
        from . import _lib

        return max(1, _lib.load().ffca_device_count())
    except Exception:  # noqa: BLE001 -- only used to pick a device index
        return 1
