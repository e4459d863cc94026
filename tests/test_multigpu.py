"""World-size-2 sharding on CPU (gloo): shards + final gather == the unsharded run.

The per-shard compute is the CPU oracle (no GPU here); the product path uses
the device kernels with exactly the same shard boundaries.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_09498_b200.multigpu import run_fastfca_sharded, shard_range


def _oracle_compute(y, P0, lam0, v0, iterations, inner, v_floor, record=False):
    from oracle import fastfca_ref

    outs = [fastfca_ref.run_fastfca(y[u], P0[u], lam0[u], v0[u], iterations=iterations,
                                    inner_iterations=inner, stats=False, record_likelihood=record)
            for u in range(y.shape[0])]
    res = (np.stack([o.P for o in outs]), np.stack([o.lam for o in outs]), np.stack([o.v for o in outs]))
    if record:
        ll = np.stack([np.array([o.loglik_init] + o.loglik_after_em + o.loglik_after_p) for o in outs])
        return res + (ll,)
    return res


def _inputs():
    from paper_1805_09498_b200.workloads import mixture

    parts = [mixture(40 + u, 3, 2, 9, 30) for u in range(3)]
    return tuple(np.stack([p[k] for p in parts]) for k in range(4))


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        y, P0, lam0, v0 = _inputs()
        P, lam, v, ll = run_fastfca_sharded(y, P0, lam0, v0, iterations=3, mode=mode, compute=_oracle_compute,
                                            record_likelihood=True)
        q.put((rank, P, lam, v, ll))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_cover_exactly():
    for total in (1, 7, 256, 1025):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(h - l for l, h in ranges) - min(h - l for l, h in ranges) <= 1


@pytest.mark.parametrize("mode", ["mixtures", "bins"])
def test_gloo_world2_matches_unsharded(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y, P0, lam0, v0 = _inputs()
    ref = _oracle_compute(y, P0, lam0, v0, 3, 1, None, True)
    for _, P, lam, v, ll in res:
        for got, want in zip((P, lam, v, ll), ref):
            assert got.shape == want.shape
            assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
