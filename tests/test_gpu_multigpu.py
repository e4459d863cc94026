"""World-size-2 sharding through the DEVICE path: two ranks on one GPU, gloo for the exchange.

Each rank runs its shard with the CUDA kernels (run_fastfca_batch via run_fastfca_sharded's
default compute) and the final gather goes through torch.distributed; the gathered result must
be bitwise the unsharded single-call result (SURVEY.md §8(e) determinism).  The complex128 case
uses 2 config-0 mixtures: unsharded, the 1026 bins run 2-bin CTAs; an F-block shard (514 bins)
runs 1-bin CTAs -- the plan-independent reduction keeps the results bitwise equal.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _inputs(dt):
    from paper_1805_09498_b200.workloads import mixture

    if dt == "c128":
        parts = [mixture(700 + u, 3, 3, 513, 626) for u in range(2)]
    else:
        parts = [mixture(710 + u, 3, 3, 37, 200) for u in range(3)]
    arrs = [np.stack([p[k] for p in parts]) for k in range(4)]
    if dt == "c64":
        arrs = [a.astype(np.complex64) if np.iscomplexobj(a) else a.astype(np.float32) for a in arrs]
    return tuple(arrs)


def _worker(rank, world, port, mode, dt, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_09498_b200 import _lib
        from paper_1805_09498_b200.multigpu import run_fastfca_sharded

        _lib.set_device(0)
        y, P0, lam0, v0 = _inputs(dt)
        P, lam, v, ll = run_fastfca_sharded(y, P0, lam0, v0, iterations=4, mode=mode, record_likelihood=True,
                                            device="cpu")
        q.put((rank, P, lam, v, ll))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("dt", ["c128", "c64"])
@pytest.mark.parametrize("mode", ["mixtures", "bins"])
def test_world2_device_shards_bitwise_unsharded(mode, dt):
    from paper_1805_09498_b200 import fastfca

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, dt, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y, P0, lam0, v0 = _inputs(dt)
    os.environ["FFCA_NO_PIPELINE"] = "1"
    try:
        P, lam, v, ll = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=4, record_likelihood=True)
    finally:
        os.environ.pop("FFCA_NO_PIPELINE")
    for _, Pg, lg, vg, llg in res:
        assert np.array_equal(Pg, P) and np.array_equal(lg, lam) and np.array_equal(vg, v)
        if mode == "mixtures":
            assert np.array_equal(llg, ll)
        else:  # per-F-block partial sums added across ranks: a different summation order
            assert np.allclose(llg, ll, rtol=1e-12 if dt == "c128" else 1e-6, atol=0)


def _nccl_worker(port, q):
    # one rank on the NCCL backend: the collectives the multi-GPU paths issue (all_gather of int64 sizes
    # and of complex shards viewed as real, all_reduce, gather of padded device buffers) run for real
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_1805_09498_b200 import _lib
        from paper_1805_09498_b200.multigpu import run_fastfca_sharded

        _lib.set_device(0)
        y, P0, lam0, v0 = _inputs("c64")
        out = run_fastfca_sharded(y, P0, lam0, v0, iterations=3, mode="bins", record_likelihood=True,
                                  device="cuda:0")
        # bench.py's Dist.gather_ms pattern: gather a padded device buffer to rank 0
        src = torch.arange(10, dtype=torch.float32, device="cuda:0")
        outs = [torch.empty_like(src)]
        dist.gather(src, outs, dst=0)
        t = torch.tensor([3.0], dtype=torch.float64, device="cuda:0")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((out, outs[0].cpu().numpy(), float(t.item()), dist.get_backend()))
    finally:
        dist.destroy_process_group()


def test_nccl_backend_world1_collectives():
    from paper_1805_09498_b200 import fastfca

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    (P, lam, v, ll), g, mx, backend = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0 and backend == "nccl"
    assert np.array_equal(g, np.arange(10, dtype=np.float32)) and mx == 3.0
    y, P0, lam0, v0 = _inputs("c64")
    P1, lam1, v1, ll1 = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=3, record_likelihood=True)
    assert np.array_equal(P, P1) and np.array_equal(lam, lam1) and np.array_equal(v, v1)
    assert np.allclose(ll, ll1, rtol=1e-6, atol=0)
