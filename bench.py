#!/usr/bin/env python
"""Benchmark of the FastFCA-AS estimation loop on B200 (BASELINE.json metric).

Workload: BASELINE.json config 3 -- 256 independent mixtures, each I=J=3
microphones/sources, F=513 bins, N=626 frames, complex64, 20 iterations
(the metric's I=3,J=3 case at a size that exercises the whole GPU; config 0
is the single-mixture CPU-runnable case).  Mixtures are independent, so the
path partitions with no data-path collective: every rank runs its own
256-mixture batch (weak scaling); `value` is the units all
ranks processed / the max-over-ranks time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one call of the estimator over all of this rank's mixtures, every
iteration executed (v, lambda and P updates; power floor computed on device).
`value` times that call with inputs resident in HBM (CUDA events on the
launch stream, max over ranks); `e2e` times the public API with pinned host
inputs (H2D + loop + D2H of P, lambda, v) on the same stream.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FastFCA-AS TF-point·iterations/sec (I=3,J=3); achieved HBM GB/s vs peak"
UNIT = "TF-point*iterations/s"
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--mixtures", type=int, default=None, help="override the mixture count (testing)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-mixtures", type=int, default=None)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference; bench.py is one of the places that may run oracle/)
# ---------------------------------------------------------------------------


def _cpu_gen(args):
    from paper_1805_09498_b200.workloads import mixture
    seed, I, J, F, N, rank, zf = args
    y, P0, lam0, v0, _ = mixture(seed, I, J, F, N, rank, zf)
    return y, P0, lam0, v0


def _cpu_run(args):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import fastfca_ref
    y, P0, lam0, v0, iters = args
    t0 = time.perf_counter()
    fastfca_ref.run_fastfca(y, P0, lam0, v0, iterations=iters, stats=True)
    return time.perf_counter() - t0


def cpu_measure(cfg, n_mix, pool):
    """Throughput of the oracle port over n_mix mixtures spread on all host cores (wall clock)."""
    inputs = pool.map(_cpu_gen, [(9000 + k, cfg.I, cfg.J, cfg.F, cfg.N, cfg.rank, cfg.zero_frac)
                                 for k in range(n_mix)])
    t0 = time.perf_counter()
    pool.map(_cpu_run, [(y, P, l, v, cfg.iterations) for (y, P, l, v) in inputs], chunksize=1)
    wall = time.perf_counter() - t0
    return n_mix * cfg.N * cfg.F * cfg.iterations / wall, wall


def cpu_pool():
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    cores = len(os.sched_getaffinity(0))
    return mp.get_context("spawn").Pool(cores), cores


def cpu_info():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(device_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    path = os.path.join(ROOT, "profiles", "loop_kernel_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d
    except (OSError, ValueError):
        return None


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1805_09498_b200 import _lib
    from paper_1805_09498_b200.fastfca import run_fastfca_batch
    from paper_1805_09498_b200.workloads import CONFIGS, make_torch

    cfg = CONFIGS[args.config]
    U = args.mixtures or cfg.mixtures  # per rank (weak scaling)
    total = U * world
    u0 = U * rank
    dev = torch.device("cuda", local_rank % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    _lib.set_device(dev.index)
    lib = _lib.require_gpu()
    code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
    I, J, N, F, T = cfg.I, cfg.J, cfg.N, cfg.F, cfg.iterations

    y, P0, lam0, v0 = make_torch(cfg, seed=1234 + u0, mixtures=U, device=dev)
    P = torch.empty_like(P0)
    lam = torch.empty_like(lam0)
    v = torch.empty_like(v0)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def step():
        rc = lib.ffca_fastfca_run(dev.index, sptr, _lib.MEM_DEVICE, code, U, I, J, N, F, y.data_ptr(),
                                  P0.data_ptr(), lam0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0, None, T, 1,
                                  0, P.data_ptr(), lam.data_ptr(), v.data_ptr(), None, None, None)
        _lib.check(rc, "ffca_fastfca_run")

    lib.ffca_set_kernel_timing(1)
    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev.index)
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kernel_ms, launches = [], 0
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        kernel_ms.append(float(lib.ffca_last_kernel_ms()))
        launches += int(lib.ffca_last_launch_count())
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    tdev = dev if dist.is_initialized() and dist.get_backend() == "nccl" else "cpu"
    t_ms = torch.tensor([elapsed_ms], dtype=torch.float64, device=tdev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(t_ms.item()) / args.steps
    total_units = total * N * F * T
    value = total_units / (ms_per_step / 1e3)

    # final gather of the per-shard estimates to rank 0 (outside the timed region)
    gather_ms = None
    if world > 1:
        torch.cuda.synchronize()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        src = torch.view_as_real(P if tdev != "cpu" else P.cpu()).contiguous()
        shards = [torch.empty_like(src) for _ in range(world)] if rank == 0 else None
        dist.gather(src, shards, dst=0)  # equal-size shards (U mixtures per rank)
        g1.record(stream)
        torch.cuda.synchronize()
        gather_ms = g0.elapsed_time(g1)

    # roofline of the loop kernel (SURVEY.md §8(d) streaming-model bytes)
    c = 8 if cfg.dtype == "c64" else 16
    r = c // 2
    algo_bytes_pt = 2 * I * c + 3 * J * r
    units_launch = U * N * F * T
    k_ms = statistics.mean(kernel_ms)
    achieved = algo_bytes_pt * units_launch / (k_ms / 1e3) / 1e9
    peak, peak_src = peak_hbm()
    tr = ncu_traffic()
    if tr and tr.get("units_per_launch") not in (None, units_launch):
        tr = None  # the committed capture is for a different launch size
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": (tr or {}).get("dram_bytes_per_launch"),
                "kernel": "ffca_loop_kernel<float,3,3,2,true>",
                "kernel_ms": round(k_ms, 4),
                "algorithmic_bytes_per_unit": algo_bytes_pt,
                "units_per_launch": units_launch,
                "peak_source": peak_src,
                "traffic_source": (tr or {}).get("source"),
                "note": ("streaming-model bytes (2*I*c + 3*J*r per TF-point-iteration); the kernel keeps each "
                         "bin resident in shared memory and reads y from HBM once per run, so frac > 1 means "
                         "it beats the two-pass streaming roofline")}

    # end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        yh = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
        yh.copy_(y)
        Ph, lh, vh = (torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (P0, lam0, v0))
        Ph.copy_(P0)
        lh.copy_(lam0)
        vh.copy_(v0)
        Yn, Pn, Ln, Vn = yh.numpy(), Ph.numpy(), lh.numpy(), vh.numpy()
        outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).numpy() for t in (P0, lam0, v0)]
        lib.ffca_set_kernel_timing(0)

        def api_step():
            return run_fastfca_batch(Yn, Pn, Ln, Vn, iterations=T, stream=sptr, out=outs)

        api_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            api_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=tdev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item()) / args.steps
        h2d = sum(a.nbytes for a in (Yn, Pn, Ln, Vn))
        d2h = sum(o.nbytes for o in outs) + U * F * 4
        e2e = {"value": total_units / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": round(e2e_ms, 3),
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h) * world,
               "api": "paper_1805_09498_b200.fastfca.run_fastfca_batch (host numpy, pinned)",
               "stats": "TransformedStats are materialised lazily on access (not in this timing)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        pool, cores = cpu_pool()
        try:
            n_mix = args.cpu_mixtures or cores
            val, wall = cpu_measure(cfg, n_mix, pool)
        finally:
            pool.close()
        cpu = {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": (f"{n_mix} mixtures of the config shape (I=J=3,F=513,N=626), full {T} iterations incl. "
                          f"stats refresh, oracle/ numpy complex128 port, 1 process/core "
                          f"(OPENBLAS_NUM_THREADS=1), wall {wall:.1f} s"),
               "cpu_model": cpu_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64 (fp32 arithmetic; fp64 per-bin solves)",
            "data": "synthetic (BASELINE.json config-3 generator, torch-seeded on device)",
            "config": {"workload": cfg.name, "mixtures": total, "mixtures_per_gpu": U, "I": I, "J": J, "F": F, "N": N,
                       "iterations": T, "inner_iterations": 1,
                       "l2_policy": "inputs larger than L2 (y 1.97 GB + v 0.99 GB vs 126 MB L2)",
                       "parallelism": f"independent {U}-mixture batch per GPU x{world} (no data-path collective)"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
        }
        if gather_ms is not None:
            line["gather_ms"] = round(gather_ms, 3)
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm's CPU implementation on the host cores
# ---------------------------------------------------------------------------


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_1805_09498_b200.workloads import CONFIGS

    cfg = CONFIGS[args.config]
    pool, cores = cpu_pool()
    try:
        n_mix = args.cpu_mixtures or cores
        for _ in range(args.warmup):
            cpu_measure(cfg, n_mix, pool)
        vals, walls = [], []
        for _ in range(args.steps):
            v, w = cpu_measure(cfg, n_mix, pool)
            vals.append(v)
            walls.append(w)
    finally:
        pool.close()
    value = statistics.mean(vals)
    sample = (f"{n_mix} mixtures of the config shape per step, full {cfg.iterations} iterations incl. stats "
              f"refresh; oracle/ numpy port of fcasep.run_fastfca (complex128; the reference has no 32-bit path)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.mean(walls), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "impl": "reference",
        "data": "synthetic (BASELINE.json generator, numpy-seeded)",
        "config": {"workload": cfg.name, "mixtures_per_step": n_mix, "I": cfg.I, "J": cfg.J, "F": cfg.F,
                   "N": cfg.N, "iterations": cfg.iterations},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        ndev = max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank % ndev)
        # FFCA_DIST_BACKEND=gloo lets the multi-rank path be exercised with several ranks per GPU
        backend = os.environ.get("FFCA_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank % ndev))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
