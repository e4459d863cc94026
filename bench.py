#!/usr/bin/env python
"""Benchmark of the FastFCA-AS estimation loop on B200 (BASELINE.json metric).

Headline workload: BASELINE.json config 3 -- 256 independent mixtures, each
I=J=3 microphones/sources, F=513 bins, N=626 frames, complex64, 20 iterations
(the metric's I=3,J=3 case at a size that fills the GPU; config 0 is the
single-mixture CPU-runnable case).  Mixtures are independent, so at N GPUs the
256 mixtures are split into contiguous blocks (strong scaling, no data-path
collective); the estimates are gathered to rank 0 afterwards,
timed separately (`gather`).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N > 1` without torchrun re-launches itself under
`torch.distributed.run` with N ranks (one per GPU; ranks share a GPU only when
the box has fewer, in which case the gloo backend is used and the line says so).

One step = one call of the estimator over all of this rank's mixtures, every
iteration executed (v, lambda and P updates; power floor computed on device).
  value    device-resident inputs, CUDA events on the launch stream, max over ranks
  e2e      the public API `run_fastfca_batch(..., stats="device")` from pinned host
           buffers: H2D of the inputs, the loop, the final statistics refresh
           (fastfca.py:466, as the reference's run_fastfca does) into a
           device-resident snapshot -- the drop-in run_fastfca's behaviour -- and
           D2H of P, lambda, v; `e2e_stats_to_host` also copies mu, phi to host
           numpy arrays, `e2e_loop_only` skips the statistics
Also reported: a complex128 line on the config-3 shape (the reference is fp64
only), the config-2 and config-4 F-sharded lines, the parity of two mixtures
of the timed batch against the CPU oracle, and the CPU baseline (the stock
reference from baseline/_ref on the host cores).
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
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
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--mixtures", type=int, default=None, help="override the total mixture count (testing)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the c128 / config-2 / config-4 lines")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--cpu-mixtures", type=int, default=None)
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU legs: the stock reference (baseline/_ref) -- or, if it is not installed,
# the oracle/ port -- on the host cores.  bench.py is one of the places allowed
# to run oracle/ (CPU baseline and the parity spot-check only).
# ---------------------------------------------------------------------------


def _cpu_gen(args):
    from paper_1805_09498_b200.workloads import mixture
    seed, I, J, F, N, rank, zf = args
    y, P0, lam0, v0, _ = mixture(seed, I, J, F, N, rank, zf)
    return y, P0, lam0, v0


def _stock_available():
    try:
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import fcasep.fastfca  # noqa: F401
        return os.path.dirname(sys.modules["fcasep"].__file__).startswith(REF_DIR)
    except Exception:  # noqa: BLE001
        return False


def _cpu_run(args):
    """One full run_fastfca (20 iterations + the final stats refresh) on one core; returns seconds."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    y, P0, lam0, v0, iters, kind = args
    if kind == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from fcasep import fastfca as ref_fastfca
        from fcasep.stft import ObservationTensor as RefObs
        obs, init = RefObs(y), ref_fastfca.FastFcaParams(P0, lam0, v0)
        t0 = time.perf_counter()
        ref_fastfca.run_fastfca(obs, init, iterations=iters)
        return time.perf_counter() - t0
    from oracle import fastfca_ref
    t0 = time.perf_counter()
    fastfca_ref.run_fastfca(y, P0, lam0, v0, iterations=iters, stats=True)
    return time.perf_counter() - t0


def cpu_measure(cfg, n_mix, pool, kind):
    """Throughput of n_mix full runs spread over the host cores (wall clock of the parallel map)."""
    inputs = pool.map(_cpu_gen, [(9000 + k, cfg.I, cfg.J, cfg.F, cfg.N, cfg.rank, cfg.zero_frac)
                                 for k in range(n_mix)])
    t0 = time.perf_counter()
    pool.map(_cpu_run, [(y, P, l, v, cfg.iterations, kind) for (y, P, l, v) in inputs], chunksize=1)
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


def cpu_sample(cfg, n_mix, kind, wall=None):
    what = ("unmodified reference fcasep.fastfca.run_fastfca from baseline/_ref" if kind == "reference"
            else "oracle/ numpy port of fcasep.run_fastfca (stock reference not installed)")
    s = (f"{n_mix} mixtures of the config shape (I={cfg.I},J={cfg.J},F={cfg.F},N={cfg.N}) per step, full "
         f"{cfg.iterations} iterations incl. the final stats refresh (fastfca.py:466), complex128 (the reference "
         f"has no 32-bit path); {what}; 1 process per core, OPENBLAS_NUM_THREADS=1")
    return s + (f"; wall {wall:.1f} s" if wall is not None else "")


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
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
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


def ncu_profile():
    """Per-launch ncu figures of the headline loop kernel (profiles/loop_kernel_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "loop_kernel_traffic.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


class Dist:
    """torch.distributed plumbing: rank / world, barrier, max over ranks, gather."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        ndev = max(1, torch.cuda.device_count())
        self.device_index = self.local_rank % ndev
        self.shared_gpu = self.world > ndev
        self.backend = None
        if self.world > 1:
            torch.cuda.set_device(self.device_index)
            # NCCL needs one GPU per rank; ranks sharing a GPU (a 1-GPU box) exchange over gloo
            self.backend = os.environ.get("FFCA_DIST_BACKEND", "gloo" if self.shared_gpu else "nccl")
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device_index))
            else:
                dist.init_process_group(self.backend)
        self.dist = dist

    @property
    def on(self):
        return self.world > 1

    def barrier(self):
        if self.on:
            self.dist.barrier()

    def tdev(self):
        import torch
        return torch.device("cuda", self.device_index) if self.backend == "nccl" else torch.device("cpu")

    def max(self, x: float) -> float:
        if not self.on:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.tdev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.on:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self.tdev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def gather_ms(self, tensors, stream):
        """Gather this rank's result tensors to rank 0 (padded to the largest shard); device ms."""
        import torch
        if not self.on:
            return None, 0
        torch.cuda.synchronize()
        self.barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        nbytes = 0
        for t in tensors:
            flat = torch.view_as_real(t).reshape(-1) if t.is_complex() else t.reshape(-1)
            n = torch.tensor([flat.numel()], dtype=torch.int64, device=self.tdev())
            self.dist.all_reduce(n, op=self.dist.ReduceOp.MAX)
            mx = int(n.item())
            src = torch.zeros(mx, dtype=flat.dtype, device=flat.device)
            src[:flat.numel()] = flat
            if self.backend != "nccl":
                src = src.cpu()
            outs = [torch.empty_like(src) for _ in range(self.world)] if self.rank == 0 else None
            self.dist.gather(src, outs, dst=0)
            nbytes += flat.numel() * flat.element_size()
        g1.record(stream)
        torch.cuda.synchronize()
        return g0.elapsed_time(g1), nbytes


def time_device_steps(lib, step, steps, warmup, D, stream, sample_clocks=False):
    """W untimed steps, then K steps between CUDA events on the launch stream (barrier + sync on
    both sides); returns (max-over-ranks ms per step, mean loop-kernel ms, launches, clocks)."""
    import torch
    lib.ffca_set_kernel_timing(1)
    for _ in range(warmup):
        step()
    D.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(D.device_index) if sample_clocks else None
    if sampler:
        time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kernel_ms, launches = [], 0
    ev0.record(stream)
    for _ in range(steps):
        step()
        kernel_ms.append(float(lib.ffca_last_kernel_ms()))
        launches += int(lib.ffca_last_launch_count())
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    D.barrier()
    lib.ffca_set_kernel_timing(0)
    ms = D.max(ev0.elapsed_time(ev1)) / steps
    return ms, statistics.mean(kernel_ms), launches, clocks


def device_runner(lib, _lib, code, dev, stream, y, P0, lam0, v0, T):
    import torch
    U, I, N, F = y.shape
    J = v0.shape[1]
    P, lam, v = torch.empty_like(P0), torch.empty_like(lam0), torch.empty_like(v0)

    def step():
        rc = lib.ffca_fastfca_run(dev.index, stream.cuda_stream, _lib.MEM_DEVICE, code, U, I, J, N, F,
                                  y.data_ptr(), P0.data_ptr(), lam0.data_ptr(), v0.data_ptr(), _lib.VF_AUTO, 0.0,
                                  None, T, 1, 0, P.data_ptr(), lam.data_ptr(), v.data_ptr(), None, None, None)
        _lib.check(rc, "ffca_fastfca_run")

    return step, (P, lam, v)


def plan_name(lib, _lib, code, U, I, J, N, F):
    out = np.zeros(8, np.int32)
    lib.ffca_plan_loop_ex(0, code, U, I, J, N, F, _lib.VF_AUTO, 1, out.ctypes.data_as(_lib._ip))
    G, C, NL, thr, res, smem, tm, tmcols = (int(x) for x in out)
    R = "float" if code == _lib.C64 else "double"
    name = f"ffca_loop_kernel<{R},{I},{J},{G},{str(bool(res)).lower()}" + (",true,true>" if tm else ">")
    return name, {"G": G, "cluster": C, "frames_per_cta": NL, "threads": thr, "resident": bool(res),
                  "smem_bytes": smem, "y_records_in_tensor_memory": bool(tm), "tmem_columns_per_cta": tmcols}


def parity_check(y, P0, lam0, v0, outs, T, picks):
    """Oracle (fp64) on a few mixtures of the timed batch vs the device results: max rel error."""
    from oracle import fastfca_ref
    worst = 0.0
    for u in picks:
        yy = y[u].cpu().numpy().astype(np.complex128)
        ref = fastfca_ref.run_fastfca(yy, P0[u].cpu().numpy().astype(np.complex128),
                                      lam0[u].cpu().numpy().astype(np.float64),
                                      v0[u].cpu().numpy().astype(np.float64), iterations=T, stats=False)
        for got, want in zip(outs, (ref.P, ref.lam, ref.v)):
            g = got[u].cpu().numpy()
            worst = max(worst, float(np.abs(g - want).max() / np.abs(want).max()))
    return worst


def run_ours(args, D):
    import torch

    from paper_1805_09498_b200 import _lib
    from paper_1805_09498_b200.fastfca import run_fastfca_batch
    from paper_1805_09498_b200.multigpu import shard_range
    from paper_1805_09498_b200.workloads import CONFIGS, make_torch, make_torch_range

    rank, world = D.rank, D.world
    cfg = CONFIGS[args.config]
    total = args.mixtures or cfg.mixtures
    u0, u1 = shard_range(total, rank, world)
    U = u1 - u0
    dev = torch.device("cuda", D.device_index)
    torch.cuda.set_device(dev)
    _lib.set_device(dev.index)
    lib = _lib.require_gpu()
    I, J, N, F, T = cfg.I, cfg.J, cfg.N, cfg.F, cfg.iterations
    stream = torch.cuda.current_stream()
    ccfg = dataclasses.replace(cfg, dtype="c128")

    # every mixture is drawn from its own generator (seed0 + u): the shards of N ranks are
    # exactly the slices of the single-GPU batch.  fp64 draws; the headline casts to complex64.
    y64, P64, l64, v64 = make_torch_range(ccfg, 1234, u0, u1, dev)
    y, P0, lam0, v0 = y64.to(torch.complex64), P64.to(torch.complex64), l64.float(), v64.float()
    if args.no_extra:
        del y64, P64, l64, v64
    torch.cuda.synchronize()
    code = _lib.C64 if cfg.dtype == "c64" else _lib.C128

    step, outs = device_runner(lib, _lib, code, dev, stream, y, P0, lam0, v0, T)
    ms_per_step, k_ms, launches, clocks = time_device_steps(lib, step, args.steps, args.warmup, D, stream,
                                                           sample_clocks=True)
    total_units = total * N * F * T
    value = total_units / (ms_per_step / 1e3)
    gather_ms, gather_bytes = D.gather_ms(outs, stream)

    # ---- roofline of the loop kernel ----
    kname, kplan = plan_name(lib, _lib, code, U, I, J, N, F)
    c = 8 if cfg.dtype == "c64" else 16
    r = c // 2
    units_launch = U * N * F * T
    one_pass = U * N * F * (I * c + 2 * J * r)  # y and v in, v out: the kernel's minimum HBM traffic per run
    streaming = (2 * I * c + 3 * J * r) * units_launch  # SURVEY §8(d) two-pass streaming model
    peak, peak_src = peak_hbm()
    prof = ncu_profile()
    if prof and prof.get("units_per_launch") not in (None, units_launch):
        prof = None  # the committed capture is for a different launch size
    achieved = one_pass / (k_ms / 1e3) / 1e9
    roofline = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4),
        "traffic": (prof or {}).get("dram_bytes_per_launch"),
        "kernel": kname, "plan": kplan, "kernel_ms": round(k_ms, 4),
        "algorithmic_bytes_per_launch": one_pass,
        "algorithmic_bytes": "one pass of y and v in, v out per run (the bin-resident kernel's minimum)",
        "units_per_launch": units_launch, "peak_source": peak_src,
        "effective_streaming_GBps": round(streaming / (k_ms / 1e3) / 1e9, 1),
        "effective_streaming_note": ("SURVEY §8(d) two-pass streaming model, 2*I*c + 3*J*r = "
                                     f"{2 * I * c + 3 * J * r} B per TF-point-iteration; a model figure, not DRAM "
                                     "traffic -- the kernel holds each bin on chip (y in tensor memory, v in shared memory) for the whole run"),
        "binding": None,
    }
    # compute roofline of the same launch: algorithmic FP32 flops of the formulation per TF-point
    # iteration (phase A: P^H y, |.|^2, weights, d, r2 - r1, v', ratio, s0, s1; phase B: weights,
    # |y|^2, off-diagonal y y^H, the I accumulations of the I x I B_i) -- per-bin reductions,
    # reciprocals and the fp64 solves not counted -- against the CUDA-core FP32 peak at the clock
    # measured during the timed region (148 SMs x 128 lanes x 2 flops)
    flops_unit = (8 * I * I + 6 * I + 6 * I * J + 7 * J) + (2 * I * J + 3 * I + 3 * I * (I - 1) + 2 * I ** 3)
    clk_mhz = (clocks or {}).get("sm_mhz") or 1965.0
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp_peak = nsm * 128 * 2 * clk_mhz * 1e6 / 1e12
    fp_ach = flops_unit * units_launch / (k_ms / 1e3) / 1e12
    roofline["compute"] = {"bound": "fp32 (CUDA cores; no tensor-core work in this path)", "achieved": round(fp_ach, 2),
                           "peak": round(fp_peak, 2), "unit": "TFLOP/s", "frac": round(fp_ach / fp_peak, 3),
                           "flops_per_unit": flops_unit,
                           "peak_source": f"{nsm} SMs x 128 FP32 lanes x 2 x {clk_mhz:.0f} MHz (median SM clock under load)"}
    if prof:
        clk = (clocks or {}).get("sm_mhz") or 1965.0
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        binding = {"resource": "FP32 FMA pipe / issue in the point phases at the 16 warps per SM the registers allow, "
                               "+ per-bin reductions / fp64 solves",
                   "source": prof.get("source")}
        if prof.get("warp_instructions_per_launch"):
            binding["issue_frac"] = round(prof["warp_instructions_per_launch"] / (4 * sms * clk * 1e6 * k_ms / 1e3), 3)
        for k in ("issue_active_pct", "fma_pipe_pct", "warps_active_pct", "fp64_pipe_pct"):
            if k in prof:
                binding[k] = prof[k]
        roofline["binding"] = binding

    # ---- end to end through the public API (host numpy, pinned), stats included ----
    e2e = e2e_loop = e2e_host = None
    if not args.no_e2e:
        def pinned_like(t):
            return torch.empty(t.shape, dtype=t.dtype, pin_memory=True)

        host_in = [pinned_like(t) for t in (y, P0, lam0, v0)]
        for h, t in zip(host_in, (y, P0, lam0, v0)):
            h.copy_(t)
        Yn, Pn, Ln, Vn = (h.numpy() for h in host_in)
        outs_h = [pinned_like(t).numpy() for t in (P0, lam0, v0)]
        mu_h = torch.empty((U, J, N, F, I), dtype=y.dtype, pin_memory=True).numpy()
        phi_h = torch.empty((U, J, N, F, I), dtype=v0.dtype, pin_memory=True).numpy()
        mu_d = torch.empty((U, J, N, F, I), dtype=y.dtype, device=dev)
        phi_d = torch.empty((U, J, N, F, I), dtype=v0.dtype, device=dev)

        def api_time(with_stats):
            def call():
                if with_stats == "device":
                    run_fastfca_batch(Yn, Pn, Ln, Vn, iterations=T, stream=stream.cuda_stream, out=outs_h,
                                      stats="device", stats_out=(mu_d, phi_d))
                elif with_stats:
                    run_fastfca_batch(Yn, Pn, Ln, Vn, iterations=T, stream=stream.cuda_stream, out=outs_h,
                                      stats=True, stats_out=(mu_h, phi_h))
                else:
                    run_fastfca_batch(Yn, Pn, Ln, Vn, iterations=T, stream=stream.cuda_stream, out=outs_h)
            call()
            D.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                call()
            e1.record(stream)
            torch.cuda.synchronize()
            return D.max(e0.elapsed_time(e1)) / args.steps

        h2d = sum(a.nbytes for a in (Yn, Pn, Ln, Vn))
        d2h = sum(o.nbytes for o in outs_h) + U * F * 4
        t_loop = api_time(False)
        t_dev = api_time("device")
        t_stats = api_time(True)
        e2e = {"value": total_units / (t_dev / 1e3), "unit": UNIT, "ms_per_step": round(t_dev, 3),
               "h2d_bytes_per_step": int(D.sum(h2d)), "d2h_bytes_per_step": int(D.sum(d2h)),
               "api": "paper_1805_09498_b200.fastfca.run_fastfca_batch(..., stats='device') (host numpy, pinned)",
               "scope": "the drop-in run_fastfca's default behaviour: H2D of y, P, lambda, v; the loop; the final "
                        "statistics refresh (fastfca.py:466) into a device-resident snapshot (copied to the host "
                        "only when read; the Wiener images consume it in place); D2H of P, lambda, v"}
        e2e_host = {"value": total_units / (t_stats / 1e3), "unit": UNIT, "ms_per_step": round(t_stats, 3),
                    "h2d_bytes_per_step": int(D.sum(h2d)),
                    "d2h_bytes_per_step": int(D.sum(d2h + mu_h.nbytes + phi_h.nbytes)),
                    "api": "run_fastfca_batch(..., stats=True)",
                    "scope": "as e2e, and the statistics mu, phi copied to host numpy arrays too (PCIe-bound)"}
        e2e_loop = {"value": total_units / (t_loop / 1e3), "unit": UNIT, "ms_per_step": round(t_loop, 3),
                    "h2d_bytes_per_step": int(D.sum(h2d)), "d2h_bytes_per_step": int(D.sum(d2h)),
                    "scope": "as e2e without the statistics refresh (P, lambda, v only)"}
        del host_in, outs_h, mu_h, phi_h, mu_d, phi_d

    # ---- parity of the timed batch (rank 0: first and last mixture of its shard vs the fp64 oracle) ----
    parity = None
    if rank == 0 and not args.no_parity and U > 0:
        picks = sorted({0, U - 1})
        t0 = time.perf_counter()
        worst = parity_check(y, P0, lam0, v0, outs, T, picks)
        parity = {"max_rel": worst, "tolerance": 1e-4, "ok": worst <= 1e-4,
                  "what": (f"mixtures {[u0 + p for p in picks]} of the timed complex64 batch: P, lambda, v after "
                           f"{T} iterations vs oracle/ (fp64, same inputs upcast); rel = max|d| / max|ref|"),
                  "cpu_s": round(time.perf_counter() - t0, 1)}

    # ---- extra lines: complex128 on the config-3 shape; config 2 / 4 F-sharded ----
    extra = {}
    if not args.no_extra:
        del step, outs
        k2 = max(2, min(args.steps, 5))
        st64, _ = device_runner(lib, _lib, _lib.C128, dev, stream, y64, P64, l64, v64, T)
        ms64, k64, _, _ = time_device_steps(lib, st64, k2, 2, D, stream)
        extra["value_c128"] = {"value": total_units / (ms64 / 1e3), "unit": UNIT, "ms_per_step": round(ms64, 3),
                               "kernel_ms": round(k64, 3), "steps": k2, "dtype": "c128 (fp64 arithmetic)",
                               "kernel": plan_name(lib, _lib, _lib.C128, U, I, J, N, F)[0],
                               "note": "the same 256 mixtures in complex128, the reference's own precision"}
        del y64, P64, l64, v64, st64
        torch.cuda.empty_cache()
        for ci in (2, 4):
            extra[f"config{ci}"] = fsharded_line(args, D, lib, _lib, CONFIGS[ci], dev, stream, make_torch)
            torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0 at N = 1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        kind = "reference" if _stock_available() else "port"
        pool, cores = cpu_pool()
        try:
            n_mix = args.cpu_mixtures or cores
            val, wall = cpu_measure(cfg, n_mix, pool, kind)
        finally:
            pool.close()
        cpu = {"value": val, "unit": UNIT, "cores": cores, "kind": kind, "sample": cpu_sample(cfg, n_mix, kind, wall),
               "cpu_model": cpu_info(), "dtype": "c128"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c64 (fp32 arithmetic; fp64 per-bin solves)",
            "data": "synthetic (BASELINE.json config-3 generator, torch-seeded on device, one seed per mixture)",
            "config": {"workload": cfg.name, "mixtures": total, "mixtures_per_gpu": [shard_range(total, q, world)[1] -
                                                                                     shard_range(total, q, world)[0]
                                                                                     for q in range(world)],
                       "I": I, "J": J, "F": F, "N": N, "iterations": T, "inner_iterations": 1,
                       "l2_policy": "inputs larger than L2 (y 1.97 GB + v 0.99 GB vs 126 MB L2)",
                       "parallelism": f"mixture blocks over {world} rank(s), no data-path collective"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_stats_to_host": e2e_host,
            "e2e_loop_only": e2e_loop,
            "clocks": clocks,
            "gpu_launches": launches,
            "parity": parity,
        }
        if world > 1:
            line["gather"] = {"ms": round(gather_ms, 3), "bytes": gather_bytes, "backend": D.backend,
                              "what": "P, lambda, v of every rank to rank 0 (after the timed region)"}
            line["ranks_share_gpu"] = D.shared_gpu
            if D.shared_gpu:
                line["note"] = (f"{world} ranks on {torch.cuda.device_count()} GPU(s): the ranks time-share a GPU, "
                                "so this exercises the multi-rank path, not multi-GPU scaling")
        line.update(extra)
        print(json.dumps(line), flush=True)


def fsharded_line(args, D, lib, _lib, cfg, dev, stream, make_torch):
    """One long mixture (config 2 / 4), contiguous F-blocks per rank, device-resident loop."""
    import torch

    from paper_1805_09498_b200.multigpu import shard_range

    f0, f1 = shard_range(cfg.F, D.rank, D.world)
    y, P0, lam0, v0 = make_torch(cfg, 4321 + cfg.I, 1, dev)  # same draws on every rank
    y = y[..., f0:f1].contiguous()
    v0 = v0[..., f0:f1].contiguous()
    P0 = P0[:, f0:f1].contiguous()
    lam0 = lam0[:, :, f0:f1].contiguous()
    torch.cuda.synchronize()
    code = _lib.C64 if cfg.dtype == "c64" else _lib.C128
    step, outs = device_runner(lib, _lib, code, dev, stream, y, P0, lam0, v0, cfg.iterations)
    k = max(2, min(args.steps, 10))
    ms, k_ms, launches, _ = time_device_steps(lib, step, k, 2, D, stream)
    gather_ms, gather_bytes = D.gather_ms(outs, stream)
    units = cfg.N * cfg.F * cfg.iterations
    c = 8 if cfg.dtype == "c64" else 16
    r = c // 2
    Fb = f1 - f0
    one_pass = cfg.N * Fb * (cfg.I * c + 2 * cfg.J * r)
    out = {"workload": cfg.name, "value": units / (ms / 1e3), "unit": UNIT, "ms_per_step": round(ms, 3),
           "kernel_ms": round(k_ms, 3), "steps": k, "launches_per_step": launches / k,
           "kernel": plan_name(lib, _lib, code, 1, cfg.I, cfg.J, cfg.N, Fb)[0],
           "bins_per_gpu": Fb, "scaling": "strong (F-blocks)",
           "one_pass_GBps": round(one_pass / (k_ms / 1e3) / 1e9, 1),
           "effective_streaming_GBps": round((2 * cfg.I * c + 3 * cfg.J * r) * cfg.N * Fb * cfg.iterations /
                                             (k_ms / 1e3) / 1e9, 1)}
    if D.on:
        out["gather"] = {"ms": round(gather_ms, 3), "bytes": gather_bytes}
    del y, P0, lam0, v0, outs
    return out


# ---------------------------------------------------------------------------
# reference arm: the stock reference's CPU implementation on the host cores
# ---------------------------------------------------------------------------


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(max(1, args.gpus))))
    if rank != 0:
        return
    from paper_1805_09498_b200.workloads import CONFIGS

    cfg = CONFIGS[args.config]
    kind = "reference" if _stock_available() else "port"
    pool, cores = cpu_pool()
    try:
        n_mix = args.cpu_mixtures or cores
        for _ in range(args.warmup):
            cpu_measure(cfg, n_mix, pool, kind)
        vals, walls = [], []
        for _ in range(args.steps):
            v, w = cpu_measure(cfg, n_mix, pool, kind)
            vals.append(v)
            walls.append(w)
    finally:
        pool.close()
    value = statistics.mean(vals)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.mean(walls), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "impl": "reference",
        "data": "synthetic (BASELINE.json generator, numpy-seeded)",
        "config": {"workload": cfg.name, "mixtures_per_step": n_mix, "I": cfg.I, "J": cfg.J, "F": cfg.F,
                   "N": cfg.N, "iterations": cfg.iterations},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": cpu_sample(cfg, n_mix, kind), "cpu_model": cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch(args):
    """`--gpus N` outside torchrun: run this script under torch.distributed.run with N ranks."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    D = Dist()
    try:
        run_ours(args, D)
    finally:
        if D.on:
            D.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
