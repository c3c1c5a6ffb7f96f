#!/usr/bin/env python
"""Benchmark of the B200-native batched signature transform (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A "step" is one pass of the hot path (sigk_signature_f32 through the C ABI)
over one batch. Default workload = BASELINE.json configs[1]: B=128 paths,
L=1000, d=5, depth N=4, fp32, synthetic Brownian paths (X0 = 0, increments
N(0, 1/(L-1)), Philox keyed by (seed, global row, t, c)). Multi-GPU (torchrun,
one rank per GPU, no data-path collective, timings = max over ranks):
c1..c4 are weak-scaled (every rank folds its own B rows); c5 (BASELINE.json
configs[4], "batch sharded across 1/2/4/8 B200") is strong-scaled: the global
B = 8192 batch is split into contiguous row shards (rank_rows, the split of
sigk_signature_sharded_*), so N=1 is exactly the single-GPU c5 run.

value  : device-resident inputs, K steps captured in CUDA graphs and replayed
         on one stream, CUDA events around the whole region. Every timed step
         reads a distinct input batch of a pool that rotates through more than
         2x the 126 MB L2, and L2 is flushed (a 512 MiB device write) right
         before the timed region, so inputs come from HBM even at small K.
e2e    : the same call with HOST (pinned) buffers: H2D of the step's paths,
         kernels, D2H of the step's signatures, every step (PCIe link rates
         reported beside it).
roofline: achieved = credited FP32 flops per step / mean step interval of the
         timed replays (back-to-back launches may overlap through programmatic
         dependent launch); `single_call` = the same credited flops over the
         fold kernel's own duration with no launch overlap (CUDA events around
         single launches inside an untimed graph replay). Peak = FFMA-pipe
         rate measured on this GPU by a register-resident microbenchmark.
cpu_baseline: the reference's own sequential_forward<double> compiled from its
         sources (oracle/_ref; else the C port), all host threads, rank 0 only;
         `variants` adds 1 thread (as shipped) and the <float> instantiation.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": (32, 100, 2, 4),
    "c2": (128, 1000, 5, 4),
    "c3": (128, 10000, 5, 4),
    "c4": (64, 500, 10, 5),
    "c5": (8192, 1000, 8, 4),
}
L2_BYTES = 126 * 1024 * 1024
TUNE = {}  # sigk_tuning overrides from the command line (chunks / prefix_len)
GRAPH_STEPS = int(os.environ.get("SIGK_BENCH_GRAPH_STEPS", "256"))  # steps captured per CUDA graph
NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def baseline_metric():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["metric"]


def work_per_path(L, d, N):
    """credited flops F = 2 W (L-1), W = Σ_k (N-k+1) d^k; bytes = 4 (L d + D)."""
    W = sum((N - k + 1) * d ** k for k in range(1, N + 1))
    D = sum(d ** n for n in range(1, N + 1))
    return 2.0 * W * (L - 1), 4.0 * (L * d + D), W, D


def rank_rows(config: str, world: int, rank: int):
    """(global batch, first row, row count, scaling) of `rank` for a config: c5
    is strong-scaled over contiguous row shards (shard_rows: the split of
    sigk_signature_sharded_*); the other configs give every rank its own B rows
    (weak scaling, rows rank*B ..)."""
    from paper_2501_08455_b200.shard import shard_rows

    B = CONFIGS[config][0]
    if config == "c5":
        lo, hi = shard_rows(B, world, rank)
        return B, lo, hi - lo, "strong"
    return B * world, rank * B, B, "weak"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """NVML SM clock + clocks-event reasons sampled every 10 ms while running."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock"}

    def __init__(self, index):
        self.index, self.samples, self.reasons, self._stop = index, [], 0, threading.Event()
        self.max_mhz = None
        self.ok = False
        if os.environ.get("SIGK_BENCH_NO_CLOCKS"):  # experiments: no sampler thread
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = nvml_handle(pynvml, index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        s = sorted(self.samples)
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(s)}


def nvml_handle(pynvml, cuda_index):
    """NVML handle of a CUDA device by PCI bus id (NVML and CUDA orders can differ,
    e.g. under CUDA_VISIBLE_DEVICES); falls back to the index."""
    try:
        import torch

        pr = torch.cuda.get_device_properties(cuda_index)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        return pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
    except Exception:
        return pynvml.nvmlDeviceGetHandleByIndex(cuda_index)


def bind_to_gpu_numa(index):
    """Run on the host cores local to the GPU (NVML CPU affinity) so pinned
    host buffers are first-touched on the GPU's NUMA node: the e2e copies then
    avoid the socket interconnect."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = nvml_handle(pynvml, index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            full = os.sched_getaffinity(0)
            os.sched_setaffinity(0, cpus)
            return full
    except Exception:
        pass
    return None


# SIGK_BENCH_SHARE_GPU=1 (plumbing checks on a one-GPU box, never a bench value): ranks
# share the visible GPUs round robin and talk over gloo (NCCL needs one GPU per rank)
SHARE_GPU = bool(os.environ.get("SIGK_BENCH_SHARE_GPU"))


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARE_GPU:
        import torch

        local %= max(1, torch.cuda.device_count())
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARE_GPU else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ---------------------------------------------------------------- CPU arms
def cpu_reference_run(X64, N, threads):
    """One pass of the reference CPU path; returns (seconds, kind)."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    if O.ref() is not None:
        O.ref_forward(X64, N, threads=threads)
        kind = "reference"
    else:
        O.signature(X64, N, threads=threads)
        kind = "port"
    return time.perf_counter() - t0, kind


def cpu_timed(X, N, threads, budget_s):
    """Best paths/s of repeated reference passes over a bounded row sample of X
    (f64 or f32: the reference's sequential_forward<double> / <float>)."""
    B = X.shape[0]
    w = max(1, min(B, threads))
    t1, kind = cpu_reference_run(X[:w], N, threads)  # one wave of `threads` rows
    rows = int(max(w, min(B, w * max(1, int(min(1.0, budget_s / 4) / max(t1, 1e-9))))))
    Xs = X[:rows]
    best, total, reps = float("inf"), 0.0, 0
    while (total < budget_s and reps < 1000) or reps == 0:
        dt, kind = cpu_reference_run(Xs, N, threads)
        best, total, reps = min(best, dt), total + dt, reps + 1
    return rows / best, rows, reps, total, kind


def cpu_baseline(X32, N, budget_s=6.0, variants=True):
    """Reference sequential_forward<double> (what signature_sequential runs) on the
    same fp32 inputs promoted to double, all host threads, repeated ~budget_s;
    plus 1 thread (the reference as shipped, README.md:65) and <float>
    (bench.cpp:29-56, 182-186) variants on bounded samples."""
    import numpy as np

    threads = os.cpu_count() or 1
    X64 = X32.astype(np.float64)
    B = X64.shape[0]
    v, rows, reps, total, kind = cpu_timed(X64, N, threads, budget_s)
    out = {"value": v, "unit": "paths/s", "cores": threads, "kind": kind,
           "sample": f"{rows} of {B} rows, best of {reps} passes ({total:.1f} s wall), f64, {threads} threads",
           "cpu_model": cpu_model()}
    if variants:
        var = []
        for prec, Xv in (("f64", X64), ("f32", np.ascontiguousarray(X32, np.float32))):
            for th in sorted({1, threads}):
                if prec == "f64" and th == threads:
                    continue  # the headline figure above
                vv, r, n, t, k = cpu_timed(Xv, N, th, budget_s / 3)
                var.append({"value": vv, "unit": "paths/s", "threads": th, "precision": prec, "kind": k,
                            "sample": f"{r} rows, best of {n} passes ({t:.1f} s)"})
        out["variants"] = var
    return out


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import numpy as np
    import torch

    import paper_2501_08455_b200 as sk

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    all_cores = bind_to_gpu_numa(torch.cuda.current_device())  # restored for the CPU baseline
    if world > 1:
        import torch.distributed as dist

        if SHARE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    _, L, d, N = CONFIGS[args.config]
    B_global, row0, B, scaling = rank_rows(args.config, world, rank)
    if scaling == "strong":
        TUNE["plan_rows"] = B_global  # same plan (hence bitwise the same rows) for any GPU count
    flops_path, bytes_path, W, D = work_per_path(L, d, N)
    stream = torch.cuda.Stream(device=dev)

    # input pool of more than 2x L2 (rotated every step), this rank's global rows
    in_bytes = B * L * d * 4
    n_buf = 2 if in_bytes > L2_BYTES else min(256, math.ceil(2 * L2_BYTES / in_bytes))
    pool = torch.empty((n_buf, B, L, d), dtype=torch.float32, device=dev)
    with torch.cuda.stream(stream):
        for i in range(n_buf):
            sk.brownian(pool[i], seed=42 + i, row0=row0)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)  # > 4x L2
    out = torch.empty((B, D), dtype=torch.float32, device=dev)
    stream.synchronize()

    st = sk.KernelStats()
    with torch.cuda.stream(stream):
        sk.signature(pool[0], N, stats=st, out=out, **TUNE)
    stream.synchronize()

    # FFMA-pipe peak on this GPU (roofline denominator)
    import ctypes as C

    lib_span = sk.lib()

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.empty(sms * 8 * 256, dtype=torch.float32, device=dev)
    fl = C.c_double(0)
    peak = 0.0
    with torch.cuda.stream(stream):
        for rep in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sk.lib().sigk_bench_ffma(sink.data_ptr(), sms * 8, 2000, C.byref(fl), C.c_void_p(stream.cuda_stream))
            e1.record(stream)
            e1.synchronize()
            if rep:
                peak = max(peak, fl.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)

    # graphs: S distinct steps per graph, every 4th step's fold kernel bracketed by events
    S = min(args.steps, GRAPH_STEPS)
    step_events = []

    def capture(nsteps, with_events, mode=0):
        g = torch.cuda.CUDAGraph()
        evs = {}
        if with_events:  # create the CUDA events (torch creates them lazily on first record)
            for j in range(0, nsteps, 4):
                evs[j] = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                evs[j][0].record(stream)
                evs[j][1].record(stream)
            stream.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for j in range(nsteps):
                _step(sk, pool[j % n_buf], N, out, evs.get(j), mode)
        return g, list(evs.values())

    # warm-up (eager + one graph replay)
    with torch.cuda.stream(stream):
        for j in range(args.warmup):
            _step(sk, pool[j % n_buf], N, out, None)
    stream.synchronize()
    reps_full, rem = divmod(args.steps, S)
    g_main = capture(S, False)[0]  # the timed graph carries no events (they would serialise launches)
    g_rem = capture(rem, False)[0] if rem else None
    g_ev, ev_main = capture(S, True)  # kernel durations, replayed outside the timed region
    lat_plan = sk.plan(B, L, d, N, mode=sk.MODE_LATENCY, **{k: v for k, v in TUNE.items() if k != "mode"})
    with torch.cuda.stream(stream):
        _step(sk, pool[0], N, out, None, sk.MODE_LATENCY)  # plan + scratch outside the capture
    stream.synchronize()
    g_lat, ev_lat = capture(min(S, 64), True, sk.MODE_LATENCY)  # the latency plan, same bracketing
    for _ in range(max(1, args.warmup // S)):
        g_main.replay()
    torch.cuda.synchronize()

    clk = ClockSampler(torch.cuda.current_device())
    barrier(world)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        with torch.cuda.stream(stream):
            # one untimed warm-up replay enqueued right before the timed region, so the
            # GPU is not idle (clocks, caches) when it starts; then the L2 flush evicts
            # that replay's inputs (the timed steps read them from HBM)
            g_main.replay()
            flush.fill_(1.0)
            t0.record(stream)
            for _ in range(reps_full):
                g_main.replay()
            if g_rem is not None:
                g_rem.replay()
            t1.record(stream)
        t1.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    elapsed = max_over_ranks(t0.elapsed_time(t1) * 1e-3, world)
    with torch.cuda.stream(stream):
        flush.fill_(2.0)
        g_ev.replay()
    stream.synchronize()
    fold_ms = [a.elapsed_time(b) for a, b in ev_main]
    fold_s = max_over_ranks(sum(fold_ms) / len(fold_ms) * 1e-3, world)
    with torch.cuda.stream(stream):
        flush.fill_(3.0)
        g_lat.replay()
    stream.synchronize()
    lat_ms = [a.elapsed_time(b) for a, b in ev_lat]
    lat_s = max_over_ranks(sum(lat_ms) / len(lat_ms) * 1e-3, world)

    # device-side span of one launch alone (pair family): %globaltimer stamps at every
    # CTA's entry and exit (sigk_tuning.phase_buf), first entry to last exit — the
    # kernel's execution without the launch latency the event bracket includes
    span_ms = {}
    if st.family == sk.FAMILY_PAIR:
        for mode_name, mode in (("throughput_plan", 0), ("latency_plan", sk.MODE_LATENCY)):
            p = sk.plan(B, L, d, N, mode=mode, **{k: v for k, v in TUNE.items() if k != "mode"})
            ph = torch.zeros((B * p.segments, 12), dtype=torch.int64, device=dev)
            spans = []
            for _ in range(5):
                with torch.cuda.stream(stream):
                    flush.fill_(4.0)
                    tun = sk._Tuning(**TUNE)
                    tun.mode = mode
                    tun.phase_buf = C.c_void_p(ph.data_ptr())
                    sk._check(lib_span.sigk_signature_f32(pool[0].data_ptr(), B, L, d, N, out.data_ptr(),
                                                          sk.SIGK_X_ON_DEVICE | sk.SIGK_OUT_ON_DEVICE,
                                                          C.c_void_p(stream.cuda_stream), C.byref(tun), None))
                stream.synchronize()
                w = ph[:, 10:12].cpu()
                spans.append(float((w[:, 1].max() - w[:, 0].min()).item()) * 1e-6)
            span_ms[mode_name] = max_over_ranks(sorted(spans)[len(spans) // 2], world)

    # single-launch (non-graph) latency of one step, for reference
    with torch.cuda.stream(stream):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _step(sk, pool[0], N, out, None)
        b.record(stream)
    b.synchronize()
    single_ms = a.elapsed_time(b)

    # e2e through the C ABI with host (pinned) buffers
    Xh = pool[0].cpu().pin_memory()
    outh = torch.empty((B, D), dtype=torch.float32).pin_memory()
    lib = sk.lib()
    tun = sk._Tuning(**TUNE)
    # the host-buffer leg runs its own fixed number of steps (the copy ring reaches
    # steady state only after a few calls); it does not depend on --steps
    e2e_steps = max(3, args.e2e_steps)

    def e2e_time(flags):
        for _ in range(8):
            sk._check(lib.sigk_signature_f32(Xh.data_ptr(), B, L, d, N, outh.data_ptr(), flags,
                                             C.c_void_p(stream.cuda_stream), C.byref(tun), None))
        stream.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            sk._check(lib.sigk_signature_f32(Xh.data_ptr(), B, L, d, N, outh.data_ptr(), flags,
                                             C.c_void_p(stream.cuda_stream), C.byref(tun), None))
        e1.record(stream)  # the stream waits for each call's D2H: e1 follows the last result
        e1.synchronize()
        wall = time.perf_counter() - w0
        return max_over_ranks(max(e0.elapsed_time(e1) * 1e-3, wall), world)

    # synchronous host calls (each returns with its result), then the
    # asynchronous host mode a pipelined caller uses (copies of consecutive
    # steps overlap on the copy engines): the e2e headline
    e2e_sync_s = e2e_time(0)
    e2e_s = e2e_time(sk.SIGK_ASYNC_HOST)

    # c5 (strong scaling): the drop-in multi-GPU entry itself, end to end on the
    # global batch from pinned host memory (sigk_signature_sharded_f32: one host
    # thread and copy stream per device, rows split like rank_rows), run by rank 0
    # over all `world` GPUs while the other ranks wait at a barrier
    sharded = None
    if scaling == "strong" and not args.no_sharded:
        barrier(world)
        if rank == 0 and torch.cuda.device_count() >= world:
            Xg = torch.empty((B_global, L, d), dtype=torch.float32).pin_memory()
            piece = torch.empty((min(B_global, 1024), L, d), dtype=torch.float32, device=dev)
            for r0 in range(0, B_global, piece.shape[0]):
                n = min(piece.shape[0], B_global - r0)
                sk.brownian(piece[:n], seed=42, row0=r0)
                Xg[r0:r0 + n].copy_(piece[:n])
            del piece
            outg = torch.empty((B_global, D), dtype=torch.float32).pin_memory()
            st_sh = sk._Stats()

            def sharded_call():
                sk._check(lib.sigk_signature_sharded_f32(Xg.data_ptr(), B_global, L, d, N, outg.data_ptr(), world,
                                                         C.byref(st_sh)))

            sharded_call()
            reps = 3
            w0 = time.perf_counter()
            for _ in range(reps):
                sharded_call()
            wall = time.perf_counter() - w0
            sharded = {"value": B_global * reps / wall, "unit": "paths/s", "gpus": world, "calls": reps,
                       "h2d_bytes_per_step": B_global * L * d * 4, "d2h_bytes_per_step": B_global * D * 4,
                       "api": "sigk_signature_sharded_f32 (C ABI; include/sigk.h): host buffers in and out, rows "
                              "split over the GPUs, one host thread per device; wall clock per synchronous call"}
        barrier(world)

    # parity spot check of this run's output (first rows) against the oracle
    parity = None
    if rank == 0:
        from oracle import oracle as O

        rows = min(B, 8)
        ref = O.signature(Xh[:rows].numpy().astype(np.float64), N, threads=os.cpu_count() or 1)
        got = outh[:rows].numpy().astype(np.float64)
        off = O.level_offsets(d, N)
        parity = max(float(np.abs(got[:, off[n]:off[n + 1]] - ref[:, off[n]:off[n + 1]]).max()
                         / np.abs(ref[:, off[n]:off[n + 1]]).max()) for n in range(N))

    if all_cores:
        os.sched_setaffinity(0, all_cores)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(pool[0].cpu().numpy(), N)
        cpu.pop("seconds_best", None)

    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    steps = args.steps
    B_all = B_global if scaling == "strong" else world * B  # rows all ranks processed per step
    value = B_all * steps / elapsed
    # credited flops of this rank's step (the slowest rank bounds the step interval)
    achieved = B * flops_path / (elapsed / steps) / 1e12
    single_tf = B * flops_path / fold_s / 1e12
    e2e_h2d, e2e_d2h = in_bytes, B * D * 4
    kernel_name = {1: "path_kernel", 2: "flat_kernel", 3: "pair_kernel", 4: "generic_fold_kernel",
                   5: "ipair_kernel"}.get(st.family, "?")
    traffic = _traffic(args.config)
    peaks = load_peaks()
    line = {
        "metric": baseline_metric(),
        "value": value,
        "unit": "paths/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed / steps * 1e3,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic Brownian paths (Philox, X0=0, N(0,1/(L-1)) increments), generated on device",
        "config": {
            "workload": f"{args.config}: B={B_global if scaling == 'strong' else B} L={L} d={d} N={N} fp32 "
                        "batched truncated signature"
                        + (" (BASELINE.json configs[1], headline)" if args.config == "c2" else "")
                        + (f", global batch sharded over {world} GPU(s) (BASELINE.json configs[4])"
                           if scaling == "strong" else " per GPU"),
            "batch_per_gpu": B, "global_batch": B_all, "seq_len": L, "dim": d, "depth": N, "sig_dim": D,
            "parallelism": f"batch-sharded x{world}, no collective",
            "l2": f"L2 flushed (512 MiB write) before the timed region, after an untimed warm-up replay enqueued "
                  f"back to back with it (the GPU is busy up to t0); every step reads a distinct batch of a "
                  f"{n_buf}-batch pool ({n_buf * in_bytes / 2**20:.0f} MiB, > 2x the 126 MB L2) so inputs come "
                  "from HBM",
            "timing": f"{steps} steps = CUDA graph of {S} steps x {reps_full}"
                      + (f" + {rem}" if rem else "") + "; CUDA events on the launch stream; max over ranks",
            "family": sk.FAMILY_NAMES.get(st.family, "?"), "segments": st.segments,
            "chunks": st.chunks, "prefix_len": st.prefix_len, "threads_per_unit": st.threads_per_unit,
            "fold_steps_per_unit": st.fold_steps, "merge_rounds": st.scan_passes,
            "single_launch_ms_eager": single_ms,
            "parity_max_level_rel_err": parity,
        },
        "roofline": {
            "bound": "fp32",
            "kernel": f"{kernel_name} (FFMA-pipe bound; tensor cores deliberately unused, SURVEY.md §8d)",
            "achieved": achieved,
            "peak": peak,
            "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None,
            "frac_of_nominal": achieved / NOMINAL_FP32_TFLOPS,
            "peak_source": "measured: register-resident FFMA microbenchmark on this GPU (sigk_bench_ffma); "
                           f"nominal {NOMINAL_FP32_TFLOPS:.2f}",
            "achieved_from": "credited flops per step / mean step interval of the timed back-to-back graph "
                             "replays (CUDA events around the timed region; includes every kernel of the step "
                             "and the inter-kernel gaps; consecutive launches may overlap via PDL)",
            "kernels_per_step": st.launches,
            "credited_flops_per_launch": B * flops_path,
            "single_call": {"kernel_ms": fold_s * 1e3, "achieved": single_tf,
                            "frac": single_tf / peak if peak else None,
                            "from": "the fold kernel alone: CUDA events around every 4th launch of an untimed "
                                    "graph replay after an L2 flush (no launch overlap); includes the launch "
                                    "latency of an idle GPU (a ~1 us C1 fold measures ~8 us this way, "
                                    "profiles/r02/mode_probe.txt)",
                            "device_span_ms": span_ms,
                            "device_span_frac": {k: B * flops_path / (v * 1e-3) / 1e12 / peak for k, v in span_ms.items()}
                            if peak else None,
                            "device_span_from": "one launch alone after an L2 flush: %globaltimer at every CTA's "
                                                "entry and exit, first entry to last exit (median of 5)",
                            "latency_plan": {"kernel_ms": lat_s * 1e3,
                                             "frac": B * flops_path / lat_s / 1e12 / peak if peak else None,
                                             "chunks": lat_plan.chunks, "segments": lat_plan.segments,
                                             "mode": "sigk_tuning.mode = SIGK_MODE_LATENCY (the plan synchronous "
                                                     "host calls use)"}},
            "hbm": {"algorithmic_bytes_per_launch": B * bytes_path,
                    "achieved_gbs": B * bytes_path / (elapsed / steps) / 1e9,
                    "peak_gbs": peaks.get("hbm_gbs"), "peak_source": "MEASURED_PEAKS.json"},
            "traffic": traffic,
        },
        "cpu_baseline": cpu,
        "e2e": {"value": B_all * e2e_steps / e2e_s, "unit": "paths/s",
                "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h, "steps": e2e_steps,
                "api": "sigk_signature_f32 (C ABI), pinned host buffers, SIGK_ASYNC_HOST: every step copies its "
                       "inputs H2D and its signatures D2H; consecutive steps overlap on the copy engines; timed "
                       "to the last result on the host",
                "link_gbs": {"h2d": e2e_h2d * e2e_steps / e2e_s / 1e9, "d2h": e2e_d2h * e2e_steps / e2e_s / 1e9,
                             "note": "per GPU; PCIe bounds e2e at these shapes (the kernel is ~"
                                     f"{(e2e_s / e2e_steps) / (elapsed / steps):.0f}x faster than the copies)"},
                "synchronous": {"value": B_all * e2e_steps / e2e_sync_s, "unit": "paths/s",
                                "api": "same call without SIGK_ASYNC_HOST (returns with each step's result)"},
                "sharded_entry": sharded},
        "clocks": clk.summary(),
        "gpu_launches": steps * max(1, st.launches),
    }
    print(json.dumps(line), flush=True)


def _step(sk, X, N, out, ev, mode=0):
    import ctypes as C

    import torch

    tun = sk._Tuning(**TUNE)
    if mode:
        tun.mode = mode
    if ev is not None:
        tun.fold_event_start = C.c_void_p(ev[0].cuda_event)
        tun.fold_event_stop = C.c_void_p(ev[1].cuda_event)
    B, L, d = X.shape
    s = torch.cuda.current_stream()
    sk._check(sk.lib().sigk_signature_f32(X.data_ptr(), B, L, d, N, out.data_ptr(),
                                          sk.SIGK_X_ON_DEVICE | sk.SIGK_OUT_ON_DEVICE,
                                          C.c_void_p(s.cuda_stream), C.byref(tun), None))


def _traffic(config):
    """dram bytes per fold launch from the committed ncu --set full capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(config)
    except (OSError, ValueError):
        return None


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the reference compiled
    from its sources; else the C port), all host threads, rank 0 only."""
    import numpy as np

    rank, world, _ = dist_env()
    if rank != 0:
        return
    B, L, d, N = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(42)
    X = np.zeros((B, L, d), np.float64)
    X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / math.sqrt(L - 1), axis=1)
    X = X.astype(np.float32).astype(np.float64)  # same fp32-representable inputs as the GPU arm
    # bounded sample per step: whole waves of `threads` rows, <= ~1 s per step and
    # <= ~90 s for the whole --steps/--warmup run
    t1, kind = cpu_reference_run(X[:threads], N, threads)  # one wave: `threads` rows in parallel
    target = min(1.0, 90.0 / max(1, args.steps + args.warmup))
    rows = int(max(1, min(B, threads * max(1, int(target / max(t1, 1e-6))))))
    Xs = X[:rows]
    for _ in range(args.warmup):
        cpu_reference_run(Xs, N, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, kind = cpu_reference_run(Xs, N, threads)
    dt = time.perf_counter() - t0
    value = rows * args.steps / dt
    # also 1 thread (as shipped) and the <float> instantiation,
    # each on a bounded sample (~3 s), reported beside the headline figure
    var = []
    for prec, Xv in (("f64", X), ("f32", X.astype(np.float32))):
        for th in sorted({1, threads}):
            if prec == "f64" and th == threads:
                continue
            vv, r, n, t, k = cpu_timed(Xv[:rows], N, th, 3.0)
            var.append({"value": vv, "unit": "paths/s", "threads": th, "precision": prec, "kind": k,
                        "sample": f"{r} rows, best of {n} passes ({t:.1f} s)"})
    line = {
        "metric": baseline_metric(), "value": value, "unit": "paths/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": rank_rows(args.config, 1, 0)[3], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic Brownian paths (numpy, seed 42)",
        "impl": "reference",
        "config": {"workload": f"{args.config}: B={B} L={L} d={d} N={N} (CPU, rank 0 only)", "batch_per_step": rows,
                   "seq_len": L, "dim": d, "depth": N},
        "cpu_baseline": {"value": value, "unit": "paths/s", "cores": threads, "kind": kind,
                         "sample": f"{rows} of {B} rows per step, sigkit_ref::detail::sequential_forward<double>, "
                                   f"{threads} threads (rows split over std::thread)",
                         "cpu_model": cpu_model(), "variants": var},
        "e2e": {"value": value, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sharded", action="store_true", help="c5: skip the sigk_signature_sharded_f32 e2e leg")
    ap.add_argument("--chunks", type=int, default=0, help="force chunks per path (0: planned)")
    ap.add_argument("--prefix-len", type=int, default=0, help="force Q (0: planned)")
    ap.add_argument("--segments", type=int, default=0, help="pair family: force CTAs per path (0: planned)")
    ap.add_argument("--family", default="auto", choices=["auto", "path", "flat", "pair", "generic", "pflat"])
    ap.add_argument("--shape", default="", help="experiments: override the config as B,L,d,N")
    args = ap.parse_args()
    if args.shape:
        CONFIGS[args.config] = tuple(int(x) for x in args.shape.split(","))
    fam = {"auto": 0, "path": 1, "flat": 2, "pair": 3, "generic": 4, "pflat": 5}[args.family]
    TUNE.update(chunks=args.chunks, prefix_len=args.prefix_len, segments=args.segments, family=fam)
    if args.impl == "reference":
        args.steps = args.steps or 5
        args.warmup = max(3, 3 if args.warmup is None else args.warmup)
        run_reference(args)
        return
    default_steps = {"c1": 20000, "c2": 20000, "c3": 2000, "c4": 500, "c5": 100}[args.config]
    args.steps = args.steps or default_steps
    args.warmup = max(3, args.warmup if args.warmup is not None else 50)
    run_ours(args)


if __name__ == "__main__":
    main()
