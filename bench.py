"""Benchmark: batched CS-WGS holograms/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
                    [--workload cfg3|cfg4]

--gpus N without torchrun relaunches itself under torch.distributed.run with
N ranks (one per GPU, NCCL); under torchrun the ranks come from the env.

Workload (configs[2] with configs[4]'s batching): CS-WGS,
1152x1152 gaussian pupil (M = 1,042,356), N = 100 random 3D foci
(x, y ~ U(+-100 um), z ~ U(+-50 um), spot seed 1000+k), compression 1/16,
I = 20, solver seed k, followed by the e/u quality report.  One step =
one batch of B independent patterns per GPU (weak scaling: B per rank).

value  : holograms/s over the whole job, inputs resident in HBM, CUDA-event
         timed per step on the solver stream (L2 flushed between steps).
e2e    : the same through the C ABI (hs_solve_host) with pinned host
         buffers: spot + theta0 upload, solve, phase[B][M] float64 +
         e/u download inside the timed region (the phases cross the link as
         4-byte codes and are widened to the identical f64 values on the
         host threads, inside the timed region).
--impl reference : the CPU oracle (bit-exact restatement of the reference
         numba kernels, oracle/) on all host threads, one hologram per step.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # CPU baseline legs only

METRIC = "holograms/sec & ms/hologram (1152², N=100, CS-WGS) at 1/2/4/8 B200 vs CPU; e,u"
SIDE, NSPOTS, COMPRESSION, ITERS = 1152, 100, 1 / 16, 20
FLOP_PER_PAIR_PASS = 8  # one complex MAC per (pixel, spot) per pass


def workload_config(batch, world=1):
    return {"workload": "cswgs_1152_n100_c1/16_i20_batched", "side_px": SIDE,
            "parallelism": f"batch-dp{world} (independent patterns per rank, no data-path "
                           "collective)",
            "spots": NSPOTS, "compression": COMPRESSION, "iterations": ITERS,
            "batch_per_gpu": batch, "pupil": "gaussian waist 6 mm, pitch 9.2 um, "
            "lambda 800 nm, f 20 mm, seed 0", "foci": "uniform xy +-100 um, z +-50 um, "
            "spot seed 1000+k, solver seed k", "l2": "flushed between timed steps "
            "(256 MiB write, outside the step events)"}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def pattern_arrays(first, count):
    import paper_2003_05293_b200 as hs
    sets = [hs.random_foci(NSPOTS, 1000 + k) for k in range(first, first + count)]
    x = np.stack([s.x for s in sets])
    y = np.stack([s.y for s in sets])
    z = np.stack([s.z for s in sets])
    a = np.stack([s.amplitude for s in sets])
    th = np.stack([np.random.default_rng(k).random(NSPOTS) * 2 * math.pi
                   for k in range(first, first + count)])
    return x, y, z, a, th


class Clocks:
    """SM clock + throttle-reason sampler running during the timed region:
    NVML from a thread every 5 ms (the timed region of a default run is
    ~0.1 s), nvidia-smi at 100 ms if NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        import threading
        self.sm, self.mx, self.reasons = [], 0.0, set()
        self.proc = None
        try:
            import pynvml
            pynvml.nvmlInit()
            # CUDA_VISIBLE_DEVICES order == NVML order is not guaranteed; map by bus id
            import torch
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            try:   # match the CUDA device by PCI bus id (CUDA and NVML orders may differ)
                want = str(torch.cuda.get_device_properties(index).pci_bus_id).lower()[-7:]
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                    bid = pynvml.nvmlDeviceGetPciInfo(hi).busId
                    bid = (bid.decode() if isinstance(bid, bytes) else str(bid)).lower()
                    if bid[-7:] == want:
                        h = hi
                        break
            except Exception:
                pass
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            masks = [(nm, getattr(pynvml, attr)) for nm, attr in self.REASONS]
            self.stop_flag = threading.Event()

            def loop():
                while not self.stop_flag.is_set():
                    self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for nm, mask in masks:
                        if r & mask:
                            self.reasons.add(nm)
                    self.stop_flag.wait(0.005)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            self.kind = "nvml"
        except Exception:
            self.kind = "smi"
            self.path = tempfile.mktemp(suffix=".csv")
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(index),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            except OSError:
                self.proc = None

    def stop(self):
        if self.kind == "nvml":
            self.stop_flag.set()
            self.thread.join()
        elif self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            names = [nm for nm, _ in self.REASONS]
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    self.sm.append(float(parts[0]))
                    self.mx = max(self.mx, float(parts[1]))
                except ValueError:
                    continue
                for nm, flag in zip(names, parts[3:7]):
                    if flag.lower() == "active":
                        self.reasons.add(nm)
            os.unlink(self.path)
        if not self.sm:
            return None
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "sampler": self.kind}


def host_threads():
    """All host cores this process may run on (torchrun pins OMP_NUM_THREADS=1,
    the oracle's OpenMP regions take an explicit thread count instead)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_rate(seconds=10.0, threads=None):
    """Oracle (bit-exact reference restatement) holograms/s on host cores."""
    import oracle
    import paper_2003_05293_b200 as hs
    pupil = hs.build_pupil(SIDE)
    threads = threads or host_threads()
    done, t0 = 0, time.perf_counter()
    while True:
        s = hs.random_foci(NSPOTS, 1000 + done)
        r = oracle.solve(pupil, s.x, s.y, s.z, s.amplitude, "cswgs", ITERS, COMPRESSION,
                         seed=done, threads=threads)
        oracle.quality(pupil, r["tables"], r["phase"], s.amplitude, threads=threads)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el, done, threads


def _pool_worker(job):
    """One process of the process-pool CPU leg: single-threaded oracle solves
    (+ e/u) of the workload until the deadline."""
    seconds, first = job
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    import paper_2003_05293_b200 as hs
    pupil = hs.build_pupil(SIDE)
    done, eu, t0 = 0, [], time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        k = first + done
        s = hs.random_foci(NSPOTS, 1000 + k)
        r = oracle.solve(pupil, s.x, s.y, s.z, s.amplitude, "cswgs", ITERS, COMPRESSION, seed=k, threads=1)
        eu.append(oracle.quality(pupil, r["tables"], r["phase"], s.amplitude, threads=1)[:2])
        done += 1
    return done, time.perf_counter() - t0, eu


def cpu_pool_rate(seconds, procs):
    """Holograms/s of `procs` single-threaded oracle processes (the reference
    bench's ProcessPoolExecutor variant, which beat its threads: SURVEY 8(d))."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    with ProcessPoolExecutor(procs, mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_pool_worker, [(seconds, 100000 * (i + 1)) for i in range(procs)]))
    rate = sum(d / el for d, el, _ in res)
    return rate, sum(d for d, _, _ in res), [x for _, _, e in res for x in e]


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import oracle
    import paper_2003_05293_b200 as hs
    oracle.build()
    pupil = hs.build_pupil(SIDE)
    threads = host_threads()

    def step(k):
        s = hs.random_foci(NSPOTS, 1000 + k)
        r = oracle.solve(pupil, s.x, s.y, s.z, s.amplitude, "cswgs", ITERS, COMPRESSION,
                         seed=k, threads=threads)
        return oracle.quality(pupil, r["tables"], r["phase"], s.amplitude, threads=threads)

    for w in range(args.warmup):
        step(w)
    t0 = time.perf_counter()
    eu = [step(args.warmup + k)[:2] for k in range(args.steps)]
    el = time.perf_counter() - t0
    thread_rate = args.steps / el
    # the process-pool variant (one single-threaded solver per core), run for
    # as long as the threaded leg; the better of the two is the reference rate
    pool_rate, pool_done, pool_eu = cpu_pool_rate(min(max(el, 5.0), 60.0), threads)
    val = max(thread_rate, pool_rate)
    variant = "process pool" if pool_rate > thread_rate else "threads"
    if pool_rate > thread_rate:
        eu = pool_eu
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "holograms/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.batch, world),
            "sample_per_step": "1 hologram of the batched workload per step (a bounded "
                               "sample; holograms are independent, so the rate is per hologram)",
            "cpu_baseline": {"value": val, "unit": "holograms/s", "cores": threads,
                             "kind": "port", "cpu_model": cpu_model(),
                             "threading": f"{variant} (the better of: OpenMP threads over the "
                                          "reference's prange units, "
                                          f"{thread_rate:.3f} holo/s; {threads} single-threaded "
                                          f"processes, {pool_rate:.3f} holo/s)",
                             "sample": f"{args.steps} holograms of the workload, 1 per step, "
                             f"threaded; {pool_done} holograms in the process pool "
                             "(C+OpenMP oracle, bit-exact vs reference)"},
            "e2e": {"value": val, "unit": "holograms/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "mean_e": float(np.mean([e for e, _ in eu])),
            "mean_u": float(np.mean([u for _, u in eu]))}
    print(json.dumps(line), flush=True)


def umma_roofline(pupil, batch, n, ms):
    """Tensor-pipe roofline of the tcgen05 full pass (csrc/hs_umma.cuh):
    executed kind::f16 MMA flops per launch (128-row x 64-column tiles over
    the aperture's row bands; per complex 16-deep k-step 6 backward MMAs
    (N = 128) and 12 forward MMAs (N = np): a 2-term fp16 hi/lo split, 3
    products per real product) against the measured dense bf16 peak (fp16
    runs at the bf16 rate)."""
    side = pupil.side_px
    rows = np.asarray(pupil.rows)
    cols = np.asarray(pupil.cols)
    kuf = 16  # K per f16 MMA (columns / spots per k-step)
    tiles = 0
    for r0 in range(0, side, 128):
        sel = (rows >= r0) & (rows < r0 + 128)
        if sel.any():
            lo, hi = int(cols[sel].min()) & ~(kuf - 1), int(cols[sel].max()) + 1
            tiles += -(-(hi - lo) // 64)
    npad = -(-n // 16) * 16
    ksteps = -(-n // kuf)
    flop = tiles * batch * 2 * 128 * kuf * (6 * 128 * ksteps + 12 * (64 // kuf) * npad)
    peaks = {}
    ppath = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(ppath):
        peaks = json.load(open(ppath))
    bf16 = peaks.get("bf16_tflops")
    peak = bf16 if bf16 else 2250.0
    achieved = flop / (ms * 1e-3) / 1e12
    return {"bound": "tensor", "executed_f16_flop_per_launch": flop, "tiles_per_pattern": tiles,
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (dense f16 = bf16 rate)"
            if bf16 else "B200_PROFILING.md nominal dense bf16/fp16 2.25 PFLOP/s",
            "note": "executed f16 flops include the 2-term split (3 products per real product) and "
                    "tile / spot padding; tensor pipe ~29% active by ncu: per tile the b and E "
                    "epilogues (CUDA cores) run serially with the MMAs inside a CTA and overlap only "
                    "across the SM's two CTAs (per-tile timeline: csrc/hs_umma.cuh, HS_PROBES=1 build "
                    "with HS_UMMA_TRACE=1)"}


def run_ours(args):
    import torch
    import paper_2003_05293_b200 as hs
    from paper_2003_05293_b200 import _lib

    rank, local, world = dist_env()
    ndev = torch.cuda.device_count()
    # one process per GPU; ranks beyond the visible GPUs (a multi-rank smoke
    # run on a 1-GPU box) share devices and time through gloo instead of NCCL
    shared = world > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
    coll_dev = "cpu" if shared else f"cuda:{local}"
    _lib.set_device(local)
    B = args.batch
    pupil = hs.build_pupil(SIDE)
    m = pupil.active_count
    subset = math.ceil(COMPRESSION * m)
    plan = _lib.Plan(pupil, local)
    first = rank * B
    x, y, z, a, th = pattern_arrays(first, B)
    plan.set_spot_arrays(x, y, z, a)
    stream = torch.cuda.ExternalStream(plan.stream(), device=torch.device("cuda", local))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        plan.solve(_lib.ALG_CSWGS, ITERS, subset, th, want_fields=True, sync=True)
    launches_per_step = plan.last_launch_count()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = Clocks(local)
    barrier()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(k))
            starts[k].record(stream)
        plan.solve(_lib.ALG_CSWGS, ITERS, subset, th, want_fields=True, sync=False)
        ends[k].record(stream)
    barrier()
    clk = clocks.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(step_ms))
    status, _ = plan.status()
    e, u, _, _, _ = plan.quality_batch()
    if np.any(status != 0):
        raise RuntimeError(f"solver failed on patterns {np.nonzero(status)[0]}")
    if dist is not None:
        t = torch.tensor([total_ms], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * B * args.steps / (total_ms * 1e-3)

    # single-hologram latency (B = 1) on the same stream
    lat_plan = _lib.Plan(pupil, local)
    lat_plan.set_spot_arrays(x[:1], y[:1], z[:1], a[:1])
    for _ in range(3):
        lat_plan.solve(_lib.ALG_CSWGS, ITERS, subset, th[:1], want_fields=True)
    ls = torch.cuda.ExternalStream(lat_plan.stream(), device=torch.device("cuda", local))
    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    l0.record(ls)
    for _ in range(reps):
        lat_plan.solve(_lib.ALG_CSWGS, ITERS, subset, th[:1], want_fields=True, sync=False)
    l1.record(ls)
    torch.cuda.synchronize()
    latency_ms = l0.elapsed_time(l1) / reps

    # e2e through the C ABI with pinned host buffers
    lib = _lib.load()
    n_in = B * NSPOTS
    h2d = 5 * n_in * 8
    bufs = {}
    for name, count in (("x", n_in), ("y", n_in), ("z", n_in), ("a", n_in), ("th", n_in),
                        ("ph", B * m), ("e", B), ("u", B)):
        p = lib.hs_host_alloc(count * 8)
        if not p:
            raise MemoryError("cudaHostAlloc failed")
        bufs[name] = (p, np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)),
                                               shape=(count,)))
    for name, src in (("x", x), ("y", y), ("z", z), ("a", a), ("th", th)):
        bufs[name][1][:] = src.ravel()
    e2e_plan = _lib.Plan(pupil, local)

    def e2e_call():
        # pipelined C-ABI call: inputs from pinned host memory, phase[B][M]
        # float64 + e/u back to pinned host memory; the phase download of
        # step k overlaps the solve of step k+1 (hs_solve_host_async)
        _lib.check(lib.hs_solve_host_async(e2e_plan.handle, _lib.ALG_CSWGS, ITERS, subset, B,
                                           NSPOTS, bufs["x"][0], bufs["y"][0], bufs["z"][0],
                                           bufs["a"][0], bufs["th"][0], bufs["ph"][0],
                                           bufs["e"][0], bufs["u"][0]))

    for _ in range(2):
        e2e_call()
    e2e_plan.sync()
    barrier()
    e2e_steps = max(3, args.steps)  # pipeline fill + drain amortised over the run
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_plan.sync()
    e2e_s = time.perf_counter() - t0
    # fp32 solves ship part of the batch as f64 (widened on the device) and
    # the rest as 4-byte codes (widened on the host threads); fp64 ones f64
    nb64 = ctypes.c_int(B)
    if e2e_plan.last_precision() == "fp32":
        _lib.check(lib.hs_host_copy_split(e2e_plan.handle, B, ctypes.byref(nb64)))
    d2h = m * (8 * nb64.value + 4 * (B - nb64.value)) + 2 * B * 8
    e2e_phase_ok = bool(np.array_equal(bufs["ph"][1].reshape(B, m)[:2], e2e_plan.phases(0, 2)))
    if dist is not None:
        t = torch.tensor([e2e_s], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * B * e2e_steps / e2e_s
    e2e_ok = bool(np.allclose(bufs["e"][1], e, rtol=0, atol=0))
    for p, _ in bufs.values():
        lib.hs_host_free(p)

    # roofline of the dominant kernel (the compressed-window pass: 19 of the
    # 22 launches, ~57% of the step) and of the full-range pass, each timed
    # live with CUDA events on the plan stream (hs_time_kernel)
    ms_full, pairs_full = plan.time_kernel(0, reps=10)
    ms_final, _ = plan.time_kernel(3, reps=10)  # last iteration's pass: + phase-code scatter
    ms_win, pairs_win = plan.time_kernel(1, subset, reps=50)
    peak = _lib.fma_peak_tflops(local)
    flops_win = 2 * FLOP_PER_PAIR_PASS * pairs_win     # backward + forward per pair
    flops_full = 2 * FLOP_PER_PAIR_PASS * pairs_full
    achieved_win = flops_win / (ms_win * 1e-3) / 1e12
    achieved_full = flops_full / (ms_full * 1e-3) / 1e12
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    n_full, n_win = 2, ITERS - 1
    step_kernel_ms = ms_full + ms_final + n_win * ms_win
    tensor = umma_roofline(pupil, B, NSPOTS, ms_full)

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        rate, done, threads = cpu_oracle_rate(args.cpu_seconds)
        rate1, done1, _ = cpu_oracle_rate(max(2.0, args.cpu_seconds / 2), threads=1)
        prate, pdone, _ = cpu_pool_rate(args.cpu_seconds, threads)
        cpu = {"value": max(rate, prate), "unit": "holograms/s", "cores": threads, "kind": "port",
               "cpu_model": cpu_model(), "threading": "the better of OpenMP (libgomp) threads over the "
               "reference's prange units (pixels for the backward pass, 1024-pixel chunks forward) "
               "and a process pool of single-threaded solvers (SURVEY 8(d), config 5)",
               "threads": {"value": rate, "unit": "holograms/s", "cores": threads,
                           "sample": f"{done} holograms"},
               "process_pool": {"value": prate, "unit": "holograms/s", "processes": threads,
                                "sample": f"{pdone} holograms"},
               "workers_1": {"value": rate1, "unit": "holograms/s", "cores": 1,
                             "sample": f"{done1} holograms"},
               "sample": f"{done} holograms of the workload (CS-WGS 1152^2 N=100 I=20 + e/u), "
               "C+OpenMP oracle bit-exact vs the reference numba kernels"}
    pairs_step = B * NSPOTS * (2 * 2 * m + 2 * (ITERS - 1) * subset)
    line = {
        "metric": METRIC, "value": value, "unit": "holograms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "ms_per_hologram": total_ms / args.steps / B,
        "latency_ms_single_hologram": latency_ms,
        "latency_ms_per_iteration": latency_ms / (ITERS + 1),  # I + 1 passes per solve (DESIGN 3)
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic", "config": workload_config(B, world),
        "e2e": {"value": e2e_value, "unit": "holograms/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps, "matches_device_e": e2e_ok,
                "phase_matches_hs_get_phase": e2e_phase_ok,
                "f64_patterns_per_step": nb64.value,
                "path": "hs_solve_host_async (C ABI, pinned host buffers; f64 storage-order "
                        "phases: f64_patterns_per_step of the batch widened on the device and "
                        "copied as f64, the rest copied as 4-byte codes and widened to the "
                        "identical f64 on the host threads; copy + widening of step k overlap "
                        "the solve of step k+1)"},
        "roofline": {"bound": "fma", "achieved": achieved_win, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved_win / peak,
                     "traffic": traffic.get("window_pass_dram_bytes_per_launch"),
                     "kernel": "hs_slab_kernel<7> compressed-window fused pass (backward + "
                               "forward + fold/update), dominant: 38 of 44 launches per step "
                               "(two graph branches of 16 patterns)",
                     "peak_source": "measured FP32 FFMA microbenchmark (hs_fma_peak, "
                                    "MEASURED_PEAKS.json has no FP32 figure)",
                     "algorithmic_flop_per_launch": flops_win,
                     "flop_per_unit": 16, "unit_def": "pixel-spot pair (backward + forward "
                     "complex MAC, SURVEY 8(d)); units per launch = S * N * B",
                     "ms_per_launch": ms_win,
                     "step_share_estimate": n_win * ms_win / step_kernel_ms,
                     "full_pass": {"kernel": "hs_umma_kernel<112> tcgen05 kind::f16 (2-term fp16 split) "
                                             "128x64-pixel tiles",
                                   "ms_per_launch": ms_full,
                                   "final_pass_ms_per_launch": ms_final,
                                   "achieved_fp32_equivalent": achieved_full,
                                   "algorithmic_flop_per_launch": flops_full,
                                   "tensor": tensor,
                                   "traffic": traffic.get("full_pass_dram_bytes_per_launch")},
                     "step_kernel_ms_estimate": step_kernel_ms},
        "pixel_spot_pairs_per_step": pairs_step,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk, "cpu_baseline": cpu,
        "mean_e": float(np.mean(e)), "mean_u": float(np.mean(u)),
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args):
    """bench.py --gpus N outside torchrun: run N ranks under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


CFG4_SPOTS, CFG4_ITERS = 1000, 30


PANEL_W, PANEL_H = 1920, 1152   # the paper's SLM


def cfg4_config(world, rect=False):
    if rect:
        return {"workload": "wgs_panel1920x1152_n1000_i30_rowsharded", "panel_px": [PANEL_H, PANEL_W],
                "active_pixels": PANEL_W * PANEL_H, "spots": CFG4_SPOTS, "iterations": CFG4_ITERS,
                "algorithm": "wgs",
                "parallelism": f"row-sharded x{world} (group partials exchanged over peer memory "
                               "each pass)" if world > 1 else "single GPU",
                "pupil": "full rectangular 1920x1152 panel (build_panel), gaussian waist 6 mm, "
                         "pitch 9.2 um, lambda 800 nm, f 20 mm, seed 0",
                "foci": "uniform xy +-150 um, z +-50 um, spot seed 4, solver seed 0",
                "l2": "inputs (tables, lists) L2-resident; one solve = 31 full passes"}
    return {"workload": "wgs_1152_n1000_i30_rowsharded", "side_px": SIDE, "spots": CFG4_SPOTS,
            "iterations": CFG4_ITERS, "algorithm": "wgs",
            "parallelism": f"row-sharded x{world} (one hologram cut at fold-group boundaries; "
                           "group partials exchanged over peer memory each pass)" if world > 1
            else "single GPU", "pupil": "gaussian waist 6 mm, pitch 9.2 um, lambda 800 nm, "
            "f 20 mm, seed 0", "foci": "uniform xy +-150 um, z +-50 um, spot seed 4, solver seed 0",
            "l2": "inputs (tables, lists) L2-resident; one solve = 31 full passes"}


def run_cfg4(args, rect=False):
    """BASELINE configs[3]: WGS N = 1000, I = 30 on the 1152^2 circular
    aperture (the parity stand-in) or, with rect=True, on the
    full 1920x1152 panel itself (build_panel; throughput-only) -- one
    hologram per step, row-sharded across the ranks (distributed.
    solve_sharded's device path: peer-memory exchange of the group partials,
    csrc/hs_xchg.cuh).  Strong scaling: the work per step is fixed; value =
    holograms/s of the whole job."""
    import torch
    import paper_2003_05293_b200 as hs
    from paper_2003_05293_b200 import _lib
    from paper_2003_05293_b200.solvers import _theta0

    rank, local, world = dist_env()
    ndev = torch.cuda.device_count()
    shared = world > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    _lib.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coll_dev = "cpu" if shared else f"cuda:{local}"

    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    pupil = hs.build_panel(PANEL_W, PANEL_H) if rect else hs.build_pupil(SIDE)
    m = pupil.active_count
    spots = hs.random_foci(CFG4_SPOTS, 4, xy=150e-6)
    plan = _lib.Plan(pupil, local)
    plan.set_spots(spots)
    th = _theta0(0, CFG4_SPOTS)[None, :]
    stream = torch.cuda.ExternalStream(plan.stream(), device=torch.device("cuda", local))

    if world > 1:
        plan.shard_begin(_lib.ALG_WGS, CFG4_ITERS, m, th, rank, world)
        plan.p2p_open(all_gather(plan.p2p_setup()))

        def solve():
            plan.shard_begin(_lib.ALG_WGS, CFG4_ITERS, m, th, rank, world)
            plan.p2p_solve()  # all passes as one captured graph (hs_shard_p2p_solve)
    else:
        def solve():
            plan.solve(_lib.ALG_WGS, CFG4_ITERS, m, th, want_fields=True, sync=False)

    for _ in range(args.warmup):
        solve()
        plan.sync()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = Clocks(local)
    for k in range(args.steps):
        starts[k].record(stream)
        solve()
        ends[k].record(stream)
    plan.sync()
    clk = clocks.stop()
    total_ms = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
    status, _ = plan.status()
    e, u, *_ = plan.quality_batch()
    if dist is not None:
        codes = all_gather(int(status[0]))
        t = torch.tensor([total_ms], device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        if world > 1:
            plan.p2p_close()
    else:
        codes = [int(status[0])]
    if any(codes):
        raise RuntimeError(f"sharded solve failed: {codes}")
    if rank != 0:
        return
    flop = 2 * FLOP_PER_PAIR_PASS * CFG4_SPOTS * m * (CFG4_ITERS + 1)
    ms = total_ms / args.steps
    line = {"metric": "holograms/s (config 4: WGS 1920x1152 panel, N=1000, I=30, row-sharded)" if rect
            else "holograms/s (config 4: WGS 1152^2, N=1000, I=30, row-sharded)",
            "value": 1e3 / ms, "unit": "holograms/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_per_hologram": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic", "config": cfg4_config(world, rect),
            "achieved_tflops_fp32_equivalent": flop / (ms * 1e-3) / 1e12,
            "e": float(e[0]), "u": float(u[0]),
            **({} if rect else {"reference_e_u": [0.906461, 0.158003]}), "clocks": clk,
            "gpu_launches": plan.last_launch_count() * args.steps if world == 1 else
            (2 + 3 * (CFG4_ITERS + 1)) * args.steps,
            "shared_gpu": shared}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg4", "cfg4rect"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    elif args.workload in ("cfg4", "cfg4rect"):
        run_cfg4(args, rect=args.workload == "cfg4rect")
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
