"""Break down the e2e (C ABI, host buffers) cost of the bench workload.

    python tools/e2e_probe.py [--batch 32] [--steps 10]

Prints: device-resident solve rate, pinned D2H bandwidth of the phase
buffer, and hs_solve_host_async rates with and without the phase download.
"""
import argparse
import ctypes
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_05293_b200 as hs  # noqa: E402
from paper_2003_05293_b200 import _lib  # noqa: E402
print("HS_E2E_F64_FRAC", os.environ.get("HS_E2E_F64_FRAC"), "HS_WIDEN_THREADS", os.environ.get("HS_WIDEN_THREADS"), "HS_E2E_CODES", os.environ.get("HS_E2E_CODES"))

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
B, N = args.batch, 100
pupil = hs.build_pupil(1152)
m = pupil.active_count
subset = math.ceil(m / 16)
sets = [hs.random_foci(N, 1000 + k) for k in range(B)]
x = np.stack([s.x for s in sets]); y = np.stack([s.y for s in sets])
z = np.stack([s.z for s in sets]); a = np.stack([s.amplitude for s in sets])
th = np.stack([np.random.default_rng(k).random(N) * 2 * math.pi for k in range(B)])
lib = _lib.load()


def pinned(count):
    p = lib.hs_host_alloc(count * 8)
    return p, np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(count,))


bufs = {k: pinned(v) for k, v in (("x", B * N), ("y", B * N), ("z", B * N), ("a", B * N), ("th", B * N),
                                   ("ph", B * m), ("e", B), ("u", B))}
for k, v in (("x", x), ("y", y), ("z", z), ("a", a), ("th", th)):
    bufs[k][1][:] = v.ravel()
plan = _lib.Plan(pupil, 0)


def call(phase=True):
    _lib.check(lib.hs_solve_host_async(plan.handle, _lib.ALG_CSWGS, 20, subset, B, N, bufs["x"][0],
                                       bufs["y"][0], bufs["z"][0], bufs["a"][0], bufs["th"][0],
                                       bufs["ph"][0] if phase else None, bufs["e"][0], bufs["u"][0]))


for phase in (True, False):
    for _ in range(3):
        call(phase)
    plan.sync()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        call(phase)
    plan.sync()
    dt = (time.perf_counter() - t0) / args.steps
    print(f"hs_solve_host_async phase={phase}: {dt * 1e3:.2f} ms/step, {B / dt:.0f} holo/s")

dev = torch.empty(B * m, dtype=torch.float64, device="cuda")
host = torch.from_numpy(bufs["ph"][1])
torch.cuda.synchronize()
for _ in range(2):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    host.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"pinned D2H {B * m * 8 / 1e6:.0f} MB: {dt * 1e3:.2f} ms = {B * m * 8 / dt / 1e9:.1f} GB/s")

# concurrency: one device-resident solve with a 267 MB D2H running beside it
plan2 = _lib.Plan(pupil, 0)
plan2.set_spot_arrays(x, y, z, a)
for _ in range(2):
    plan2.solve(_lib.ALG_CSWGS, 20, subset, th, want_fields=True, sync=True)
side = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
plan2.solve(_lib.ALG_CSWGS, 20, subset, th, want_fields=True, sync=True)
solo = time.perf_counter() - t0
t0 = time.perf_counter()
with torch.cuda.stream(side):
    host.copy_(dev, non_blocking=True)
plan2.solve(_lib.ALG_CSWGS, 20, subset, th, want_fields=True, sync=False)
ev = torch.cuda.Event()
ev.record(side)
plan2.sync()
t_solve = time.perf_counter() - t0
ev.synchronize()
t_both = time.perf_counter() - t0
print(f"solve alone {solo * 1e3:.2f} ms; with concurrent D2H: solve done {t_solve * 1e3:.2f} ms, "
      f"both done {t_both * 1e3:.2f} ms")

# timeline: event after each pipelined call on the plan stream
ps = torch.cuda.ExternalStream(plan.stream())
evs = []
for _ in range(3):
    call(True)
plan.sync()
t0 = time.perf_counter()
host_t = []
for k in range(8):
    call(True)
    host_t.append(time.perf_counter() - t0)
    e = torch.cuda.Event(enable_timing=True)
    e.record(ps)
    evs.append(e)
plan.sync()
gaps = [evs[i].elapsed_time(evs[i + 1]) for i in range(len(evs) - 1)]
print("solve-completion gaps (ms):", " ".join(f"{g:.2f}" for g in gaps))
print("host enqueue times (ms):", " ".join(f"{t * 1e3:.2f}" for t in host_t))

# host widening of 4-byte phase codes (hs_widen_phases, csrc/hs_host.cu)
lib.hs_widen_phases.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
lib.hs_widen_phases.restype = None
src = lib.hs_host_alloc(B * m * 4)
srcv = np.ctypeslib.as_array(ctypes.cast(src, ctypes.POINTER(ctypes.c_float)), shape=(B * m,))
srcv[:] = np.random.default_rng(0).uniform(-3.14, 3.14, B * m).astype(np.float32)
for _ in range(2):
    lib.hs_widen_phases(src, bufs["ph"][0], B * m)
t0 = time.perf_counter()
for _ in range(5):
    lib.hs_widen_phases(src, bufs["ph"][0], B * m)
dt = (time.perf_counter() - t0) / 5
print(f"host widening {B * m / 1e6:.1f} M codes: {dt * 1e3:.2f} ms")
dev32 = torch.empty(B * m, dtype=torch.float32, device="cuda")
host32 = torch.from_numpy(srcv)
t0 = time.perf_counter()
for _ in range(5):
    host32.copy_(dev32, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"pinned D2H {B * m * 4 / 1e6:.0f} MB: {dt * 1e3:.2f} ms")
# widening while a D2H runs
t0 = time.perf_counter()
host.copy_(dev, non_blocking=True)
lib.hs_widen_phases(src, bufs["ph"][0], B * m)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"widening with a concurrent 267 MB D2H: {(t1 - t0) * 1e3:.2f} ms (both {(time.perf_counter() - t0) * 1e3:.2f})")
