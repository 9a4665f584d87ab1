"""ctypes binding of ``libholospots_b200.so`` (include/holospots_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute entry point raises :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

from .errors import (DegenerateFieldError, DeviceError, GeometryMismatchError,
                     InvalidParameterError, UndefinedUniformityError,
                     ZeroIlluminationError)

LIB_PATH = os.environ.get("HS_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libholospots_b200.so")

HS_OK, HS_EINVAL, HS_EGEOMETRY, HS_EDEGENERATE, HS_EDIVERGED, HS_ECUDA, \
    HS_EZEROILLUM, HS_EUNDEFINED = range(8)
ALG_RS, ALG_WGS, ALG_CSWGS = 0, 1, 2
WANT_FIELDS = 1
WANT_RASTER = 2
WANT_PHASE32 = 4   # fp32 solves ship 4-byte phase codes, widened on the host (same f64 bits)
PREC_AUTO, PREC_FP32, PREC_FP64 = 0, 1, 2
PRECISIONS = {"auto": PREC_AUTO, "fp32": PREC_FP32, "fp64": PREC_FP64}

_ERRORS = {
    HS_EINVAL: InvalidParameterError,
    HS_EGEOMETRY: GeometryMismatchError,
    HS_EDEGENERATE: DegenerateFieldError,
    HS_EDIVERGED: DegenerateFieldError,
    HS_ECUDA: DeviceError,
    HS_EZEROILLUM: ZeroIlluminationError,
    HS_EUNDEFINED: UndefinedUniformityError,
}

# Every symbol include/holospots_b200.h declares (tests check the exports).
EXPORTS = (
    "hs_last_error", "hs_device_count", "hs_max_spots", "hs_plan_create",
    "hs_plan_destroy", "hs_set_spots", "hs_superpose", "hs_forward", "hs_quality",
    "hs_solve_async", "hs_solve", "hs_sync", "hs_get_status", "hs_get_trace",
    "hs_get_phase", "hs_get_quality", "hs_solve_host", "hs_plan_stream",
    "hs_last_launch_count", "hs_time_kernel", "hs_fma_peak", "hs_host_alloc",
    "hs_host_free", "hs_probe", "hs_solve_host_async", "hs_shard_begin", "hs_shard_pass",
    "hs_shard_update", "hs_padded_spots", "hs_shard_groups", "hs_raster", "hs_get_raster",
    "hs_shard_p2p_setup", "hs_shard_p2p_open", "hs_shard_p2p_pass", "hs_shard_p2p_solve", "hs_shard_p2p_close",
    "hs_set_precision", "hs_get_precision", "hs_get_tables", "hs_set_tables",
    "hs_debug_update", "hs_host_copy_split",
)

IPC_HANDLE_BYTES = 64  # HS_IPC_HANDLE_BYTES

_lib = None
_lock = threading.Lock()


def load():
    """Load the CUDA library (raises DeviceError if it was never built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"CUDA library not built ({LIB_PATH}); run "
                "`python -m paper_2003_05293_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        PP = ctypes.POINTER(ctypes.c_void_p)
        sig = {
            "hs_last_error": (ctypes.c_char_p, []),
            "hs_device_count": (I, [ctypes.POINTER(I)]),
            "hs_max_spots": (I, []),
            "hs_plan_create": (I, [I, I, I64, P, P, P, P, D, D, D, PP]),
            "hs_plan_destroy": (None, [P]),
            "hs_set_spots": (I, [P, I, I, P, P, P, P]),
            "hs_superpose": (I, [P, P, P, I64, I64, P]),
            "hs_forward": (I, [P, P, I64, I64, P]),
            "hs_quality": (I, [P, P, P, P, P, P, P]),
            "hs_solve_async": (I, [P, I, I, I64, P, I]),
            "hs_solve": (I, [P, I, I, I64, P, I]),
            "hs_sync": (I, [P]),
            "hs_get_status": (I, [P, P, P]),
            "hs_get_trace": (I, [P, P, P]),
            "hs_get_phase": (I, [P, I, I, P]),
            "hs_get_quality": (I, [P, P, P, P, P, P]),
            "hs_solve_host": (I, [P, I, I, I64, I, I, P, P, P, P, P, P, P, P]),
            "hs_solve_host_async": (I, [P, I, I, I64, I, I, P, P, P, P, P, P, P, P]),
            "hs_plan_stream": (P, [P]),
            "hs_last_launch_count": (I, [P, ctypes.POINTER(I64)]),
            "hs_time_kernel": (I, [P, I, I64, I, ctypes.POINTER(D), ctypes.POINTER(D)]),
            "hs_fma_peak": (I, [I, ctypes.POINTER(D)]),
            "hs_shard_begin": (I, [P, I, I, I64, P, I, I]),
            "hs_shard_pass": (I, [P, I, P, ctypes.POINTER(I), ctypes.POINTER(I), ctypes.POINTER(I)]),
            "hs_shard_update": (I, [P, I, P, I]),
            "hs_raster": (I, [P, P, P, P]),
            "hs_get_raster": (I, [P, I, I, P]),
            "hs_shard_groups": (I, [P, I, ctypes.POINTER(I), ctypes.POINTER(I), ctypes.POINTER(I)]),
            "hs_padded_spots": (I, [P]),
            "hs_probe": (I, [P, P, I64, P, I, P]),
            "hs_host_alloc": (P, [I64]),
            "hs_host_free": (None, [P]),
            "hs_shard_p2p_setup": (I, [P, P]),
            "hs_shard_p2p_open": (I, [P, P]),
            "hs_shard_p2p_pass": (I, [P, I]),
            "hs_shard_p2p_solve": (I, [P]),
            "hs_shard_p2p_close": (I, [P]),
            "hs_set_precision": (I, [P, I]),
            "hs_get_precision": (I, [P, ctypes.POINTER(I), ctypes.POINTER(I)]),
            "hs_get_tables": (I, [P, P, P, P, P]),
            "hs_set_tables": (I, [P, I, P, P, P, P]),
            "hs_debug_update": (I, [I, P, P, P, P, ctypes.POINTER(I), ctypes.POINTER(I)]),
            "hs_host_copy_split": (I, [P, I, ctypes.POINTER(I)]),
        }
        for name, (res, args) in sig.items():
            if os.environ.get("HS_LIB_PATH") and not hasattr(lib, name):
                continue  # an older build under A/B test (tools/ab_time.py)
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != HS_OK:
        msg = (load().hs_last_error() or b"").decode(errors="replace")
        raise _ERRORS.get(rc, DeviceError)(msg or f"holospots_b200 status {rc}")


def device_count() -> int:
    n = ctypes.c_int(0)
    check(load().hs_device_count(ctypes.byref(n)))
    return n.value


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


_default_device = int(os.environ.get("HOLOSPOTS_DEVICE", "0"))


def set_device(index: int) -> None:
    """Select the CUDA device new plans bind to (one process per GPU)."""
    global _default_device
    _default_device = int(index)


def get_device() -> int:
    return _default_device


_precision = os.environ.get("HS_PRECISION", "auto")
if _precision not in PRECISIONS:
    _precision = "auto"


def set_precision(mode: str) -> None:
    """Pixel-pass arithmetic of every plan: "auto" (default), "fp32", "fp64".

    The reference computes in fp64 throughout.  "fp32" runs the fast fp32
    pixel kernels (fp64 tables, folds and updates); "fp64" runs every pixel
    product in fp64; "auto" picks fp64 when the smallest pixel set a call
    projects over holds fewer than 512 pixels per spot (or n > 1024), where
    WGS amplifies fp32 rounding past the parity tolerances."""
    global _precision
    if mode not in PRECISIONS:
        raise InvalidParameterError(f"precision must be one of {sorted(PRECISIONS)}, got {mode!r}")
    _precision = mode


def get_precision() -> str:
    return _precision


class Plan:
    """One pupil's geometry resident on one device (hs_plan)."""

    def __init__(self, pupil, device: int | None = None):
        lib = load()
        if device_count() < 1:
            raise DeviceError("no CUDA device visible; the B200 path has no CPU fallback")
        self.device = get_device() if device is None else int(device)
        self.m = pupil.active_count
        self.side = pupil.side_px
        h = ctypes.c_void_p()
        rows = np.ascontiguousarray(pupil.rows, dtype=np.int64)
        cols = np.ascontiguousarray(pupil.cols, dtype=np.int64)
        amp = f64(pupil.amplitude)
        axis = f64(pupil.axis_coords())
        check(lib.hs_plan_create(self.device, self.side, self.m, ptr(rows), ptr(cols), ptr(amp),
                                 ptr(axis), float(pupil.prism_coeff), float(pupil.lens_coeff),
                                 float(pupil.sum_amplitude), ctypes.byref(h)))
        self.handle = h
        self._prec = None
        self._spots_key = None
        self.batch = 0
        self.n = 0
        self._finalizer = weakref.finalize(self, lib.hs_plan_destroy, h)

    # ---- spot batches --------------------------------------------------
    def set_spots(self, spot_sets) -> None:
        """Upload ``spot_sets`` (a SpotSet or a sequence of equal-size sets)."""
        sets = list(spot_sets) if isinstance(spot_sets, (list, tuple)) else [spot_sets]
        key = tuple(id(s) for s in sets)
        if key == self._spots_key and all(s is not None for s in sets):
            return
        n = sets[0].count
        if any(s.count != n for s in sets):
            raise InvalidParameterError("all patterns of a batch need the same spot count")
        x = f64(np.stack([s.x for s in sets]))
        y = f64(np.stack([s.y for s in sets]))
        z = f64(np.stack([s.z for s in sets]))
        a = f64(np.stack([s.amplitude for s in sets]))
        self.set_spot_arrays(x, y, z, a)
        self._spots_key = key
        self._spot_refs = sets  # keep ids stable while cached

    def set_spot_arrays(self, x, y, z, a0) -> None:
        x, y, z, a0 = (f64(np.atleast_2d(v)) for v in (x, y, z, a0))
        b, n = x.shape
        check(load().hs_set_spots(self.handle, b, n, ptr(x), ptr(y), ptr(z), ptr(a0)))
        self.batch, self.n = b, n
        self._spots_key = None

    def _sync_precision(self) -> None:
        if self._prec != _precision and hasattr(load(), "hs_set_precision"):
            check(load().hs_set_precision(self.handle, PRECISIONS[_precision]))
            self._prec = _precision

    def last_precision(self) -> str:
        """Arithmetic of the plan's last solve: "fp32" or "fp64"."""
        mode, last = ctypes.c_int(), ctypes.c_int()
        check(load().hs_get_precision(self.handle, ctypes.byref(mode), ctypes.byref(last)))
        return "fp64" if last.value == PREC_FP64 else "fp32"

    def get_tables(self):
        """fp64 phasor tables of pattern 0: (gx_re, gx_im, gy_re, gy_im), [side][n]."""
        out = [np.empty((self.side, self.n)) for _ in range(4)]
        check(load().hs_get_tables(self.handle, *[ptr(o) for o in out]))
        return tuple(out)

    def set_tables(self, gx_re, gx_im, gy_re, gy_im) -> None:
        """Install caller tables for pattern 0 (kept until the spots change)."""
        arrs = [f64(a) for a in (gx_re, gx_im, gy_re, gy_im)]
        if any(a.shape != (self.side, self.n) for a in arrs):
            raise InvalidParameterError(
                f"tables must be ({self.side}, {self.n}) arrays, got {[a.shape for a in arrs]}")
        check(load().hs_set_tables(self.handle, self.n, *[ptr(a) for a in arrs]))
        self._spots_key = None   # the next set_spots re-uploads (and rebuilds the tables)

    # ---- kernels --------------------------------------------------------
    def superpose(self, amplitude, theta, start: int, stop: int) -> np.ndarray:
        self._sync_precision()
        out = np.empty(stop - start, dtype=np.float64)
        a, t = f64(amplitude), f64(theta)
        check(load().hs_superpose(self.handle, ptr(a), ptr(t), start, stop, ptr(out)))
        return out

    def forward(self, phase, start: int, stop: int) -> np.ndarray:
        self._sync_precision()
        ph = f64(phase)
        out = np.empty(2 * self.n, dtype=np.float64)
        check(load().hs_forward(self.handle, ptr(ph), start, stop, ptr(out)))
        return out[0::2] + 1j * out[1::2]

    def quality(self, phase):
        self._sync_precision()
        ph = f64(phase)
        e, u = ctypes.c_double(), ctypes.c_double()
        inten = np.empty(self.n)
        rel = np.empty(self.n)
        fields = np.empty(2 * self.n)
        check(load().hs_quality(self.handle, ptr(ph), ctypes.byref(e), ctypes.byref(u),
                                ptr(inten), ptr(rel), ptr(fields)))
        return e.value, u.value, inten, rel, fields[0::2] + 1j * fields[1::2]

    # ---- solver ---------------------------------------------------------
    def solve(self, algorithm: int, iterations: int, subset: int, theta0,
              want_fields: bool = True, sync: bool = True, raster: bool = False) -> None:
        self._sync_precision()
        th = f64(theta0)
        fn = load().hs_solve if sync else load().hs_solve_async
        flags = (WANT_FIELDS if want_fields else 0) | (WANT_RASTER if raster else 0) | WANT_PHASE32
        check(fn(self.handle, algorithm, iterations, subset, ptr(th), flags))

    def rasters(self, first: int = 0, count: int | None = None) -> np.ndarray:
        count = self.batch - first if count is None else count
        out = np.empty((count, self.side, self.side), dtype=np.uint8)
        check(load().hs_get_raster(self.handle, first, count, ptr(out)))
        return out

    def raster(self, phase, lut=None) -> np.ndarray:
        out = np.empty((self.side, self.side), dtype=np.uint8)
        tab = None if lut is None else f64(lut)
        check(load().hs_raster(self.handle, ptr(f64(phase)), ptr(tab), ptr(out)))
        return out

    def sync(self) -> None:
        check(load().hs_sync(self.handle))

    def status(self):
        st = np.zeros(self.batch, dtype=np.int32)
        dg = np.zeros(self.batch, dtype=np.int32)
        check(load().hs_get_status(self.handle, ptr(st), ptr(dg)))
        return st, dg

    def trace(self, iterations: int):
        w = np.empty((self.batch, iterations, self.n))
        m = np.empty((self.batch, iterations, self.n))
        if iterations:
            check(load().hs_get_trace(self.handle, ptr(w), ptr(m)))
        return w, m

    def phases(self, first: int = 0, count: int | None = None) -> np.ndarray:
        count = self.batch - first if count is None else count
        out = np.empty((count, self.m), dtype=np.float64)
        check(load().hs_get_phase(self.handle, first, count, ptr(out)))
        return out

    def quality_batch(self):
        b, n = self.batch, self.n
        e, u = np.empty(b), np.empty(b)
        inten, rel, fields = np.empty((b, n)), np.empty((b, n)), np.empty((b, 2 * n))
        check(load().hs_get_quality(self.handle, ptr(e), ptr(u), ptr(inten), ptr(rel),
                                    ptr(fields)))
        return e, u, inten, rel, fields[:, 0::2] + 1j * fields[:, 1::2]

    def probe(self, phase, points, batch: int = 1024) -> np.ndarray:
        self._sync_precision()
        pts = f64(np.atleast_2d(points))
        out = np.empty(pts.shape[0], dtype=np.float64)
        try:
            check(load().hs_probe(self.handle, ptr(f64(phase)), pts.shape[0], ptr(pts),
                                  int(batch), ptr(out)))
        finally:
            self._spots_key = None  # hs_probe replaced the device spot set
        return out

    # ---- row-sharded solve (distributed.solve_sharded) -----------------
    def shard_begin(self, algorithm: int, iterations: int, subset: int, theta0, rank: int,
                    world: int) -> None:
        self._sync_precision()
        check(load().hs_shard_begin(self.handle, algorithm, iterations, subset,
                                    ptr(f64(theta0)), rank, world))

    def shard_pass(self, j: int):
        """Run pass j on this rank's chunk range -> (group partials
        complex128 [B][g_hi - g_lo][np], g_lo, g_hi, total groups)."""
        lib = load()
        np_ = lib.hs_padded_spots(self.handle)
        lo, hi, ng = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib.hs_shard_groups(self.handle, j, ctypes.byref(lo), ctypes.byref(hi),
                                  ctypes.byref(ng)))
        local = np.zeros((self.batch, hi.value - lo.value, np_), dtype=np.complex128)
        check(lib.hs_shard_pass(self.handle, j, ptr(local), ctypes.byref(lo), ctypes.byref(hi),
                                ctypes.byref(ng)))
        return local, lo.value, hi.value, ng.value

    def shard_update(self, j: int, all_groups: np.ndarray) -> None:
        g = np.ascontiguousarray(all_groups, dtype=np.complex128)
        check(load().hs_shard_update(self.handle, j, ptr(g), g.shape[1]))

    # ---- the same over peer memory (csrc/hs_xchg.cuh) -------------------
    def p2p_setup(self) -> bytes:
        """Allocate this rank's exchange buffer; returns its CUDA IPC handle."""
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        check(load().hs_shard_p2p_setup(self.handle, buf))
        return buf.raw

    def p2p_open(self, handles) -> None:
        """Map the world's exchange buffers (handles in rank order)."""
        blob = b"".join(bytes(h) for h in handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        check(load().hs_shard_p2p_open(self.handle, buf))

    def p2p_pass(self, j: int) -> None:
        """Enqueue pass j (chunk range + peer publish + gather/update); async."""
        check(load().hs_shard_p2p_pass(self.handle, j))

    def p2p_solve(self) -> None:
        """Every pass of the begun sharded solve as one captured CUDA graph."""
        check(load().hs_shard_p2p_solve(self.handle))

    def p2p_close(self) -> None:
        check(load().hs_shard_p2p_close(self.handle))

    def padded_spots(self) -> int:
        return int(load().hs_padded_spots(self.handle))

    def stream(self) -> int:
        return int(load().hs_plan_stream(self.handle) or 0)

    def last_launch_count(self) -> int:
        v = ctypes.c_int64()
        check(load().hs_last_launch_count(self.handle, ctypes.byref(v)))
        return v.value

    def time_kernel(self, which: int, subset: int = 0, reps: int = 20):
        ms, pairs = ctypes.c_double(), ctypes.c_double()
        check(load().hs_time_kernel(self.handle, which, subset, reps, ctypes.byref(ms),
                                    ctypes.byref(pairs)))
        return ms.value, pairs.value


def fma_peak_tflops(device: int | None = None) -> float:
    """Measured FP32 FFMA peak of the device (TFLOP/s)."""
    v = ctypes.c_double()
    check(load().hs_fma_peak(get_device() if device is None else int(device), ctypes.byref(v)))
    return v.value


_plans: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def plan_for(pupil, device: int | None = None) -> Plan:
    """The cached device plan of ``pupil`` (geometry uploaded once)."""
    dev = get_device() if device is None else int(device)
    per = _plans.get(pupil)
    if per is None:
        per = {}
        _plans[pupil] = per
    plan = per.get(dev)
    if plan is None:
        plan = Plan(pupil, dev)
        per[dev] = plan
    return plan
