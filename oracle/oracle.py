"""CPU oracle for the CS-WGS hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module, and only as the checker / the timed CPU
baseline.  The product package never imports it.

It restates the reference ``holospots`` algorithm (files under
``/root/reference/pkg/src/holospots``):

* kernels   -> ``holo_oracle.c`` (fp64 C, OpenMP), loaded with ctypes;
* the fixed-shape reduction tree, the weight update, the iteration
  schedule and the metrics -> numpy code below, each function citing the
  reference lines it follows.

Pinning: ``tests/test_oracle_golden.py`` checks every function here
against vectors produced by the reference itself
(``tests/golden/make_golden.py``), bitwise where the reference is
deterministic and the operation order is restated exactly.

Inputs are duck-typed: any pupil object exposing ``rows``, ``cols``,
``amplitude``, ``axis_coords()``, ``prism_coeff``, ``lens_coeff``,
``active_count`` and ``sum_amplitude`` works (the reference ``Pupil`` and the
product ``Pupil`` both do); spots are passed as plain arrays.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libholo_oracle.so")
_lib = None
_lock = threading.Lock()

DEFAULT_CHUNK = 1024          # kernels.py:36
DEGENERACY_FLOOR = 1e-6       # solvers.py:35
TWO_PI = 2.0 * math.pi        # optics.py:28


def build(force: bool = False) -> str:
    """Compile holo_oracle.c into oracle/_build/libholo_oracle.so."""
    src = os.path.join(_HERE, "holo_oracle.c")
    if not force and os.path.exists(_LIB_PATH) and \
            os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src):
        return _LIB_PATH
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"]
    subprocess.run(cmd, check=True)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                build()
            lib = ctypes.CDLL(_LIB_PATH)
            P = ctypes.c_void_p
            I64 = ctypes.c_int64
            D = ctypes.c_double
            lib.or_build_tables.argtypes = [I64, P, D, D, I64, P, P, P, P, P, P, P]
            lib.or_superpose_mag.argtypes = [P, P, I64, I64, I64, P, P, P, P, P, P,
                                             ctypes.c_int]
            lib.or_forward.argtypes = [P, P, P, P, I64, I64, I64, I64, P, P, P, P,
                                       I64, P, P, ctypes.c_int]
            lib.or_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return int(_load().or_max_threads())


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# --------------------------------------------------------------------------
# optics.py restatements
# --------------------------------------------------------------------------

def wrap_phase(phase):
    """[-pi, pi) wrap via exact fmod (optics.py:31-45)."""
    w = np.fmod(phase, TWO_PI)
    w = np.where(w >= math.pi, w - TWO_PI, w)
    w = np.where(w < -math.pi, w + TWO_PI, w)
    return w


# --------------------------------------------------------------------------
# kernels.py restatements
# --------------------------------------------------------------------------

class Tables:
    """Separable column/row phasor tables (kernels.py:61-76)."""

    def __init__(self, gx_re, gx_im, gy_re, gy_im):
        self.gx_re, self.gx_im, self.gy_re, self.gy_im = gx_re, gx_im, gy_re, gy_im
        self.count = gx_re.shape[1]


def tables(pupil, x, y, z) -> Tables:
    """kernels.py:177-183 -> _build_tables (kernels.py:78-96)."""
    lib = _load()
    axis = _c64(pupil.axis_coords())
    x, y, z = _c64(x), _c64(y), _c64(z)
    side, n = axis.shape[0], x.shape[0]
    out = [np.empty((side, n)) for _ in range(4)]
    lib.or_build_tables(side, _p(axis), float(pupil.prism_coeff),
                        float(pupil.lens_coeff), n, _p(x), _p(y), _p(z),
                        *[_p(o) for o in out])
    return Tables(*out)


def superpose(pupil, tab: Tables, amplitude, theta, start=0, stop=None,
              threads=None, want_mag=False):
    """kernels.py:186-214: coef=a*e^{i wrap(theta)}, U=gx*coef, per-pixel atan2."""
    lib = _load()
    m = pupil.active_count
    stop = m if stop is None else stop
    theta = wrap_phase(_c64(theta))
    amplitude = _c64(amplitude)
    cr = amplitude * np.cos(theta)
    ci = amplitude * np.sin(theta)
    u_re = np.ascontiguousarray(tab.gx_re * cr - tab.gx_im * ci)
    u_im = np.ascontiguousarray(tab.gx_re * ci + tab.gx_im * cr)
    out = np.empty(stop - start)
    mag = np.empty(stop - start) if want_mag else None
    if stop > start:
        cols, rows = _i64(pupil.cols), _i64(pupil.rows)
        lib.or_superpose_mag(_p(cols), _p(rows), start, stop, tab.count,
                             _p(u_re), _p(u_im), _p(tab.gy_re), _p(tab.gy_im),
                             _p(out), _p(mag) if want_mag else None,
                             threads or max_threads())
    return (out, mag) if want_mag else out


def reduce_columns(values: np.ndarray, chunk: int) -> np.ndarray:
    """Fixed-shape tree over axis 0 (kernels.py:249-263): groups of ``chunk``
    rows are summed left to right, then the group sums recurse."""
    level = values
    while level.shape[0] > 1:
        groups = []
        for lo in range(0, level.shape[0], chunk):
            block = level[lo:lo + chunk]
            acc = block[0].copy()
            for row in block[1:]:
                acc += row
            groups.append(acc)
        level = np.stack(groups)
    return level[0]


def forward(pupil, tab: Tables, phase, start=0, stop=None, chunk=DEFAULT_CHUNK,
            threads=None) -> np.ndarray:
    """kernels.py:217-246: chunked per-spot fields + fixed tree."""
    lib = _load()
    m = pupil.active_count
    stop = m if stop is None else stop
    n = tab.count
    if stop == start:
        return np.zeros(n, dtype=np.complex128)
    nchunks = -(-(stop - start) // chunk)
    part_re = np.empty((nchunks, n))
    part_im = np.empty((nchunks, n))
    cols, rows = _i64(pupil.cols), _i64(pupil.rows)
    amp, ph = _c64(pupil.amplitude), _c64(phase)
    lib.or_forward(_p(cols), _p(rows), _p(amp), _p(ph), start, stop, chunk, n,
                   _p(tab.gx_re), _p(tab.gx_im), _p(tab.gy_re), _p(tab.gy_im),
                   nchunks, _p(part_re), _p(part_im), threads or max_threads())
    return reduce_columns(part_re + 1j * part_im, chunk)


def tree_reduce(values, chunk=DEFAULT_CHUNK) -> complex:
    """reduce_complex (kernels.py:266-283)."""
    vals = np.ascontiguousarray(values, dtype=np.complex128)
    if vals.shape[0] == 0:
        return 0j
    return complex(reduce_columns(vals[:, None], chunk)[0])


# --------------------------------------------------------------------------
# solvers.py restatements
# --------------------------------------------------------------------------

class OracleDegenerate(RuntimeError):
    pass


def field_phases(fields):
    """solvers.py:96-101."""
    ph = np.arctan2(fields.imag, fields.real)
    ph = np.where(ph == math.pi, -math.pi, ph)
    zero = (fields.real == 0.0) & (fields.imag == 0.0)
    return np.where(zero, 0.0, ph)


def rebalance(weights, mags):
    """solvers.py:104-129 -> (new weights, magnitudes used, degenerate)."""
    mags = np.asarray(mags, dtype=np.float64)
    degenerate = bool(np.any(mags == 0.0))
    if degenerate:
        pos = mags[mags > 0.0]
        if pos.size == 0:
            raise OracleDegenerate("all spot fields vanished")
        mags = np.where(mags == 0.0, pos.min() * DEGENERACY_FLOOR, mags)
    with np.errstate(over="ignore"):
        w = weights * (np.mean(mags) / mags)
    if not np.all(np.isfinite(w)):
        raise OracleDegenerate("weights diverged")
    return w, mags, degenerate


def schedule(m, subset, iterations):
    """Read/write ranges of _iterate (solvers.py:210-230)."""
    cs = max(0, iterations - 2) if subset < m else 0
    half = max(1, subset // 2)
    read = (0, subset) if cs else (0, m)
    steps = []
    for j in range(1, iterations + 1):
        if j <= cs:
            off = ((j - 1) * half) % (m - subset + 1)
            write = (off, off + subset)
        else:
            write = (0, m)
        steps.append((read, write))
        read = write
    return steps


def solve(pupil, x, y, z, a0, algorithm, iterations=1, compression=1.0, seed=0,
          chunk=DEFAULT_CHUNK, threads=None):
    """rs / wgs / cswgs (solvers.py:166-269).  Returns a dict with the final
    phase (storage order), per-iteration weights/magnitudes/subset sizes,
    the op count, the degeneracy flag and the final coefficients."""
    m = pupil.active_count
    a0 = _c64(a0)
    n = a0.shape[0]
    tab = tables(pupil, x, y, z)
    rng = np.random.default_rng(seed)                   # solvers.py:169
    thetas = rng.random(n) * (2.0 * math.pi)            # solvers.py:170
    weights = np.ones(n)
    amps = weights * a0
    phase = superpose(pupil, tab, amps, thetas, threads=threads)
    if algorithm == "rs":
        return dict(phase=phase, weights=np.zeros((0, n)), mags=np.zeros((0, n)),
                    sizes=[], ops=m * n, degenerate=False, amps=amps, thetas=thetas,
                    tables=tab)
    if algorithm == "wgs":
        subset = m
    else:
        subset = math.ceil(compression * m)             # optics.py:297-302
    ops, degenerate = 0, False
    ws, ms, sizes = [], [], []
    for read, write in schedule(m, subset, iterations):
        fields = forward(pupil, tab, phase, read[0], read[1], chunk, threads)
        mags = np.hypot(fields.real, fields.imag)        # solvers.py:148
        weights, mags, deg = rebalance(weights, mags)
        amps = weights * a0
        thetas = field_phases(fields)
        frag = superpose(pupil, tab, amps, thetas, write[0], write[1], threads)
        phase = np.array(phase)
        phase[write[0]:write[1]] = frag
        degenerate = degenerate or deg
        size = write[1] - write[0]
        ops += size * n
        ws.append(weights)
        ms.append(mags)
        sizes.append(size)
    return dict(phase=phase, weights=np.array(ws), mags=np.array(ms), sizes=sizes,
                ops=ops, degenerate=degenerate, amps=amps, thetas=thetas, tables=tab)


# --------------------------------------------------------------------------
# metrics.py restatements
# --------------------------------------------------------------------------

def quality(pupil, tab: Tables, phase, a0, chunk=DEFAULT_CHUNK, threads=None):
    """quality_report (metrics.py:33-79) -> (e, u, intensities, relative)."""
    fields = forward(pupil, tab, phase, chunk=chunk, threads=threads)
    norm = pupil.sum_amplitude * pupil.sum_amplitude
    inten = (fields.real * fields.real + fields.imag * fields.imag) / norm
    rel = inten / (_c64(a0) * _c64(a0))
    e = float(np.sum(inten))
    hi, lo = float(np.max(rel)), float(np.min(rel))
    u = 1.0 - (hi - lo) / (hi + lo)
    return e, u, inten, rel
