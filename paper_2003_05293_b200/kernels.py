"""Hologram kernels: drop-in for holospots/kernels.py, executed on the B200.

``superpose`` and ``forward_project`` keep the reference signatures,
validation order and exceptions (kernels.py:186-246) and run the sm_100a
pass kernel through the C ABI.  ``chunk`` and ``workers`` are accepted and
validated for signature compatibility; like the reference's ``workers``
they never change results (the device reduction tree is fixed by the list
length alone).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import GeometryMismatchError, InvalidParameterError
from .optics import Hologram, Pupil, SpotSet

DEFAULT_CHUNK = 1024


@dataclass(frozen=True)
class SpotCoefficients:
    """Superposition amplitudes (>= 0) and phase offsets (kernels.py:39-58)."""

    amplitude: np.ndarray
    theta: np.ndarray

    def __post_init__(self):
        amp = np.ascontiguousarray(self.amplitude, dtype=np.float64)
        th = np.ascontiguousarray(self.theta, dtype=np.float64)
        if amp.ndim != 1 or amp.shape != th.shape:
            raise InvalidParameterError("amplitude and theta must be equal-length 1-D arrays")
        if np.any(amp < 0):
            raise InvalidParameterError("spot amplitudes must be >= 0")
        object.__setattr__(self, "amplitude", amp)
        object.__setattr__(self, "theta", th)

    @property
    def count(self) -> int:
        return int(self.amplitude.shape[0])


class SpotTables:
    """Per-spot column/row phasor tables (kernels.py:61-76).

    ``gx[j, n] = exp(i (c1 x_n axis[j] + c2 z_n axis[j]^2))``, ``gy`` likewise
    with ``y_n``; fp64 [side, n] arrays ``gx_re, gx_im, gy_re, gy_im`` and
    ``count``, as the reference.  :func:`spot_tables` builds them on the device
    (the solver's own table kernel, fp64) and copies them to the host on first
    access; constructing one from arrays (``SpotTables(gx_re, gx_im, gy_re,
    gy_im, count)``) gives caller tables, which ``tables=`` then uploads and
    the passes use instead of tables derived from the spot positions.
    """

    __slots__ = ("count", "_arrays", "_source")

    def __init__(self, gx_re=None, gx_im=None, gy_re=None, gy_im=None, count=None, *,
                 _source=None):
        object.__setattr__(self, "_source", _source)
        if _source is not None:
            object.__setattr__(self, "_arrays", None)
            object.__setattr__(self, "count", int(_source[1].count))
            return
        arrs = []
        for a in (gx_re, gx_im, gy_re, gy_im):
            v = np.array(a, dtype=np.float64)
            v.setflags(write=False)
            arrs.append(v)
        if arrs[0].ndim != 2 or any(v.shape != arrs[0].shape for v in arrs):
            raise InvalidParameterError("tables must be four equal-shape 2-D arrays")
        object.__setattr__(self, "_arrays", tuple(arrs))
        object.__setattr__(self, "count", int(arrs[0].shape[1] if count is None else count))

    def __setattr__(self, name, value):
        raise AttributeError("SpotTables is immutable")

    def _get(self):
        if self._arrays is None:
            pupil, spots = self._source
            plan = _lib.plan_for(pupil)
            plan.set_spots(spots)
            arrs = plan.get_tables()
            for v in arrs:
                v.setflags(write=False)
            object.__setattr__(self, "_arrays", arrs)
        return self._arrays

    @property
    def gx_re(self) -> np.ndarray:
        return self._get()[0]

    @property
    def gx_im(self) -> np.ndarray:
        return self._get()[1]

    @property
    def gy_re(self) -> np.ndarray:
        return self._get()[2]

    @property
    def gy_im(self) -> np.ndarray:
        return self._get()[3]


def _use_tables(plan, pupil: Pupil, spots: SpotSet, tables) -> None:
    """Bind the spot set (and caller tables, if any) to the device plan."""
    plan.set_spots(spots)
    if tables is None:
        return
    if tables._source is not None and tables._source[0] is pupil and tables._source[1] is spots:
        return   # device-built for exactly these spots: the plan rebuilds the same tables
    if tables.count != spots.count:
        raise InvalidParameterError(f"tables carry {tables.count} spots, spot set {spots.count}")
    plan.set_tables(tables.gx_re, tables.gx_im, tables.gy_re, tables.gy_im)


def effective_workers(workers: int) -> int:
    """Validated worker count (kernels.py:147-151); has no effect on the GPU."""
    if workers < 1:
        raise InvalidParameterError("workers must be >= 1")
    return int(workers)


def _check_range(pixel_range, m: int) -> tuple[int, int]:
    if pixel_range is None:
        return 0, m
    start, stop = int(pixel_range[0]), int(pixel_range[1])
    if not 0 <= start <= stop <= m:
        raise InvalidParameterError(f"pixel range {pixel_range} outside 0..{m}")
    return start, stop


def spot_tables(pupil: Pupil, spots: SpotSet) -> SpotTables:
    """Phasor tables of (pupil, spots) (kernels.py:177-183), built on the device."""
    return SpotTables(_source=(pupil, spots))


def superpose(pupil: Pupil, spots: SpotSet, coeffs: SpotCoefficients, pixel_range=None,
              workers: int = 1, tables: SpotTables | None = None) -> np.ndarray:
    """Backward pass over a storage-order range (kernels.py:186-214)."""
    if coeffs.count != spots.count:
        raise InvalidParameterError(
            f"coefficient length {coeffs.count} != spot count {spots.count}")
    start, stop = _check_range(pixel_range, pupil.active_count)
    effective_workers(workers)
    if stop == start:
        return np.empty(0, dtype=np.float64)
    plan = _lib.plan_for(pupil)
    _use_tables(plan, pupil, spots, tables)
    return plan.superpose(coeffs.amplitude, coeffs.theta, start, stop)


def forward_project(pupil: Pupil, hologram: Hologram, spots: SpotSet, pixel_range=None,
                    chunk: int = DEFAULT_CHUNK, workers: int = 1,
                    tables: SpotTables | None = None) -> np.ndarray:
    """Forward pass: per-spot complex fields over a range (kernels.py:217-246)."""
    if chunk < 1:
        raise InvalidParameterError("chunk must be >= 1")
    if hologram.pupil is not pupil and \
            hologram.pupil.geometry_signature() != pupil.geometry_signature():
        raise GeometryMismatchError("hologram was computed for a different pupil")
    start, stop = _check_range(pixel_range, pupil.active_count)
    effective_workers(workers)
    if stop == start:
        return np.zeros(spots.count, dtype=np.complex128)
    plan = _lib.plan_for(pupil)
    _use_tables(plan, pupil, spots, tables)
    return plan.forward(hologram.phase, start, stop)


def reduce_complex(values, chunk: int = DEFAULT_CHUNK) -> complex:
    """Deterministic fixed-shape tree sum (kernels.py:266-283).

    Host utility kept for API parity: consecutive groups of ``chunk`` values
    are summed left to right and the group sums recurse.  The device kernels
    use their own fixed-shape trees.
    """
    if chunk < 1:
        raise InvalidParameterError("chunk must be >= 1")
    vals = np.ascontiguousarray(values, dtype=np.complex128)
    if vals.ndim != 1:
        raise InvalidParameterError("reduce_complex expects a 1-D sequence")
    if vals.shape[0] == 0:
        return 0j
    level = vals
    while level.shape[0] > 1:
        # acc[g] = ((x[g*c] + x[g*c+1]) + x[g*c+2]) + ...: position j of every
        # group is added in one vectorised step; only the last group is short.
        acc = level[0::chunk].copy()
        for j in range(1, min(chunk, level.shape[0])):
            col = level[j::chunk]
            acc[:col.shape[0]] += col
        level = acc
    return complex(level[0])


def warm_up() -> None:
    """Load the CUDA library and run one tiny pass (no JIT involved)."""
    from .optics import build_pupil

    pupil = build_pupil(4, illumination="uniform", seed=0)
    spots = SpotSet.from_points([[1e-6, -1e-6, 0.0]])
    frag = superpose(pupil, spots, SpotCoefficients(np.ones(1), np.zeros(1)))
    forward_project(pupil, Hologram(frag, pupil), spots)
