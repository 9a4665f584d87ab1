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


@dataclass(frozen=True)
class SpotTables:
    """Handle for one (pupil, spots) pairing (kernels.py:61-76).

    The phasor tables themselves live on the device, rebuilt by the table
    kernel whenever the spot batch changes; this handle only pins the pair
    so callers can pass ``tables=`` exactly as with the reference.
    """

    pupil: Pupil
    spots: SpotSet
    count: int


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
    plan = _lib.plan_for(pupil)
    plan.set_spots(spots)
    return SpotTables(pupil, spots, spots.count)


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
    plan.set_spots(spots)
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
    plan.set_spots(spots)
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
