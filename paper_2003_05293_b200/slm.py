"""Phase -> gray lookup and SLM rasters.

``PhaseLut`` restates the reference's 256-level lookup (fileio.py:159-228)
for API parity (host numpy, N-free).  The SLM raster itself -- storage-order
phase scattered onto the (side, side) grid through the LUT, 0 outside the
aperture, exactly the raster ``write_hologram_pgm`` stores (fileio.py:233-241)
-- is built on the device:

* ``slm_raster(pupil, hologram, lut)``: standalone kernel (hs_raster),
  default linear table or a custom table by first-minimum circular distance;
* ``solve_rasters(...)``: batched solve whose final pass writes the raster
  while it writes the phase (linear LUT fused into the epilogue), i.e. the
  SLM-ready output of the paper's texture path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidParameterError
from .optics import Hologram, Pupil, wrap_phase

LUT_LEVELS = 256


def _linear_table() -> np.ndarray:
    g = np.arange(LUT_LEVELS, dtype=np.float64)
    return -math.pi + 2.0 * math.pi * g / LUT_LEVELS


@dataclass(frozen=True)
class PhaseLut:
    """256-level phase/gray lookup (fileio.py:159-213)."""

    table: np.ndarray

    def __post_init__(self):
        tab = np.ascontiguousarray(self.table, dtype=np.float64)
        if tab.shape != (LUT_LEVELS,):
            raise InvalidParameterError(f"LUT must have {LUT_LEVELS} entries")
        tab = wrap_phase(tab)
        tab.setflags(write=False)
        object.__setattr__(self, "table", tab)
        object.__setattr__(self, "_linear", bool(np.array_equal(tab, _linear_table())))

    @classmethod
    def default(cls) -> "PhaseLut":
        return cls(table=_linear_table())

    @classmethod
    def from_file(cls, path) -> "PhaseLut":
        entries = []
        with open(path, "r", encoding="utf-8") as fh:
            for lineno, raw in enumerate(fh, start=1):
                line = raw.strip()
                if not line or line.startswith("#"):
                    continue
                try:
                    entries.append(float(line))
                except ValueError as exc:
                    raise InvalidParameterError(f"{path}:{lineno}: {exc}") from exc
        if len(entries) != LUT_LEVELS:
            raise InvalidParameterError(f"{path}: expected {LUT_LEVELS} entries, got {len(entries)}")
        return cls(table=np.array(entries))

    @property
    def linear(self) -> bool:
        return self._linear

    def phase(self, gray) -> np.ndarray:
        g = np.asarray(gray)
        if np.any(g < 0) or np.any(g > 255):
            raise InvalidParameterError("gray levels must be 0..255")
        return self.table[g]

    def gray(self, phase):
        """Nearest gray level (circular distance); host utility."""
        p = wrap_phase(np.asarray(phase, dtype=np.float64))
        if self._linear:
            g = np.rint((p + math.pi) * (LUT_LEVELS / (2.0 * math.pi)))
            return (np.asarray(g).astype(np.int64) % LUT_LEVELS).astype(np.uint8)
        flat = np.atleast_1d(p).ravel()
        out = np.empty(flat.shape[0], dtype=np.uint8)
        for lo in range(0, flat.shape[0], 8192):
            d = np.abs(wrap_phase(flat[lo:lo + 8192, None] - self.table[None, :]))
            out[lo:lo + 8192] = np.argmin(d, axis=1).astype(np.uint8)
        return out.reshape(np.shape(p)) if np.ndim(p) else out[0]


def slm_raster(pupil: Pupil, hologram: Hologram, lut: PhaseLut | None = None) -> np.ndarray:
    """(side, side) uint8 raster of the hologram through ``lut`` (device)."""
    if hologram.pupil is not pupil and \
            hologram.pupil.geometry_signature() != pupil.geometry_signature():
        from .errors import GeometryMismatchError
        raise GeometryMismatchError("hologram was computed for a different pupil")
    lut = lut or PhaseLut.default()
    return _lib.plan_for(pupil).raster(hologram.phase, None if lut.linear else lut.table)


def solve_rasters(pupil: Pupil, spot_sets, config, seeds=None):
    """Batched solve + fused SLM rasters (default LUT).

    Returns ``(results, rasters)``: ``results`` as :func:`solve_batch`,
    ``rasters`` uint8 [B, side, side] written by the final pass.
    """
    from .solvers import solve_batch
    results = solve_batch(pupil, spot_sets, config, seeds=seeds, raster=True)
    return results, _lib.plan_for(pupil).rasters()
