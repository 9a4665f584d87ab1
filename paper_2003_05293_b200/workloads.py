"""Synthetic spot patterns for the benchmark configurations.

``grid_spots`` restates the unrotated planar grids of holospots/scenarios.py
(grid_scenario 56-75, named_scenario 145-156): ``grid100`` (10x10) and
``grid36`` (6x6) at 10 um spacing, z = 0, unit amplitudes.  ``random_foci``
draws x, y ~ U(-xy, xy) then z ~ U(-z, z) from ``default_rng(seed)``.
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidParameterError
from .optics import SpotSet

_GRIDS = {"grid100": (10, 10), "grid36": (6, 6)}


def grid_spots(rows: int, cols: int, spacing: float = 10e-6) -> SpotSet:
    if rows < 1 or cols < 1:
        raise InvalidParameterError("rows and cols must be >= 1")
    if spacing <= 0:
        raise InvalidParameterError("spacing must be > 0")
    jj, ii = np.meshgrid(np.arange(cols), np.arange(rows))
    x = (jj.ravel() - (cols - 1) / 2.0) * spacing
    y = (ii.ravel() - (rows - 1) / 2.0) * spacing
    return SpotSet.from_points(np.stack([x, y, np.zeros_like(x)], axis=1))


def named_spots(name: str) -> SpotSet:
    if name not in _GRIDS:
        raise InvalidParameterError(f"unknown scenario {name!r}")
    return grid_spots(*_GRIDS[name])


def random_foci(n: int, seed: int, xy: float = 100e-6, z: float = 50e-6) -> SpotSet:
    rng = np.random.default_rng(seed)
    x = rng.uniform(-xy, xy, n)
    y = rng.uniform(-xy, xy, n)
    zz = rng.uniform(-z, z, n)
    return SpotSet(x=x, y=y, z=zz, amplitude=np.ones(n))
