"""Video-rate hologram sequences.

A sequence is an ordered list of spot frames with equal spot counts -- the
reference's ``rotation_sweep`` (scenarios.py:126-142) is the canonical
source.  Two modes:

* ``warm_start=False``: frames are independent reference solves (solver
  seed ``seeds[k]``); the whole sequence is ONE batched device solve, so
  its throughput is the batched rate of the benchmark.
* ``warm_start=True`` (an extension, not in the reference): frame k+1
  starts from theta0 = arg of frame k's final spot fields instead of a
  random phase.  Neighbouring frames differ by a small rotation, so the
  previous solution is a near-optimal start; frames run one after another
  on the device (each is one graph replay), frame 0 from its seed.

Both return the same ``(Hologram, SolverTrace)`` pairs as ``solve``.
"""

from __future__ import annotations

import time

import numpy as np

from . import solvers
from .errors import InvalidParameterError
from .optics import CompressionPlan, Pupil
from .scenarios import Scenario, rotation_sweep


def _subset(pupil: Pupil, config: solvers.SolverConfig) -> int:
    if config.algorithm == "cswgs":
        return CompressionPlan.for_pupil(pupil, config.compression).subset_size
    return pupil.active_count


def solve_sequence(pupil: Pupil, frames, config: solvers.SolverConfig, seeds=None,
                   warm_start: bool = False):
    """Solve ``frames`` in order; see the module docstring for the modes."""
    frames = list(frames)
    if not frames:
        return []
    n = frames[0].count
    if any(f.count != n for f in frames):
        raise InvalidParameterError("sequence frames need equal spot counts")
    seeds = [config.seed + k for k in range(len(frames))] if seeds is None else list(seeds)
    if len(seeds) != len(frames):
        raise InvalidParameterError("one seed per frame")
    if not warm_start:
        return solvers.solve_batch(pupil, frames, config, seeds=seeds)
    subset = _subset(pupil, config)
    out = []
    theta = None
    for frame, seed in zip(frames, seeds):
        t0 = time.perf_counter()
        res = solvers._run_batch(config.algorithm, pupil, [frame], config.iterations, subset,
                                 [seed], theta0=None if theta is None else theta[None, :])
        out.append(solvers._assemble(config.algorithm, pupil, frame, res, 0, config.iterations,
                                     subset, t0))
        theta = solvers._field_phases(res.fields[0])
    return out


def rotation_sequence(pupil: Pupil, scenario: Scenario, frames: int,
                      config: solvers.SolverConfig, step_angle: float | None = None,
                      warm_start: bool = False):
    """``solve_sequence`` over ``rotation_sweep(scenario, frames, step_angle)``."""
    return solve_sequence(pupil, rotation_sweep(scenario, frames, step_angle), config,
                          warm_start=warm_start)


def sequence_quality(results) -> np.ndarray:
    """(frames, 2) array of the fused e, u per frame."""
    return np.array([[t.quality.efficiency, t.quality.uniformity] for _, t in results])
