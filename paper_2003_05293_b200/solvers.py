"""RS / WGS / CS-WGS solvers: drop-in for holospots/solvers.py on the B200.

Every iterative run is ONE CUDA-graph replay on the device (hs_solve):
tables -> seed coefficients -> for each iteration a fused
superpose+forward pass over the window the next iteration reads, and a
single-CTA weight/theta update.  The schedule reproduces
``holospots.solvers._iterate`` exactly (solvers.py:192-235): the sliding
half-step window offsets, read-the-window-you-just-wrote, the last two
iterations at full size, the op count and the per-iteration trace.

Dead work the reference performs but never observes is not repeated: the
seed superposition is only evaluated where iteration 1 reads it, and
compressed-iteration phases are consumed on chip by the next forward pass
instead of being stored, because iteration I-1 rewrites every pixel before
anything else reads them.

Batched entry point :func:`solve_batch` runs many independent patterns
(same pupil and spot count) through one graph replay.
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DegenerateFieldError, InvalidParameterError
from .kernels import DEFAULT_CHUNK, SpotCoefficients, SpotTables, forward_project, superpose
from .optics import CompressionPlan, Hologram, Pupil, SpotSet

ALGORITHMS = ("rs", "wgs", "cswgs")
DEGENERACY_FLOOR = 1e-6
_ALG_CODE = {"rs": _lib.ALG_RS, "wgs": _lib.ALG_WGS, "cswgs": _lib.ALG_CSWGS}


@dataclass(frozen=True)
class SolverConfig:
    """Run parameters (solvers.py:38-58)."""

    algorithm: str
    iterations: int = 30
    compression: float = 1.0
    seed: int = 0
    budget_ops: int | None = None

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise InvalidParameterError(f"unknown algorithm {self.algorithm!r}")
        if self.iterations < 1:
            raise InvalidParameterError("iterations must be >= 1")
        if self.algorithm == "cswgs":
            if self.iterations < 2:
                raise InvalidParameterError(
                    "cswgs needs iterations >= 2 (the two final full passes)")
            if not 0.0 < self.compression <= 1.0:
                raise InvalidParameterError("compression must be in (0, 1]")


@dataclass(frozen=True)
class StepRecord:
    iteration: int
    weights: np.ndarray
    magnitudes: np.ndarray
    subset_size: int
    ops: int
    degenerate: bool


@dataclass(frozen=True)
class SolverTrace:
    algorithm: str
    records: tuple
    operation_count: int
    wall_time_s: float
    degenerate: bool
    hologram: Hologram
    # extension: e/u of the final fused pass (QualityReport), computed on the
    # device with no extra projection; quality_report() re-projects instead
    quality: object = None


@dataclass(frozen=True)
class WgsState:
    weights: np.ndarray
    amplitudes: np.ndarray
    thetas: np.ndarray
    hologram: Hologram
    degenerate: bool = False


# ---------------------------------------------------------------- host utils
def _field_phases(fields: np.ndarray) -> np.ndarray:
    """arg in [-pi, pi), arg(0) = 0 (solvers.py:96-101)."""
    ph = np.arctan2(fields.imag, fields.real)
    ph = np.where(ph == math.pi, -math.pi, ph)
    return np.where((fields.real == 0.0) & (fields.imag == 0.0), 0.0, ph)


def rebalance_weights(weights, magnitudes):
    """Mean-over-own weight update with degeneracy floor (solvers.py:104-129).

    Host utility for API parity; solver runs perform the same update on the
    device (hs_update_kernel)."""
    mags = np.asarray(magnitudes, dtype=np.float64)
    degenerate = bool(np.any(mags == 0.0))
    if degenerate:
        positive = mags[mags > 0.0]
        if positive.size == 0:
            raise DegenerateFieldError("all spot fields vanished; cannot rebalance")
        mags = np.where(mags == 0.0, positive.min() * DEGENERACY_FLOOR, mags)
    with np.errstate(over="ignore"):
        new = np.asarray(weights, dtype=np.float64) * (np.mean(mags) / mags)
    if not np.all(np.isfinite(new)):
        raise DegenerateFieldError("spot weights diverged beyond float range")
    return new, mags, degenerate


def _theta0(seed: int, n: int) -> np.ndarray:
    """Random-phase start (solvers.py:169-170)."""
    return np.random.default_rng(seed).random(n) * (2.0 * math.pi)


def window_sizes(m: int, subset: int, iterations: int) -> list[int]:
    """Write-window sizes of _iterate (solvers.py:210-226)."""
    cs = max(0, iterations - 2) if subset < m else 0
    return [subset if j <= cs else m for j in range(1, iterations + 1)]


# ------------------------------------------------------------------ runs
@dataclass
class BatchResult:
    """Device results of one batched run (host copies)."""

    phases: np.ndarray          # [B, M]
    weights: np.ndarray         # [B, I, N]
    magnitudes: np.ndarray      # [B, I, N]
    status: np.ndarray          # [B]
    first_degenerate: np.ndarray  # [B] 1-based iteration, 0 = never
    efficiency: np.ndarray      # [B]
    uniformity: np.ndarray      # [B]
    intensities: np.ndarray     # [B, N]
    relative: np.ndarray        # [B, N]
    fields: np.ndarray          # [B, N] complex


def _run_batch(algorithm: str, pupil: Pupil, spot_sets, iterations: int, subset: int,
               seeds, fetch_phase: bool = True, raster: bool = False,
               theta0: np.ndarray | None = None) -> BatchResult:
    plan = _lib.plan_for(pupil)
    plan.set_spots(spot_sets)
    n = plan.n
    if theta0 is None:
        theta0 = np.stack([_theta0(int(s), n) for s in seeds])
    else:
        theta0 = np.ascontiguousarray(theta0, dtype=np.float64).reshape(len(spot_sets), n)
    iters = 0 if algorithm == "rs" else iterations
    # the fused e/u projection needs illumination (metrics.py:37-38); without
    # it RS still succeeds and WGS / CS-WGS fail on the all-zero fields with
    # DegenerateFieldError, as in the reference (solvers.py:117-119)
    lit = pupil.sum_amplitude > 0.0
    plan.solve(_ALG_CODE[algorithm], iters, subset, theta0, want_fields=lit, raster=raster)
    status, deg = plan.status()
    w, mg = plan.trace(iters)
    if lit:
        e, u, inten, rel, fields = plan.quality_batch()
    else:
        b = plan.batch
        e, u = np.full(b, np.nan), np.full(b, np.nan)
        inten, rel = np.full((b, n), np.nan), np.full((b, n), np.nan)
        fields = np.full((b, n), np.nan, dtype=np.complex128)
    phases = plan.phases() if fetch_phase else np.empty((plan.batch, 0))
    return BatchResult(phases, w, mg, status, deg, e, u, inten, rel, fields)


def _raise_status(code: int) -> None:
    if code == _lib.HS_EDEGENERATE:
        raise DegenerateFieldError("all spot fields vanished; cannot rebalance")
    if code == _lib.HS_EDIVERGED:
        raise DegenerateFieldError("spot weights diverged beyond float range")
    if code != 0:
        _lib.check(code)


def _assemble(algorithm: str, pupil: Pupil, spots: SpotSet, res: BatchResult, b: int,
              iterations: int, subset: int, t0: float):
    _raise_status(int(res.status[b]))
    m, n = pupil.active_count, spots.count
    holo = Hologram(res.phases[b], pupil)
    from .metrics import QualityReport
    fused = None
    if np.isfinite(res.efficiency[b]):   # no fused estimate for an unlit pupil
        fused = QualityReport(efficiency=float(res.efficiency[b]), uniformity=float(res.uniformity[b]),
                              intensities=res.intensities[b].copy(),
                              target_relative=res.relative[b].copy())
    if algorithm == "rs":
        trace = SolverTrace("rs", (), m * n, time.perf_counter() - t0, False, holo, fused)
        return holo, trace
    records, ops = [], 0
    first_deg = int(res.first_degenerate[b])
    for j, size in enumerate(window_sizes(m, subset, iterations), start=1):
        ops += size * n
        records.append(StepRecord(iteration=j, weights=res.weights[b, j - 1].copy(),
                                  magnitudes=res.magnitudes[b, j - 1].copy(),
                                  subset_size=size, ops=ops,
                                  degenerate=bool(first_deg and j >= first_deg)))
    trace = SolverTrace(algorithm, tuple(records), ops, time.perf_counter() - t0,
                        bool(first_deg), holo, fused)
    return holo, trace


def _single(algorithm, pupil, spots, iterations, subset, seed):
    t0 = time.perf_counter()
    res = _run_batch(algorithm, pupil, [spots], iterations, subset, [seed])
    return _assemble(algorithm, pupil, spots, res, 0, iterations, subset, t0)


def rs(pupil: Pupil, spots: SpotSet, seed: int = 0,
       workers: int = 1) -> tuple[Hologram, SolverTrace]:
    """One-shot random superposition (solvers.py:179-189)."""
    if workers < 1:
        raise InvalidParameterError("workers must be >= 1")
    return _single("rs", pupil, spots, 0, pupil.active_count, seed)


def wgs(pupil: Pupil, spots: SpotSet, iterations: int = 30, seed: int = 0,
        chunk: int = DEFAULT_CHUNK, workers: int = 1) -> tuple[Hologram, SolverTrace]:
    """Weighted iterations over the full pupil (solvers.py:238-244)."""
    if iterations < 1:
        raise InvalidParameterError("iterations must be >= 1")
    if chunk < 1 or workers < 1:
        raise InvalidParameterError("chunk and workers must be >= 1")
    return _single("wgs", pupil, spots, iterations, pupil.active_count, seed)


def cswgs(pupil: Pupil, spots: SpotSet, iterations: int, compression: float,
          seed: int = 0, chunk: int = DEFAULT_CHUNK,
          workers: int = 1) -> tuple[Hologram, SolverTrace]:
    """Compressed-subset weighted run (solvers.py:247-269)."""
    if iterations < 2:
        raise InvalidParameterError("cswgs needs iterations >= 2")
    plan = CompressionPlan.for_pupil(pupil, compression)
    if plan.subset_size < spots.count:
        warnings.warn(
            f"compressed subset of {plan.subset_size} pixels is smaller than "
            f"the {spots.count}-spot system; iterations are underdetermined",
            RuntimeWarning, stacklevel=2)
    if chunk < 1 or workers < 1:
        raise InvalidParameterError("chunk and workers must be >= 1")
    return _single("cswgs", pupil, spots, iterations, plan.subset_size, seed)


def solve(pupil: Pupil, spots: SpotSet, config: SolverConfig, chunk: int = DEFAULT_CHUNK,
          workers: int = 1) -> tuple[Hologram, SolverTrace]:
    """Dispatch a SolverConfig (solvers.py:272-282)."""
    if config.algorithm == "rs":
        return rs(pupil, spots, seed=config.seed, workers=workers)
    if config.algorithm == "wgs":
        return wgs(pupil, spots, iterations=config.iterations, seed=config.seed,
                   chunk=chunk, workers=workers)
    return cswgs(pupil, spots, iterations=config.iterations,
                 compression=config.compression, seed=config.seed, chunk=chunk,
                 workers=workers)


def solve_batch(pupil: Pupil, spot_sets, config: SolverConfig, seeds=None, raster: bool = False):
    """Solve many independent patterns (equal spot counts) in one graph replay.

    Returns a list of ``(Hologram, SolverTrace)``; pattern k uses solver seed
    ``seeds[k]`` (default ``config.seed + k``).  Each result is bitwise
    identical to solving that pattern alone.  A degenerate pattern raises
    :class:`DegenerateFieldError` only when its result is assembled.
    """
    sets = list(spot_sets)
    if not sets:
        return []
    seeds = [config.seed + k for k in range(len(sets))] if seeds is None else list(seeds)
    if len(seeds) != len(sets):
        raise InvalidParameterError("one seed per pattern")
    m = pupil.active_count
    subset = m
    if config.algorithm == "cswgs":
        subset = CompressionPlan.for_pupil(pupil, config.compression).subset_size
    t0 = time.perf_counter()
    res = _run_batch(config.algorithm, pupil, sets, config.iterations, subset, seeds,
                     raster=raster)
    return [_assemble(config.algorithm, pupil, s, res, b, config.iterations, subset, t0)
            for b, s in enumerate(sets)]


def wgs_step(pupil: Pupil, spots: SpotSet, state: WgsState, pixel_range=None,
             write_range=None, chunk: int = DEFAULT_CHUNK, workers: int = 1,
             tables: SpotTables | None = None):
    """One weighted iteration driven from the host (solvers.py:132-163).

    Uses the device forward and backward passes; the N-element weight update
    runs on the host like the reference's.  Solver runs never call this (they
    keep the whole loop on the device)."""
    fields = forward_project(pupil, state.hologram, spots, pixel_range, chunk=chunk,
                             workers=workers, tables=tables)
    mags = np.hypot(fields.real, fields.imag)
    weights, mags, degenerate = rebalance_weights(state.weights, mags)
    amplitudes = weights * spots.amplitude
    thetas = _field_phases(fields)
    if write_range is None:
        write_range = pixel_range
    frag = superpose(pupil, spots, SpotCoefficients(amplitudes, thetas), write_range,
                     workers=workers, tables=tables)
    start, stop = (0, pupil.active_count) if write_range is None else write_range
    phase = np.array(state.hologram.phase)
    phase[start:stop] = frag
    return WgsState(weights=weights, amplitudes=amplitudes, thetas=thetas,
                    hologram=Hologram(phase, pupil),
                    degenerate=state.degenerate or degenerate), mags


def predict_ops(algorithm: str, m: int, n: int, iterations: int = 1,
                compression: float = 1.0) -> int:
    """Cost-model units (solvers.py:285-295)."""
    if algorithm == "rs":
        return m * n
    if algorithm == "wgs":
        return m * n * iterations
    if algorithm == "cswgs":
        return 2 * m * n + math.ceil(compression * m) * n * (iterations - 2)
    raise InvalidParameterError(f"unknown algorithm {algorithm!r}")


@dataclass(frozen=True)
class PlannedRun:
    algorithm: str
    iterations: int
    over_budget: bool
    predicted_ops: int


def budget_controller(algorithm: str, m: int, n: int, budget_ops: int,
                      compression: float = 1.0) -> PlannedRun:
    """Largest iteration count within an op budget (solvers.py:308-331)."""
    if budget_ops <= 0:
        raise InvalidParameterError("budget_ops must be > 0")
    if algorithm == "rs":
        cost = predict_ops("rs", m, n)
        return PlannedRun("rs", 1, cost > budget_ops, cost)
    if algorithm == "wgs":
        iters = max(1, budget_ops // (m * n))
        cost = predict_ops("wgs", m, n, iters)
        return PlannedRun("wgs", iters, cost > budget_ops, cost)
    if algorithm == "cswgs":
        subset = math.ceil(compression * m)
        spare = budget_ops - 2 * m * n
        iters = 2 + max(0, spare // (subset * n)) if spare >= 0 else 2
        cost = predict_ops("cswgs", m, n, iters, compression)
        return PlannedRun("cswgs", iters, cost > budget_ops, cost)
    raise InvalidParameterError(f"unknown algorithm {algorithm!r}")
