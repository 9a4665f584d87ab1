"""Budgeted sweeps, three-way comparisons and machine calibration on the device.

The reference's ``holospots.bench`` harness (bench.py:1-282) runs every
(scenario, algorithm, c, seed) cell as its own CPU solve.  Here the cells
that share (algorithm, c) -- one per seed, on rotation frame k for seed k
(bench.py:120-126) -- are one batched device solve: the patterns are
independent and equal-sized, so the whole seed axis replays one CUDA graph
(``solvers._run_batch``), and each record's ``wall_ms`` is that batch's
wall time divided by its cells (the amortised per-hologram cost).  Every
other column follows the reference: iteration counts from
``budget_controller`` (solvers.py:322-331), exact ``ops``, e / u from the
final pass's fields (the fused quality report, within 1e-5 / 1e-4 of a
re-projected ``quality_report``), flags ``over_budget`` / ``degenerate`` /
``failed:<Error>``, NaN metrics on failure, and the pinned CSV layout
(bench.py:223-262).  Re-running a configuration reproduces every column
bit for bit except wall time.

``calibrate_ops_per_ms`` measures the device's cost-model units per
millisecond, so a frame budget (``DEFAULT_FRAME_MS`` = 64 ms) becomes an
operation budget via ``frame_budget_ops``.
"""

from __future__ import annotations

import io
import math
import time
from dataclasses import dataclass

import numpy as np

from . import solvers
from .errors import DegenerateFieldError, HoloError, InvalidParameterError
from .kernels import DEFAULT_CHUNK
from .optics import CompressionPlan, Pupil, SpotSet, build_pupil
from .scenarios import Scenario, grid_scenario, rotation_sweep

CSV_HEADER = "scenario,algorithm,c,iterations,ops,wall_ms,efficiency,uniformity,seed,flags"
DEFAULT_C_SWEEP = tuple(2.0 ** -k for k in range(1, 9))   # 2^-1 .. 2^-8
DEFAULT_FRAME_MS = 64.0


@dataclass(frozen=True)
class BenchRecord:
    """One (scenario, algorithm, c, seed) cell (bench.py:34-46)."""

    scenario: str
    algorithm: str
    c: float
    iterations: int
    ops: int
    wall_ms: float
    efficiency: float
    uniformity: float
    seed: int
    flags: str


@dataclass(frozen=True)
class CellStats:
    """Across-seed statistics of one (scenario, algorithm, c) cell (bench.py:49-61)."""

    scenario: str
    algorithm: str
    c: float
    iterations: int
    runs: int
    mean_efficiency: float
    std_efficiency: float
    mean_uniformity: float
    std_uniformity: float


@dataclass(frozen=True)
class BudgetComparison:
    """RS / WGS / best-c compressed summary at one budget (bench.py:166-179)."""

    scenario: str
    budget_ops: int
    rs: CellStats
    wgs: CellStats
    cswgs_cells: tuple
    best: CellStats

    @property
    def best_c(self) -> float:
        return self.best.c


def _g9(x: float) -> str:
    return format(x, ".9g")


def _failed(scenario, algorithm, c, iterations, seed, wall_ms, flags, exc) -> BenchRecord:
    return BenchRecord(scenario=scenario, algorithm=algorithm, c=c, iterations=iterations, ops=0,
                       wall_ms=wall_ms, efficiency=float("nan"), uniformity=float("nan"),
                       seed=seed, flags="+".join(flags + [f"failed:{type(exc).__name__}"]))


def run_cells(pupil: Pupil, frames, scenario_name: str, algorithm: str, c: float,
              budget_ops: int, seeds) -> list[BenchRecord]:
    """The cells of one (algorithm, c) over a seed axis as ONE batched device
    solve; frame k pairs with seed k.  Per-cell failures are isolated."""
    frames, seeds = list(frames), [int(s) for s in seeds]
    if len(frames) != len(seeds):
        raise InvalidParameterError("one frame per seed")
    m = pupil.active_count
    n = frames[0].count
    plan = solvers.budget_controller(algorithm, m, n, budget_ops, compression=c)
    base_flags = ["over_budget"] if plan.over_budget else []
    iters = plan.iterations
    t0 = time.perf_counter()
    try:
        if any(f.count != n for f in frames):
            raise InvalidParameterError("a batched cell needs equal spot counts")
        subset = m
        if algorithm == "cswgs":
            subset = CompressionPlan.for_pupil(pupil, c).subset_size
        res = solvers._run_batch(algorithm, pupil, frames, iters, subset, seeds, fetch_phase=False)
    except HoloError:
        if len(frames) == 1:
            raise
        # isolate the failing cell(s): fall back to one solve per cell
        out = []
        for f, s in zip(frames, seeds):
            try:
                out.extend(run_cells(pupil, [f], scenario_name, algorithm, c, budget_ops, [s]))
            except HoloError as exc:
                out.append(_failed(scenario_name, algorithm, c, iters, s,
                                   (time.perf_counter() - t0) * 1e3, base_flags, exc))
        return out
    wall_ms = (time.perf_counter() - t0) * 1e3 / len(frames)
    sizes = [m] if algorithm == "rs" else solvers.window_sizes(m, subset, iters)
    ops = sum(sizes) * n
    records = []
    for b, seed in enumerate(seeds):
        flags = list(base_flags)
        try:
            solvers._raise_status(int(res.status[b]))
        except (DegenerateFieldError, HoloError) as exc:
            records.append(_failed(scenario_name, algorithm, c, iters, seed, wall_ms, flags, exc))
            continue
        if algorithm != "rs" and int(res.first_degenerate[b]):
            flags.append("degenerate")
        records.append(BenchRecord(scenario=scenario_name, algorithm=algorithm, c=c,
                                   iterations=iters, ops=ops, wall_ms=wall_ms,
                                   efficiency=float(res.efficiency[b]),
                                   uniformity=float(res.uniformity[b]), seed=seed,
                                   flags="+".join(flags)))
    return records


def run_cell(pupil: Pupil, spots: SpotSet, scenario_name: str, algorithm: str,
             c: float, budget_ops: int, seed: int, chunk: int = DEFAULT_CHUNK,
             workers: int = 1) -> BenchRecord:
    """One budgeted cell (bench.py:69-98); ``chunk`` / ``workers`` are
    accepted for signature compatibility and never change results."""
    if chunk < 1 or workers < 1:
        raise InvalidParameterError("chunk and workers must be >= 1")
    t0 = time.perf_counter()
    try:
        return run_cells(pupil, [spots], scenario_name, algorithm, c, budget_ops, [seed])[0]
    except HoloError as exc:
        plan = solvers.budget_controller(algorithm, pupil.active_count, spots.count, budget_ops,
                                         compression=c)
        flags = ["over_budget"] if plan.over_budget else []
        return _failed(scenario_name, algorithm, c, plan.iterations, seed,
                       (time.perf_counter() - t0) * 1e3, flags, exc)


def sweep(pupil: Pupil, scenarios, algorithms, c_values, budget_ops: int, seeds,
          chunk: int = DEFAULT_CHUNK, workers: int = 1) -> list[BenchRecord]:
    """Full factorial sweep in configuration order (bench.py:101-126): exactly
    len(scenarios) * len(algorithms) * len(c_values) * len(seeds) rows;
    the seed axis of each (scenario, algorithm, c) is one device batch."""
    scenarios, algorithms = list(scenarios), list(algorithms)
    c_values, seeds = [float(c) for c in c_values], list(seeds)
    if not scenarios or not algorithms or not c_values or not seeds:
        raise InvalidParameterError("sweep axes must be non-empty")
    if budget_ops <= 0:
        raise InvalidParameterError("budget_ops must be > 0")
    if chunk < 1 or workers < 1:
        raise InvalidParameterError("chunk and workers must be >= 1")
    records = []
    for scenario in scenarios:
        frames = rotation_sweep(scenario, len(seeds))
        for algorithm in algorithms:
            for c in c_values:
                records.extend(run_cells(pupil, frames, scenario.name, algorithm, c,
                                         budget_ops, seeds))
    return records


def summarize(records) -> list[CellStats]:
    """Across-seed mean and sample std per cell, failed runs excluded, cells in
    first-occurrence order (bench.py:129-163)."""
    groups: dict[tuple, list[BenchRecord]] = {}
    for rec in records:
        groups.setdefault((rec.scenario, rec.algorithm, rec.c), []).append(rec)
    out = []
    for key, recs in groups.items():
        ok = [r for r in recs if "failed" not in r.flags]
        if not ok:
            nan = float("nan")
            out.append(CellStats(*key, iterations=0, runs=0, mean_efficiency=nan,
                                 std_efficiency=nan, mean_uniformity=nan, std_uniformity=nan))
            continue
        e = np.array([r.efficiency for r in ok])
        u = np.array([r.uniformity for r in ok])
        out.append(CellStats(*key, iterations=ok[0].iterations, runs=len(ok),
                             mean_efficiency=float(np.mean(e)),
                             std_efficiency=float(np.std(e, ddof=1)) if e.size > 1 else 0.0,
                             mean_uniformity=float(np.mean(u)),
                             std_uniformity=float(np.std(u, ddof=1)) if u.size > 1 else 0.0))
    return out


def compare_at_budget(pupil: Pupil, scenario: Scenario, budget_ops: int, seeds,
                      c_values=DEFAULT_C_SWEEP, chunk: int = DEFAULT_CHUNK,
                      workers: int = 1) -> tuple[BudgetComparison, list[BenchRecord]]:
    """RS and WGS once per seed, CS-WGS over the c axis, best c by mean
    uniformity (bench.py:182-214)."""
    seeds = list(seeds)
    if not seeds:
        raise InvalidParameterError("seeds must be non-empty")
    if chunk < 1 or workers < 1:
        raise InvalidParameterError("chunk and workers must be >= 1")
    frames = rotation_sweep(scenario, len(seeds))
    records: list[BenchRecord] = []
    for algorithm, cs in (("rs", [1.0]), ("wgs", [1.0]), ("cswgs", [float(c) for c in c_values])):
        for c in cs:
            records.extend(run_cells(pupil, frames, scenario.name, algorithm, c, budget_ops, seeds))
    stats = summarize(records)
    rs_cell = next(s for s in stats if s.algorithm == "rs")
    wgs_cell = next(s for s in stats if s.algorithm == "wgs")
    cs_cells = tuple(s for s in stats if s.algorithm == "cswgs")
    best = max(cs_cells, key=lambda s: -1.0 if math.isnan(s.mean_uniformity) else s.mean_uniformity)
    return BudgetComparison(scenario=scenario.name, budget_ops=budget_ops, rs=rs_cell,
                            wgs=wgs_cell, cswgs_cells=cs_cells, best=best), records


# ---------------------------------------------------------------- CSV output
def format_records_csv(records) -> str:
    """Pinned per-run table: UTF-8, LF, floats at 9 significant digits (bench.py:223-235)."""
    buf = io.StringIO()
    buf.write(CSV_HEADER + "\n")
    for r in records:
        buf.write(",".join([r.scenario, r.algorithm, _g9(r.c), str(r.iterations), str(r.ops),
                            _g9(r.wall_ms), _g9(r.efficiency), _g9(r.uniformity), str(r.seed),
                            r.flags]) + "\n")
    return buf.getvalue()


def write_records_csv(path, records) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(format_records_csv(records))


def format_summary_csv(stats) -> str:
    """Across-seed statistics table (bench.py:243-256)."""
    buf = io.StringIO()
    buf.write("scenario,algorithm,c,iterations,runs,"
              "mean_efficiency,std_efficiency,mean_uniformity,std_uniformity\n")
    for s in stats:
        buf.write(",".join([s.scenario, s.algorithm, _g9(s.c), str(s.iterations), str(s.runs),
                            _g9(s.mean_efficiency), _g9(s.std_efficiency),
                            _g9(s.mean_uniformity), _g9(s.std_uniformity)]) + "\n")
    return buf.getvalue()


def write_summary_csv(path, stats) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(format_summary_csv(stats))


# ------------------------------------------------------------ calibration
def calibrate_ops_per_ms(side_px: int = 256, n_spots: int = 36, iterations: int = 6,
                         chunk: int = DEFAULT_CHUNK, workers: int = 1, batch: int = 1,
                         repeats: int = 5) -> float:
    """Device cost-model units per millisecond (bench.py:265-282).

    Same representative run as the reference -- WGS on a uniform
    ``side_px`` pupil with a ~``n_spots`` grid -- but warmed (graph built)
    and timed as the best of ``repeats`` wall-clock solves.  ``batch`` > 1
    times that many patterns per solve (throughput calibration for batched
    sweeps; 1 = single-frame latency, the video-rate case).
    """
    if chunk < 1 or workers < 1 or batch < 1 or repeats < 1:
        raise InvalidParameterError("chunk, workers, batch and repeats must be >= 1")
    pupil = build_pupil(side_px, illumination="uniform", seed=0)
    rows = max(1, int(round(n_spots ** 0.5)))
    spots = grid_scenario(rows, max(1, n_spots // rows), 10e-6)
    m, n = pupil.active_count, spots.count
    seeds = list(range(batch))
    solvers._run_batch("wgs", pupil, [spots] * batch, iterations, m, seeds, fetch_phase=False)
    best = math.inf
    for _ in range(repeats):
        t0 = time.perf_counter()
        solvers._run_batch("wgs", pupil, [spots] * batch, iterations, m, seeds, fetch_phase=False)
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return batch * m * n * iterations / best


def frame_budget_ops(frame_ms: float = DEFAULT_FRAME_MS, ops_per_ms: float | None = None) -> int:
    """Operation budget of one frame: ``frame_ms`` x the calibrated rate."""
    if frame_ms <= 0:
        raise InvalidParameterError("frame_ms must be > 0")
    rate = calibrate_ops_per_ms() if ops_per_ms is None else ops_per_ms
    if rate <= 0:
        raise InvalidParameterError("ops_per_ms must be > 0")
    return max(1, int(frame_ms * rate))
