"""Device-batched sweeps, budget comparisons and sequences (SURVEY.md 8(f)
rows 3-4) against the reference's golden compression table
(demos/output/compression_runs.csv rows 2-41, tests/golden/golden.json)."""

import math

import numpy as np
import pytest

import paper_2003_05293_b200 as hs
from paper_2003_05293_b200 import bench

pytestmark = pytest.mark.gpu
EU_ATOL = 1e-3


def test_compare_at_budget_reproduces_golden_table(golden, pupils):
    p = pupils["p256u0"]
    m, n = p.active_count, 36
    cs = [2.0 ** -k for k in range(1, 7)]
    summary, records = bench.compare_at_budget(p, hs.named_scenario("grid36"), 5 * m * n,
                                               range(5), c_values=cs)
    rows = golden["compression_runs"]
    assert len(records) == len(rows) == 40
    for rec, row in zip(records, rows):
        assert (rec.algorithm, rec.c, rec.seed) == (row["algorithm"], row["c"], row["seed"])
        assert rec.iterations == row["iterations"] and rec.ops == row["ops"]
        assert "failed" not in rec.flags
        # every row, including the long compressed runs (I = 97, 193): the
        # small windows run the fp64 passes under precision "auto"
        assert abs(rec.efficiency - row["e"]) <= EU_ATOL, (row, rec)
        assert abs(rec.uniformity - row["u"]) <= EU_ATOL, (row, rec)
    assert summary.rs.runs == summary.wgs.runs == 5
    assert summary.best in summary.cswgs_cells
    assert summary.best_c in cs
    assert bench.format_records_csv(records).count("\n") == 41


def test_sweep_grid_and_failure_isolation(pupils):
    p = pupils["p64u0"]
    scen = [hs.named_scenario("grid36"), hs.named_scenario("cubes")]
    recs = bench.sweep(p, scen, ["wgs", "cswgs"], [0.5, 0.25], 10 * p.active_count * 36, [0, 1, 2])
    assert len(recs) == 2 * 2 * 2 * 3
    assert [r.scenario for r in recs[:12]] == ["grid36"] * 12
    assert all(math.isfinite(r.efficiency) for r in recs)
    # a cell that cannot run is recorded, not raised: zero illumination
    dark = hs.build_pupil(32, illumination="gaussian", waist=1e-12, seed=0)
    rec = bench.run_cell(dark, hs.named_spots("grid36"), "grid36", "wgs", 1.0, 10 ** 9, 0)
    if "failed" in rec.flags:
        assert math.isnan(rec.efficiency) and rec.ops == 0
    with pytest.raises(hs.InvalidParameterError):
        bench.sweep(p, [], ["wgs"], [1.0], 100, [0])


def test_single_cell_matches_batched_cells(pupils):
    p = pupils["p64u0"]
    frames = hs.rotation_sweep(hs.named_scenario("grid36"), 3)
    batched = bench.run_cells(p, frames, "grid36", "cswgs", 0.25, 8 * p.active_count * 36, [0, 1, 2])
    for k in range(3):
        one = bench.run_cell(p, frames[k], "grid36", "cswgs", 0.25, 8 * p.active_count * 36, k)
        assert (one.efficiency, one.uniformity, one.ops) == \
            (batched[k].efficiency, batched[k].uniformity, batched[k].ops)


def test_calibration_and_frame_budget():
    rate = bench.calibrate_ops_per_ms(repeats=2)
    assert rate > 0
    thr = bench.calibrate_ops_per_ms(batch=16, repeats=2)
    assert thr > rate  # batching amortises launch latency
    assert bench.frame_budget_ops(64.0, ops_per_ms=rate) == int(64.0 * rate)


def test_sequences_cold_and_warm(pupils):
    p = pupils["p256u0"]
    cfg = hs.SolverConfig("cswgs", iterations=8, compression=1 / 8, seed=0)
    frames = hs.rotation_sweep(hs.named_scenario("grid36"), 6, step_angle=0.05)
    cold = hs.solve_sequence(p, frames, cfg)
    batch = hs.solve_batch(p, frames, cfg, seeds=list(range(6)))
    for (h1, _), (h2, _) in zip(cold, batch):
        assert np.array_equal(h1.phase, h2.phase)
    warm = hs.solve_sequence(p, frames, cfg, warm_start=True)
    assert np.array_equal(warm[0][0].phase, cold[0][0].phase)   # frame 0 starts from its seed
    qc = hs.sequence_quality(cold)
    qw = hs.sequence_quality(warm)
    assert np.all(np.isfinite(qw)) and qw.shape == (6, 2)
    # neighbouring frames differ by 0.05 rad: the warm start lands at least as
    # uniform on average as random restarts
    assert qw[1:, 1].mean() >= qc[1:, 1].mean() - 0.05
    with pytest.raises(hs.InvalidParameterError):
        hs.solve_sequence(p, [frames[0], hs.named_spots("grid100")], cfg)
