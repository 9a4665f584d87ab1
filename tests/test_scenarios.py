"""Scenario frames and sweep CSV layouts vs fixtures made by the reference
(tests/golden/make_scenarios.py; holospots/scenarios.py, bench.py)."""

import json
import math
import os

import numpy as np
import pytest

import paper_2003_05293_b200 as hs
from paper_2003_05293_b200 import bench

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scenarios.json")))


def same(spots, ref):
    return all(np.array_equal(getattr(spots, k), np.array(ref[v]))
               for k, v in (("x", "x"), ("y", "y"), ("z", "z"), ("amplitude", "a0")))


@pytest.mark.parametrize("key", sorted(GOLD["frames"]))
def test_rotation_frames_bitwise(key):
    name, frames, step, axis = key.split("_", 3)
    step = None if step == "None" else float(step)
    axis = None if axis == "None" else tuple(float(v) for v in axis.strip("()").split(","))
    got = hs.rotation_sweep(hs.named_scenario(name), int(frames), step, axis)
    assert len(got) == len(GOLD["frames"][key])
    for s, ref in zip(got, GOLD["frames"][key]):
        assert same(s, ref)


def test_scenario_file(tmp_path):
    p = tmp_path / "pair.txt"
    p.write_text(GOLD["file_text"])
    sc = hs.load_scenario_file(p)
    assert sc.name == "pair" and sc.kind == "cubes"
    for s, ref in zip(hs.rotation_sweep(sc, 3), GOLD["file_frames"]):
        assert same(s, ref)


def test_scenario_validation(tmp_path):
    with pytest.raises(hs.InvalidParameterError):
        hs.named_scenario("nope")
    with pytest.raises(hs.InvalidParameterError):
        hs.rotation_sweep(hs.named_scenario("grid36"), 0)
    with pytest.raises(hs.OutOfFieldError):
        hs.grid_scenario(50, 50, 10e-6)
    with pytest.raises(hs.InvalidParameterError):
        hs.cubes_scenario(10e-6, (0, 0, 0), (0, 0, 0))
    with pytest.raises(hs.InvalidParameterError):
        hs.rotate_points(np.zeros((2, 3)), (0, 0, 0), 1.0)
    bad = tmp_path / "bad.txt"
    bad.write_text("type = ring\n")
    with pytest.raises(hs.InvalidParameterError):
        hs.load_scenario_file(bad)
    # frame 0 of a grid is the unrotated grid of workloads.grid_spots
    assert same(hs.rotation_sweep(hs.named_scenario("grid100"), 3)[0],
                {"x": hs.named_spots("grid100").x, "y": hs.named_spots("grid100").y,
                 "z": hs.named_spots("grid100").z, "a0": hs.named_spots("grid100").amplitude})


def test_csv_layouts_match_reference():
    recs = [bench.BenchRecord(*r) for r in GOLD["csv_records"]]
    assert bench.format_records_csv(recs) == GOLD["csv_records_text"]
    assert bench.format_summary_csv(bench.summarize(recs)) == GOLD["csv_summary_text"]
    stats = bench.summarize(recs)
    assert [s.runs for s in stats] == [1, 1, 2]
    assert math.isclose(stats[2].mean_efficiency, 0.6)


def test_budget_planning_host():
    m, n = 51472, 36
    plan = hs.budget_controller("cswgs", m, n, 5 * m * n, compression=1 / 16)
    assert plan.iterations == 2 + (3 * m * n) // (math.ceil(m / 16) * n)
    assert not plan.over_budget
    assert bench.frame_budget_ops(64.0, ops_per_ms=1e6) == 64_000_000
    with pytest.raises(hs.InvalidParameterError):
        bench.frame_budget_ops(0.0, ops_per_ms=1.0)
