"""Generate tests/golden/scenarios.json from the reference's scenarios module.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_scenarios.py

Frames of the stock scenarios under rotation_sweep (scenarios.py:126-142),
a custom step / axis, and a parsed scenario file (scenarios.py:162-205),
so tests/test_scenarios.py can check the restatement bit for bit without
the reference present.
"""
import json
import os
import tempfile

import holospots as ref


def pts(s):
    return {"x": s.x.tolist(), "y": s.y.tolist(), "z": s.z.tolist(), "a0": s.amplitude.tolist()}


out = {"frames": {}}
for name, frames, step, axis in [("grid100", 4, None, None), ("cubes", 6, None, None),
                                 ("grid36", 3, 0.3, (0.0, 1.0, 1.0)), ("cubes", 2, 1.1, (1.0, 0.0, 0.0))]:
    key = f"{name}_{frames}_{step}_{axis}"
    out["frames"][key] = [pts(s) for s in ref.rotation_sweep(ref.named_scenario(name), frames, step, axis)]
text = """# test scenario
name = pair
type = cubes
edge_um = 40
center1_um = -50, 10, 0
center2_um = 55, -5, 10
axis = 0, 1, 0.5
step_deg = 15
fov_um = 300
"""
with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as fh:
    fh.write(text)
sc = ref.load_scenario_file(fh.name)
os.unlink(fh.name)
out["file_text"] = text
out["file_frames"] = [pts(s) for s in ref.rotation_sweep(sc, 3)]
# CSV layouts (bench.py:223-262) on records with every column kind
from holospots import bench as rb  # noqa: E402

recs = [rb.BenchRecord("grid36", "rs", 1.0, 1, 1852848, 6.817206, 0.84010388, 0.285852468, 1, ""),
        rb.BenchRecord("grid36", "cswgs", 0.0625, 50, 123456789, 0.1234567891, 0.9187, 0.9423, 2,
                       "over_budget"),
        rb.BenchRecord("cubes", "wgs", 1.0, 3, 0, 1.5, float("nan"), float("nan"), 3,
                       "over_budget+failed:DegenerateFieldError"),
        rb.BenchRecord("cubes", "wgs", 1.0, 3, 999, 2.0, 0.5, 0.25, 4, "degenerate"),
        rb.BenchRecord("cubes", "wgs", 1.0, 3, 999, 2.0, 0.7, 0.35, 5, "")]
out["csv_records"] = [[r.scenario, r.algorithm, r.c, r.iterations, r.ops, r.wall_ms, r.efficiency,
                       r.uniformity, r.seed, r.flags] for r in recs]
out["csv_records_text"] = rb.format_records_csv(recs)
out["csv_summary_text"] = rb.format_summary_csv(rb.summarize(recs))
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenarios.json"), "w"))
print("wrote", len(out["frames"]), "frame sets")
