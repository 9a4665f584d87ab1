"""Single-hologram (B = 1) breakdown: per-pass kernel times (back-to-back
launches, L2-warm, CUDA events) next to the whole solve-graph replay.

    python tools/b1_probe.py
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_05293_b200 as hs  # noqa: E402
from paper_2003_05293_b200 import _lib  # noqa: E402

p = hs.build_pupil(1152)
sub = math.ceil(p.active_count / 16)
plan = _lib.Plan(p, 0)
plan.set_spots([hs.named_spots("grid100")])
th = np.random.default_rng(0).random((1, 100)) * 2 * math.pi
for _ in range(3):
    plan.solve(_lib.ALG_CSWGS, 20, sub, th, want_fields=True)
st = torch.cuda.ExternalStream(plan.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(50):
    plan.solve(_lib.ALG_CSWGS, 20, sub, th, want_fields=True, sync=False)
e1.record(st)
torch.cuda.synchronize()
solve = e0.elapsed_time(e1) / 50
full = plan.time_kernel(0, reps=50)[0]
final = plan.time_kernel(3, reps=50)[0]
win = plan.time_kernel(1, sub, reps=100)[0]
print(f"B=1 solve {solve * 1e3:.1f} us; per launch (back to back): full {full * 1e3:.1f} us, "
      f"final {final * 1e3:.1f} us, window {win * 1e3:.1f} us; "
      f"2 full + 19 windows = {(full + final + 19 * win) * 1e3:.1f} us")
