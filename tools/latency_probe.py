"""Single-hologram (B = 1) solve: CUDA-event time of one graph replay.

    python tools/latency_probe.py [--reps 20] [--solves 1]

Used under ncu to get the per-kernel launch list of one B = 1 solve.
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_05293_b200 as hs  # noqa: E402
from paper_2003_05293_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--batch", type=int, default=1)
args = ap.parse_args()
pupil = hs.build_pupil(1152)
subset = math.ceil(pupil.active_count / 16)
plan = _lib.Plan(pupil, 0)
sets = [hs.named_spots("grid100")] * args.batch
plan.set_spots(sets)
th = np.stack([np.random.default_rng(k).random(100) * 2 * math.pi for k in range(args.batch)])
for _ in range(3):
    plan.solve(_lib.ALG_CSWGS, 20, subset, th, want_fields=True)
st = torch.cuda.ExternalStream(plan.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(args.reps):
    plan.solve(_lib.ALG_CSWGS, 20, subset, th, want_fields=True, sync=False)
e1.record(st)
torch.cuda.synchronize()
print(f"B={args.batch}: {e0.elapsed_time(e1) / args.reps:.4f} ms per solve")
