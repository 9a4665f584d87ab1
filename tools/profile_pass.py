"""Launch one pass kernel configuration for ncu capture.

    python tools/profile_pass.py --which 0|1 --batch B [--reps R] [--solve]

which 0 = full-range fused pass, 1 = compressed-window pass (c = 1/16);
--solve runs one full CS-WGS solve instead (for launch lists).
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2003_05293_b200 as hs  # noqa: E402
from paper_2003_05293_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", type=int, default=0)
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--spots", type=int, default=100)
ap.add_argument("--solve", action="store_true")
ap.add_argument("--alg", default="cswgs", choices=["cswgs", "wgs"])
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()

pupil = hs.build_pupil(1152)
subset = math.ceil(pupil.active_count / 16)
plan = _lib.Plan(pupil, 0)
sets = [hs.random_foci(args.spots, 1000 + k) for k in range(args.batch)]
plan.set_spots(sets)
th = np.stack([np.random.default_rng(k).random(args.spots) * 2 * math.pi for k in range(args.batch)])
alg = _lib.ALG_CSWGS if args.alg == "cswgs" else _lib.ALG_WGS
sub = subset if args.alg == "cswgs" else pupil.active_count
plan.solve(alg, args.iters, sub, th)
if args.solve:
    plan.solve(alg, args.iters, sub, th)
else:
    ms, pairs = plan.time_kernel(args.which, subset, reps=args.reps)
    print(f"which={args.which} batch={args.batch} ms/launch={ms:.4f} pairs={pairs:.3e} "
          f"Gpairs/s={pairs / ms / 1e6:.1f}")
