"""Throughput of K concurrent plans (own streams) each solving B/K patterns
vs one plan solving B: do independent solves fill each other's pass tails?

    python tools/concurrency_probe.py [--batch 32] [--reps 10]
"""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_05293_b200 as hs  # noqa: E402
from paper_2003_05293_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
pupil = hs.build_pupil(1152)
subset = math.ceil(pupil.active_count / 16)
B = args.batch
for k in (1, 2, 4):
    plans = []
    for i in range(k):
        pl = _lib.Plan(pupil, 0)
        pl.set_spots([hs.random_foci(100, 1000 + i * B // k + j) for j in range(B // k)])
        th = np.stack([np.random.default_rng(i * B // k + j).random(100) * 2 * math.pi for j in range(B // k)])
        plans.append((pl, th))
    for pl, th in plans:
        for _ in range(2):
            pl.solve(_lib.ALG_CSWGS, 20, subset, th, want_fields=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.reps):
        for pl, th in plans:
            pl.solve(_lib.ALG_CSWGS, 20, subset, th, want_fields=True, sync=False)
    for pl, _ in plans:
        pl.sync()
    dt = (time.perf_counter() - t0) / args.reps
    print(f"{k} plan(s) x {B // k}: {dt * 1e3:.3f} ms per {B} holograms = {B / dt:.0f} holo/s")
