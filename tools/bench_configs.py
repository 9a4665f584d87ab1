"""Per-configuration timings on one GPU (SURVEY.md 8(d) configs 1-4 + batch sweep).

    python tools/bench_configs.py [--out profiles/round1/configs.jsonl]

Each line: config, ms per solve (CUDA events on the plan stream, graph
replay, B patterns per solve), holograms/s, e / u of pattern 0, and the
reference's e / u for the same inputs where tests/golden holds them.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_05293_b200 as hs  # noqa: E402
from paper_2003_05293_b200 import _lib  # noqa: E402

GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def time_solve(plan, alg, iters, subset, theta0, reps):
    plan.solve(alg, iters, subset, theta0)           # graph build + warm
    plan.solve(alg, iters, subset, theta0)
    st = torch.cuda.ExternalStream(plan.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        plan.solve(alg, iters, subset, theta0, sync=False)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(name, pupil, sets, alg, iters, subset, reps, golden=None, ref=None):
    plan = _lib.Plan(pupil, 0)
    plan.set_spots(sets)
    n = sets[0].count
    th = np.stack([np.random.default_rng(k).random(n) * 2 * math.pi for k in range(len(sets))])
    ms = time_solve(plan, alg, iters, subset, th, reps)
    e, u, *_ = plan.quality_batch()
    line = {"config": name, "batch": len(sets), "spots": n, "side": pupil.side_px,
            "ms_per_solve": ms, "ms_per_hologram": ms / len(sets),
            "holograms_per_s": 1e3 * len(sets) / ms, "e": float(e[0]), "u": float(u[0])}
    if golden:
        g = GOLDEN["solves"][golden]
        line.update(ref_e=g["e"], ref_u=g["u"], de=abs(g["e"] - float(e[0])),
                    du=abs(g["u"] - float(u[0])))
    if ref:
        line.update(ref)
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    lines = []
    p512 = hs.build_pupil(512)
    p1152 = hs.build_pupil(1152)
    m512, m1152 = p512.active_count, p1152.active_count
    # golden inputs use solver seed 0 for pattern 0
    lines.append(run("1: cswgs 512^2 N=10 c=1/8 I=10", p512, [hs.random_foci(10, 12345)],
                     _lib.ALG_CSWGS, 10, math.ceil(m512 / 8), 50, golden="cfg1"))
    lines.append(run("2: rs 1152^2 N=100", p1152, [hs.random_foci(100, 12345)],
                     _lib.ALG_RS, 0, m1152, 50, golden="cfg2_rs"))
    lines.append(run("3: cswgs 1152^2 N=100 c=1/16 I=20 grid100", p1152, [hs.named_spots("grid100")],
                     _lib.ALG_CSWGS, 20, math.ceil(m1152 / 16), 20, golden="cfg3_grid100"))
    lines.append(run("3: cswgs 1152^2 N=100 c=1/16 I=20 random", p1152, [hs.random_foci(100, 12345)],
                     _lib.ALG_CSWGS, 20, math.ceil(m1152 / 16), 20, golden="cfg3_random"))
    lines.append(run("4: wgs 1152^2 N=1000 I=30 (square proxy of 1920x1152)", p1152,
                     [hs.random_foci(1000, 4, xy=150e-6)], _lib.ALG_WGS, 30, m1152, 3,
                     ref={"ref_e": 0.9065, "ref_u": 0.1580,
                          "ref_source": "SURVEY.md 6.2 (reference, 8 cores, 17.66 s)"}))
    for b in (8, 32, 64, 128):
        sets = [hs.random_foci(100, 1000 + k) for k in range(b)]
        lines.append(run(f"5: batched cswgs 1152^2 N=100 c=1/16 I=20 (B={b})", p1152, sets,
                         _lib.ALG_CSWGS, 20, math.ceil(m1152 / 16), 5))
    if args.out:
        with open(args.out, "w") as fh:
            for ln in lines:
                fh.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()
