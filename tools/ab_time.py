"""A/B kernel timings of two library builds (HS_LIB_PATH selects the .so).

    HS_LIB_PATH=abtest/old.so python tools/ab_time.py; python tools/ab_time.py
Prints the bench workload's per-launch pass times (hs_time_kernel) and the
B = 32 solve time."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_05293_b200 as hs  # noqa: E402
from paper_2003_05293_b200 import _lib  # noqa: E402

B = int(os.environ.get("AB_BATCH", "32"))
p = hs.build_pupil(1152)
m = p.active_count
sub = math.ceil(m / 16)
plan = _lib.Plan(p, 0)
sets = [hs.random_foci(100, 1000 + k) for k in range(B)]
plan.set_spots(sets)
th = np.stack([np.random.default_rng(k).random(100) * 2 * math.pi for k in range(B)])
for _ in range(3):
    plan.solve(_lib.ALG_CSWGS, 20, sub, th)
st = torch.cuda.ExternalStream(plan.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20):
    plan.solve(_lib.ALG_CSWGS, 20, sub, th, sync=False)
e1.record(st)
torch.cuda.synchronize()
print(os.environ.get("HS_LIB_PATH", "current"), "solve B=%d: %.3f ms" % (B, e0.elapsed_time(e1) / 20),
      "full %.4f final %.4f window %.4f" % (plan.time_kernel(0, reps=10)[0], plan.time_kernel(2, reps=10)[0],
                                             plan.time_kernel(1, sub, reps=30)[0]),
      "final-codes %.4f" % plan.time_kernel(3, reps=10)[0] if os.environ.get("HS_LIB_PATH") is None else "")
