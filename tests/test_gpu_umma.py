"""Both full-range pass implementations stay under the parity bar.  The
default for np <= 112 is the tcgen05 pass (csrc/hs_umma.cuh), which the rest
of the GPU suite exercises; this re-runs the solver cases of
test_gpu_parity.py (golden runs, the grid100 quality gate, bitwise
repeatability / batch invariance, c=1 == WGS) in a child process with the
FFMA tile pass (csrc/hs_tile.cuh, HS_UMMA=0) selected at plan creation.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_parity_with_ffma_full_pass():
    env = dict(os.environ, HS_UMMA="0", HS_PRECISION="fp32")
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
         os.path.join(HERE, "test_gpu_parity.py"), os.path.join(HERE, "test_gpu_spot_chunks.py"),
         "-k", "solver_matches or quality_gate or bitwise or wgs_equals or trace_weight or pipelined"
               " or spot_chunk"],
        env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= 21, r.stdout[-2000:]
