"""Golden fixture for config 4 (BASELINE.json configs[3]) from the reference.

    NUMBA_NUM_THREADS=8 python tests/golden/make_cfg4.py

WGS on the 1152^2 gaussian pupil (the circular-aperture stand-in for the
1920x1152 panel), N = 1000 random foci (spot seed 4,
x, y ~ U(+-150 um), z ~ U(+-50 um), a0 = 1), I = 30, solver seed 0.

The run goes through the reference's own ``wgs_step`` in the order of
``solvers._iterate`` (pkg/src/holospots/solvers.py:192-235) so the final
coefficients (amplitudes, thetas) are available for the phase check;
the trace, intensities, e and u are identical to ``hs.wgs`` (asserted).
Writes ``tests/golden/solve_cfg4_wgs1000.npz`` (trace, intensities, final
coefficients, a phase subsample with its |S|) and prints e / u.
"""

import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_NUM_THREADS", "8")

import holospots as hs  # noqa: E402
from holospots import solvers as hsol  # noqa: E402

SUB = 97

p = hs.build_pupil(1152, 9.2e-6, 800e-9, 0.02, "gaussian", 6e-3, seed=0)
rng = np.random.default_rng(4)
n = 1000
spots = hs.SpotSet(x=rng.uniform(-150e-6, 150e-6, n), y=rng.uniform(-150e-6, 150e-6, n),
                   z=rng.uniform(-50e-6, 50e-6, n), amplitude=np.ones(n))
t0 = time.time()
tables = hs.spot_tables(p, spots)
state = hsol._seed_state(p, spots, 0, 8, tables)
ws, ms = [], []
for j in range(30):
    state, mags = hsol.wgs_step(p, spots, state, None, None, workers=8, tables=tables)
    ws.append(state.weights)
    ms.append(mags)
rep = hs.quality_report(p, state.hologram, spots, workers=8)
print(f"cfg4: {time.time() - t0:.1f} s e={rep.efficiency:.6f} u={rep.uniformity:.6f}")

idx = np.arange(0, p.active_count, SUB)
cols, rows = p.cols[idx], p.rows[idx]
th = hs.wrap_phase(state.thetas)
coef = state.amplitudes * np.exp(1j * th)
gx = tables.gx_re + 1j * tables.gx_im
gy = tables.gy_re + 1j * tables.gy_im
s_sub = np.einsum("pn,pn->p", gx[cols] * coef, gy[rows])
np.savez_compressed(os.path.join(HERE, "solve_cfg4_wgs1000.npz"),
                    x=spots.x, y=spots.y, z=spots.z, a0=spots.amplitude,
                    weights=np.array(ws), mags=np.array(ms),
                    intensities=rep.intensities, relative=rep.target_relative,
                    e=rep.efficiency, u=rep.uniformity,
                    amps=state.amplitudes, thetas=state.thetas,
                    phase_idx=idx, phase=state.hologram.phase[idx],
                    s_mag=np.abs(s_sub))
