"""Golden fixtures for rectangular full panels (``build_panel``) from the reference.

    NUMBA_NUM_THREADS=8 python tests/golden/make_panel.py

The reference only builds circular apertures (pkg/src/holospots/optics.py:
150-214), but its ``Pupil`` is a plain dataclass of storage-order arrays and
every kernel and solver reads only those arrays (kernels.py:78-144,
solvers.py:166-269).  So a rectangular panel is fed to the reference's own
code by constructing its ``Pupil`` from the arrays of our ``build_panel``
(the geometry is ours; the algorithm under test is the reference's).
Writes ``tests/golden/panel.npz`` (full phases, trace, intensities, e, u,
ops per case) and pins the oracle and the device path for non-circular
apertures, including the 1920 x 1152 panel's shape at reduced size.
"""

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
os.environ.setdefault("NUMBA_NUM_THREADS", "8")
sys.path.insert(0, ROOT)
import paper_2003_05293_b200 as ours  # noqa: E402  (geometry only: build_panel)

sys.path.insert(0, REF)
import holospots as hs  # noqa: E402

# (name, width, height, illumination kwargs, spots: (n, seed, xy, z), algorithm, I, c, seed)
CASES = [
    ("wgs_40x24", 40, 24, dict(illumination="uniform"), (6, 11, 6e-5, 2e-4), "wgs", 6, 1.0, 1),
    ("cswgs_64x36", 64, 36, dict(illumination="gaussian", waist=2e-4), (20, 12, 6e-5, 2e-4),
     "cswgs", 8, 0.25, 2),
    ("rs_96x64", 96, 64, dict(illumination="gaussian", waist=3e-4), (40, 13, 8e-5, 3e-5),
     "rs", 1, 1.0, 3),
    ("cswgs_96x64", 96, 64, dict(illumination="gaussian", waist=3e-4), (40, 13, 8e-5, 3e-5),
     "cswgs", 6, 0.125, 4),
    # the 1920x1152 aspect (5:3) at 1/6 size, N = 100 (tensor-core full passes,
    # slab window passes)
    ("cswgs_320x192", 320, 192, dict(illumination="gaussian", waist=1.2e-3), (100, 14, 1e-4, 5e-5),
     "cswgs", 10, 1 / 16, 5),
]


def ref_pupil(p):
    return hs.Pupil(side_px=p.side_px, pitch=p.pitch, wavelength=p.wavelength,
                    focal_length=p.focal_length, illumination=p.illumination, waist=p.waist,
                    seed=p.seed, aperture=p.aperture, xs=p.xs, ys=p.ys, amplitude=p.amplitude,
                    rows=p.rows, cols=p.cols, permutation=p.permutation,
                    sum_amplitude=p.sum_amplitude)


out = {}
for name, w, h, ill, (n, sseed, xy, z), alg, iters, c, seed in CASES:
    p = ours.build_panel(w, h, seed=7, **ill)
    rp = ref_pupil(p)
    rng = np.random.default_rng(sseed)
    spots = hs.SpotSet(x=rng.uniform(-xy, xy, n), y=rng.uniform(-xy, xy, n),
                       z=rng.uniform(-z, z, n), amplitude=rng.uniform(0.5, 1.5, n))
    holo, trace = hs.solve(rp, spots, hs.SolverConfig(alg, iterations=iters, compression=c,
                                                      seed=seed), workers=8)
    rep = hs.quality_report(rp, holo, spots, workers=8)
    recs = trace.records
    d = dict(w=w, h=h, waist=-1.0 if p.waist is None else p.waist, n=n, x=spots.x, y=spots.y,
             z=spots.z, a0=spots.amplitude, iterations=iters, compression=c, seed=seed,
             algorithm=alg, phase=holo.phase, intensities=rep.intensities,
             e=rep.efficiency, u=rep.uniformity, ops=trace.operation_count,
             weights=np.array([r.weights for r in recs]) if recs else np.zeros((0, n)),
             mags=np.array([r.magnitudes for r in recs]) if recs else np.zeros((0, n)),
             sizes=np.array([r.subset_size for r in recs], dtype=np.int64))
    out.update({f"{name}.{k}": np.asarray(v) for k, v in d.items()})
    print(f"{name}: M={p.active_count} e={rep.efficiency:.6f} u={rep.uniformity:.6f} "
          f"ops={trace.operation_count}", flush=True)
np.savez_compressed(os.path.join(HERE, "panel.npz"), **out)
print("wrote", os.path.join(HERE, "panel.npz"))
