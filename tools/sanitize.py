"""Small solves that launch every pass kernel once, for compute-sanitizer.

    compute-sanitizer --tool racecheck|synccheck|memcheck python tools/sanitize.py

Covers: tables + seed, the slab window pass (hs_slab_kernel, whole- and
half-chunk CTAs), the tcgen05 full pass (hs_umma_kernel, one spot chunk and
the spot-chunked n > 128 variant), the FFMA tile pass (n <= 32), the generic
row-run pass (pixel ranges), the fp64 passes, the far-field probe and the
SLM raster.  Sizes are small: the sanitizer serialises and instruments
every access.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2003_05293_b200 as hs  # noqa: E402

p = hs.build_pupil(128, waist=6e-4)
for n, alg, kw in [(64, "cswgs", dict(iterations=4, compression=0.25)),   # slab + umma
                   (10, "cswgs", dict(iterations=3, compression=0.5)),    # FFMA tiles
                   (200, "wgs", dict(iterations=2)),                      # umma spot chunks
                   (40, "rs", {})]:
    s = hs.random_foci(n, 100 + n, xy=5e-5, z=2e-5)
    with hs.precision("fp32"):
        holo, trace = hs.solve(p, s, hs.SolverConfig(alg, **kw))
        rep = hs.quality_report(p, holo, s)
    print(alg, n, f"e={rep.efficiency:.4f} u={rep.uniformity:.4f}", flush=True)
s = hs.random_foci(24, 5, xy=5e-5, z=2e-5)
with hs.precision("fp64"):
    holo, _ = hs.cswgs(p, s, iterations=3, compression=0.5)
    print("fp64", hs.quality_report(p, holo, s).efficiency, flush=True)
co = hs.SpotCoefficients(np.ones(24), np.zeros(24))
frag = hs.superpose(p, s, co, (100, 900))                          # generic row-run pass
f = hs.forward_project(p, hs.Hologram(np.zeros(p.active_count), p), s, (50, 2000))
img = hs.render_plane(p, holo, 2e-4, 0.0, 16)                         # far-field probe
ras = hs.slm_raster(p, holo)                                          # SLM raster
print("ok", frag.shape, f.shape, np.asarray(img.intensity).shape, np.asarray(ras).shape, flush=True)
