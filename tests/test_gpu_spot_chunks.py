"""The full pass across its spot-count variants, against the CPU oracle on
identical seeded inputs (same tolerances as test_gpu_parity.py), with the
fp32 passes forced (precision "fp32"):

* n = 48, 100   -- tcgen05, one forward spot chunk of np spots (two CTAs per SM);
* n = 120       -- tcgen05, np = 128: the spot-chunked variant (one chunk of
                   128, backward accumulated in groups of 8 k-steps);
* n = 200, 600  -- tcgen05 spot-chunked with several forward chunks (np =
                   256, 1024) on pupils holding >= 512 pixels per spot;
                   test_gpu_umma.py re-runs this file on the FFMA tiles.

WGS runs full passes only; CS-WGS mixes them with window passes.  Fewer
pixels per spot make WGS amplify fp32 rounding (600 random-amplitude spots
on a 256^2 pupil reach 5e-4 in the final intensities, CS-WGS at n = 200
with c = 1/4 2.4e-4 by iteration 4); precision "auto" runs such cases on the
fp64 passes, tested in test_gpu_precision.py::test_auto_precision_ill_conditioned.
"""

import numpy as np
import pytest

import oracle
import paper_2003_05293_b200 as hs
from test_gpu_parity import INTEN_RTOL, masked_phase_check

pytestmark = pytest.mark.gpu


def _spots(n, seed):
    rng = np.random.default_rng(seed)
    amp = rng.uniform(0.5, 1.5, n)
    return hs.SpotSet(x=rng.uniform(-1e-4, 1e-4, n), y=rng.uniform(-1e-4, 1e-4, n),
                      z=rng.uniform(-5e-5, 5e-5, n), amplitude=amp)


CASES = [(alg, n) for n in (48, 100, 120, 200) for alg in ("wgs", "cswgs")] + [("wgs", 600)]
# pupil and CS-WGS compression per n: >= 512 pixels per spot in every window
PUPIL = {48: ("p256u0", 0.25), 100: ("p256u0", 0.25), 120: ("p256u0", 0.25),
         200: ("p512g0", 0.5), 600: ("p1152g0", 1.0)}


@pytest.mark.parametrize("alg,n", CASES)
def test_spot_chunk_variants_match_oracle(pupils, alg, n):
    key, cc = PUPIL[n]
    p = pupils[key]
    s = _spots(n, 1000 + n)
    iters, c = (3, 1.0) if alg == "wgs" else (4, cc)
    cfg = hs.SolverConfig(alg, iterations=iters, compression=c, seed=7)
    with hs.precision("fp32"):
        holo, trace = hs.solve(p, s, cfg)
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, alg, iters, c, 7)
    mags = np.array([rec.magnitudes for rec in trace.records])
    w = np.array([rec.weights for rec in trace.records])
    assert np.all(np.abs(mags - r["mags"]) <= INTEN_RTOL * r["mags"]), \
        float(np.max(np.abs(mags - r["mags"]) / r["mags"]))
    assert np.all(np.abs(w - r["weights"]) <= INTEN_RTOL * r["weights"])
    masked_phase_check(p, s, holo.phase, r["amps"], r["thetas"], tab=r["tables"])
