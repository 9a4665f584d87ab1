"""Rectangular full panels on the GPU (``build_panel``; config 4 as named in
BASELINE.json: WGS on the 1920 x 1152 panel, N = 1000, I = 30).

* reduced panels against the reference's own solvers run on the same
  geometry (tests/golden/make_panel.py) at the north-star tolerances, in the
  default precision and in fp64 (tight);
* the full 1920 x 1152 panel, which the reference takes about an hour for
  (throughput-only), through size-independent checks: the
  fp32 tensor-core solve against the fp64 FMA solve of the same inputs
  (two independent pixel pipelines), the exact operation count, and the
  first iteration's field magnitudes against the oracle's full-size forward
  projection of the seed hologram.
"""

import numpy as np
import pytest

import oracle
import paper_2003_05293_b200 as hs
from test_gpu_parity import EU_ATOL, INTEN_RTOL, masked_phase_check
from test_panel import CASES, panel_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", CASES)
def test_panel_solve_matches_reference(name):
    p, s, d = panel_case(name)
    cfg = hs.SolverConfig(str(d["algorithm"]), iterations=int(d["iterations"]),
                          compression=float(d["compression"]), seed=int(d["seed"]))
    holo, trace = hs.solve(p, s, cfg)
    rep = hs.quality_report(p, holo, s)
    assert trace.operation_count == int(d["ops"])
    assert [r.subset_size for r in trace.records] == list(d["sizes"])
    assert abs(rep.efficiency - float(d["e"])) <= EU_ATOL
    assert abs(rep.uniformity - float(d["u"])) <= EU_ATOL
    want = d["intensities"]
    assert np.all(np.abs(rep.intensities - want) <= INTEN_RTOL * want), \
        float(np.max(np.abs(rep.intensities - want) / want))
    if trace.records:
        mags = np.array([r.magnitudes for r in trace.records])
        assert np.all(np.abs(mags - d["mags"]) <= 1e-4 * d["mags"])
    r = oracle.solve(p, s.x, s.y, s.z, s.amplitude, str(d["algorithm"]), int(d["iterations"]),
                     float(d["compression"]), int(d["seed"]))
    masked_phase_check(p, s, holo.phase, r["amps"], r["thetas"], None, r["tables"])
    with hs.precision("fp64"):
        h64, t64 = hs.solve(p, s, cfg)
        r64 = hs.quality_report(p, h64, s)
    assert abs(r64.efficiency - float(d["e"])) <= 1e-9 and abs(r64.uniformity - float(d["u"])) <= 1e-9
    assert np.all(np.abs(r64.intensities - want) <= 1e-9 * want)


def test_full_1920x1152_panel_config4():
    """BASELINE configs[3] on the panel itself: WGS, N = 1000, I = 30."""
    p = hs.build_panel(1920, 1152)
    s = hs.random_foci(1000, 4, xy=150e-6)
    holo, trace = hs.wgs(p, s, iterations=30, seed=0)
    rep = hs.quality_report(p, holo, s)
    m = 1920 * 1152
    assert trace.operation_count == hs.predict_ops("wgs", m, 1000, 30) == 30 * m * 1000
    assert hs._lib.plan_for(p).last_precision() == "fp32"   # 2212 pixels per spot
    with hs.precision("fp64"):
        h64, t64 = hs.wgs(p, s, iterations=30, seed=0)
        r64 = hs.quality_report(p, h64, s)
    assert abs(rep.efficiency - r64.efficiency) <= EU_ATOL
    assert abs(rep.uniformity - r64.uniformity) <= EU_ATOL
    assert np.all(np.abs(rep.intensities - r64.intensities) <= INTEN_RTOL * r64.intensities), \
        float(np.max(np.abs(rep.intensities - r64.intensities) / r64.intensities))
    w = np.array([r.weights for r in trace.records])
    w64 = np.array([r.weights for r in t64.records])
    assert np.all(np.abs(w - w64) <= 1e-4 * w64)
    # iteration 1 reads the seed hologram: its magnitudes are the oracle's
    # full-size forward projection of the seed superposition
    tab = oracle.tables(p, s.x, s.y, s.z)
    th0 = np.random.default_rng(0).random(1000) * 2 * np.pi
    seed_phase = oracle.superpose(p, tab, s.amplitude, th0)
    f = oracle.forward(p, tab, seed_phase, 0, m)
    assert np.all(np.abs(trace.records[0].magnitudes - np.abs(f)) <= 1e-4 * np.abs(f))
    assert rep.efficiency > 0.85
